cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in A B; do
cp tools/ab/libdass_$v.so paper_2411_14847_b200/libdass.so
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b6.json 2>/dev/null
python -c "
import json;d=json.loads(open('gpurun_out/b6.json').read().strip().splitlines()[-1]);p=d['roofline']['in_step']['phases_ms'];e=p.pop('per_view_ends_ms');print('$v', d['ms_per_step'], p); print(' sort ends', sorted(round(x[0],3) for x in e)); print(' fwd ends', sorted(round(x[1],3) for x in e))"
done
