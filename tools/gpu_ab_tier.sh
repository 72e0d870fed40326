cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2 3; do for f in "" "--tiered-prio"; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e $f > gpurun_out/t.json 2>/dev/null
python -c "
import json;d=json.loads(open('gpurun_out/t.json').read().strip().splitlines()[-1]);p=d['roofline']['in_step']['phases_ms'];e=p.pop('per_view_ends_ms');print('$rep [$f]', d['ms_per_step'], p, 'fwd ends', round(min(x[1] for x in e),3), round(max(x[1] for x in e),3), 'bwd', round(min(x[2] for x in e),3), round(max(x[2] for x in e),3))"
done; done
