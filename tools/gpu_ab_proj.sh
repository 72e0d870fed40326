cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2 3; do
for c in 1 2 4; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --proj-chunks $c > gpurun_out/pj.json 2>/dev/null
python -c "
import json;d=json.loads(open('gpurun_out/pj.json').read().strip().splitlines()[-1]);p=d['roofline']['in_step']['phases_ms'];e=p.pop('per_view_ends_ms');print('$rep proj_chunks=$c', d['ms_per_step'], p)"
done; done
