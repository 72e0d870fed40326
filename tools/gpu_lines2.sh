cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-l}
timeout 900 python bench.py > gpurun_out/bench_c3_$TAG.json 2> gpurun_out/bench_c3_$TAG.err
timeout 900 python bench.py --nccl-single --emulate 0/8 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_emul8_$TAG.json 2> gpurun_out/bench_emul8_$TAG.err
for c in c3 emul8; do
python -c "
import json;d=json.loads(open('gpurun_out/bench_${c}_$TAG.json').read().strip().splitlines()[-1]);r=d['roofline'];i=r.get('in_step') or {};o=(r.get('other_raster_kernel') or {});oi=o.get('in_step') or {}
print('$c', d['value'], d['ms_per_step'], r['kernel'].split()[0], r['frac'], (r.get('issue_view') or {}).get('frac'), i.get('frac'), i.get('span_frac'), i.get('issue_frac'), 'other', o.get('frac'), oi.get('frac'), oi.get('span_frac'))"
done
