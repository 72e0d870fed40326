# Every config's bench line (C1-C5, the emulated rank 0 of 8) under gpurun.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-lines}
timeout 900 python bench.py > gpurun_out/bench_c3_$TAG.json 2> gpurun_out/bench_c3_$TAG.err
for c in c1 c2 c4 c5; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_${c}_$TAG.json 2> gpurun_out/bench_${c}_$TAG.err
done
timeout 900 python bench.py --nccl-single --emulate 0/8 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_emul8_$TAG.json 2> gpurun_out/bench_emul8_$TAG.err
for c in c1 c2 c3 c4 c5 emul8; do
python -c "
import json;d=json.loads(open('gpurun_out/bench_${c}_$TAG.json').read().strip().splitlines()[-1]);r=d['roofline'];i=r.get('in_step') or {};o=(r.get('other_raster_kernel') or {});oi=o.get('in_step') or {}
print('$c', d['value'], d['ms_per_step'], r['kernel'].split()[0], r['frac'], i.get('frac'), i.get('span_frac'), 'other', o.get('frac'), oi.get('frac'), oi.get('span_frac'))"
done
