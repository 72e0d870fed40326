# A/B of env knobs on the 10-step bench, 3 interleaved repeats (under gpurun):
#   bash tools/gpu_ab_env3.sh "VAR=a" "VAR=b" ...
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2 3; do
  for cfg in "$@"; do
    env $cfg python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/ab.json')); o=d['ops_ms_per_step_rank0']
print('$cfg', d['ms_per_step'], 'fwd', o['render_fwd'], 'bwd', o['render_bwd_raster'])"
  done
done
