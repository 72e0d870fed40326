# A/B of env knobs on the full (non-lean) bench: bash tools/gpu_ab_env_full.sh "VAR=a W=b" ...
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for cfg in "$@"; do
  for rep in 1 2; do
    env $cfg python bench.py --lean --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('$cfg', d['ms_per_step'])"
  done
done
