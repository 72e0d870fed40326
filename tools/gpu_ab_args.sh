# A/B of bench.py arguments (under gpurun): bash tools/gpu_ab_args.sh "--streams 3" "--streams 4" ...
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for cfg in "$@"; do
  for rep in 1 2; do
    python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --lean $cfg > gpurun_out/ab.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('$cfg', d['ms_per_step'], d['value'])"
  done
done
