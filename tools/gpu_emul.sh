# Per-rank step time of a W-GPU view plan on one GPU (under gpurun), for env configs:
#   bash tools/gpu_emul.sh "R/W" "VAR=a" "VAR=b" ...
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
RW=$1; shift
for cfg in "$@"; do
  env $cfg python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --emulate $RW > gpurun_out/em.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/em.json'))
print('$RW $cfg', d['ms_per_step'], d['value'], d['config'].get('parallelism'))"
done
