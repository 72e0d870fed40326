# A/B of bench.py arguments without --lean (under gpurun)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for cfg in "$@"; do
  python bench.py --no-e2e --no-cpu-baseline $cfg > gpurun_out/ab.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('$cfg', d['ms_per_step'], d['value'])"
done
