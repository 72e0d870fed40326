# Interleaved A/B of bench.py flag sets on the C3 step (3 repeats each).
# usage: bash tools/gpu_ab_flags.sh TAG "flagsA" "flagsB" ...
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=$1; shift
for rep in 1 2 3; do
  i=0
  for f in "$@"; do
    timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --lean $f > gpurun_out/ab_${TAG}_${i}_${rep}.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/ab_${TAG}_${i}_${rep}.json'));print('$rep', '[$f]', d['ms_per_step'])"
    i=$((i+1))
  done
done
