cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-v}
timeout 900 python -m pytest tests -m gpu -q --maxfail=20 -k "not c2_full" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -3 gpurun_out/pytest_$TAG.log
for V in "--streams 4" "--streams 1" "--streams 8" "--streams 4 --no-graph"; do
  N=$(echo $V | tr -d ' -')
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e $V > gpurun_out/bench_${TAG}_$N.json 2> gpurun_out/bench_${TAG}_$N.err
  python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_$N.json')); print('$V', d['value'], d['ms_per_step'], d['ops_ms_per_step_rank0'], d['roofline']['frac'], d['gpu_launches'])" || tail -5 gpurun_out/bench_${TAG}_$N.err
done
