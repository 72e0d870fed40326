cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for M in 16 12 8; do
  DASS_BWD_MINB=$M timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_minb$M.json 2> gpurun_out/bench_minb$M.err
  python -c "import json; d=json.load(open('gpurun_out/bench_minb$M.json')); print($M, d['value'], d['ops_ms_per_step_rank0'])"
done
