cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-sweep}
timeout 900 python -m pytest tests -m gpu -q --maxfail=20 -k "not c2_full" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
for P in 1 2 4 8; do
  DASS_FWD_PPT=$P DASS_BWD_PPT=$P timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "c1_full or ragged" > gpurun_out/pytest_${TAG}_ppt$P.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_${TAG}_ppt$P.log
  DASS_FWD_PPT=$P DASS_BWD_PPT=$P timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_ppt$P.json 2> gpurun_out/bench_${TAG}_ppt$P.err
done
tail -3 gpurun_out/pytest_$TAG.log
for P in 1 2 4 8; do tail -1 gpurun_out/pytest_${TAG}_ppt$P.log; python -c "import json,sys; d=json.load(open('gpurun_out/bench_${TAG}_ppt$P.json')); print($P, d['value'], d['ms_per_step'], d['ops_ms_per_step_rank0'], d['roofline']['frac'])"; done
