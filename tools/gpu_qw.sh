cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for CFG in "4 16" "2 8" "4 8" "2 16"; do
  set -- $CFG
  DASS_FWD_PPT=$1 DASS_FWD_QW=$2 DASS_BWD_PPT=$1 DASS_BWD_QW=$2 timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "c1_full or ragged" > gpurun_out/pyt_qw_$1_$2.log 2>&1
  echo "PPT=$1 QW=$2 tests: $(tail -1 gpurun_out/pyt_qw_$1_$2.log)"
  DASS_FWD_PPT=$1 DASS_FWD_QW=$2 DASS_BWD_PPT=$1 DASS_BWD_QW=$2 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_qw_$1_$2.json 2> gpurun_out/bench_qw_$1_$2.err
  python -c "import json; d=json.load(open('gpurun_out/bench_qw_$1_$2.json')); print('  ', d['value'], d['ms_per_step'], d['ops_ms_per_step_rank0'])" || tail -3 gpurun_out/bench_qw_$1_$2.err
done
