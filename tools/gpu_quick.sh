# Quick loop: key GPU parity tests, bench line, fwd/bwd ncu.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-q}
DASS_PARITY_STATS=gpurun_out/parity_stats_$TAG.json timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_step.py -m gpu -q -x -k "${2:-c1 or ragged or c2_full or multiview or ties or c3_captured}" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -3 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
python - <<PY
import json
d=json.loads(open("gpurun_out/bench_$TAG.json").read())
print("value", d["value"], "ms", d["ms_per_step"], "ops", d.get("ops_ms_per_step_rank0"))
PY
CMD2="python bench.py --views 2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-graph --streams 1 --lean"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:render_fwd_tw -s 2 -c 1 -o gpurun_out/prof_fwd_$TAG -f $CMD2 > gpurun_out/ncu_fwd_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:render_bwd_tw -s 2 -c 1 -o gpurun_out/prof_bwd_$TAG -f $CMD2 > gpurun_out/ncu_bwd_$TAG.log 2>&1
ls gpurun_out | grep $TAG
