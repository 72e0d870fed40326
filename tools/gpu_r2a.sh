# Round-2 check: GPU parity (with measured tie/κ stats), smoke, bench, fwd ncu source profile.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-r2a}
DASS_PARITY_STATS=gpurun_out/parity_stats_$TAG.json timeout 1800 python -m pytest tests -m gpu -q -rs --durations=15 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
CMD2="python bench.py --views 2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-graph --streams 1 --lean"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:render_fwd -s 2 -c 1 -o gpurun_out/prof_fwd_$TAG -f $CMD2 > gpurun_out/ncu_fwd_$TAG.log 2>&1
tail -3 gpurun_out/pytest_gpu_$TAG.log; tail -3 gpurun_out/smoke_$TAG.log; head -c 400 gpurun_out/bench_$TAG.json; tail -2 gpurun_out/bench_$TAG.err
