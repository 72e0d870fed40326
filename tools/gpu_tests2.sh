cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-t}
DASS_PARITY_STATS=gpurun_out/parity_stats_$TAG.json timeout 1800 python -m pytest tests -m gpu -q -rs --durations=12 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
tail -3 gpurun_out/pytest_gpu_$TAG.log; tail -3 gpurun_out/smoke_$TAG.log
