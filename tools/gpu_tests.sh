cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/nvsmi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q --maxfail=20 -k "not c2_full" > gpurun_out/pytest_gpu1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu1.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke1.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke1.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo "bench rc=$?" >> gpurun_out/bench1.err
tail -5 gpurun_out/pytest_gpu1.log
