# Split projection: parity tests, then an interleaved A/B against the one-stream projection.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -m paper_2411_14847_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_step.py tests/test_gpu_kernel_variants.py tests/test_abi.py -q -x > gpurun_out/split_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/split_pytest.log
tail -3 gpurun_out/split_pytest.log
bash tools/gpu_ab_flags.sh split "" "--no-split-project"
timeout 600 python tools/timeline.py > gpurun_out/split_timeline.txt 2>&1; tail -30 gpurun_out/split_timeline.txt
timeout 600 python tools/timeline.py 20 0 0 > gpurun_out/split_timeline_off.txt 2>&1; head -3 gpurun_out/split_timeline_off.txt
