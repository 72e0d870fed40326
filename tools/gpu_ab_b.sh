# Parity of tools/ab/libdass_B.so on the render tests, then the interleaved A/B.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
cp tools/ab/libdass_B.so paper_2411_14847_b200/libdass.so; touch paper_2411_14847_b200/libdass.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_step.py -q -x -k "not c5" > gpurun_out/abb_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/abb_pytest.log; tail -2 gpurun_out/abb_pytest.log
grep -q "rc=0" gpurun_out/abb_pytest.log || exit 1
bash tools/gpu_ab_libs.sh 2>&1 | head -6
