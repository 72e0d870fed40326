cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
cp paper_2411_14847_b200/libdass_checked.so /tmp/chk.so
cp /tmp/chk.so paper_2411_14847_b200/libdass.so; touch paper_2411_14847_b200/libdass.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_binsort_views.py tests/test_gpu_step.py -q -x -k "not c5" > gpurun_out/se_pytest_chk.log 2>&1; echo "checked pytest rc=$?" >> gpurun_out/se_pytest_chk.log; tail -2 gpurun_out/se_pytest_chk.log
grep -h "DASS_CHECK failed" gpurun_out/se_pytest_chk.log | head -3
cp tools/ab/libdass_B.so paper_2411_14847_b200/libdass.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_binsort_views.py tests/test_gpu_step.py tests/test_gpu_kernel_variants.py -q -x > gpurun_out/se_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/se_pytest.log; tail -2 gpurun_out/se_pytest.log
grep -q "rc=0" gpurun_out/se_pytest.log || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_se.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --lean --no-graph > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_se.csv | grep -E "emit|scan|presort|onesweep|finalize"; timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "c5 or pair_key" > gpurun_out/se_c5.log 2>&1; tail -1 gpurun_out/se_c5.log
bash tools/gpu_ab_libs.sh 2>&1 | head -6
