cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
cp tools/ab/libdass_B.so paper_2411_14847_b200/libdass.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_binsort_views.py -q -x -k "sort or bucket or dense or c3 or ragged or tie" > gpurun_out/bucket_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/bucket_pytest.log; tail -2 gpurun_out/bucket_pytest.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bucket.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --lean --no-graph > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_bucket.csv | grep -E "seg_sort|bucket"
bash tools/gpu_ab_libs.sh 2>&1 | head -6
