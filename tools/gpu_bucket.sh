# Bucket sort: binsort parity first (bit-exact), then the interleaved A/B (A = previous sort).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
cp tools/ab/libdass_B.so paper_2411_14847_b200/libdass.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_binsort_views.py -q -x -k "sort or bucket or dense or c3 or ragged or tie" > gpurun_out/bucket_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/bucket_pytest.log; tail -3 gpurun_out/bucket_pytest.log
grep -q "rc=0" gpurun_out/bucket_pytest.log || exit 1
bash tools/gpu_ab_libs.sh
python - <<'P'
P
timeout 600 python tools/timeline.py > gpurun_out/bucket_timeline.txt 2>&1; head -4 gpurun_out/bucket_timeline.txt
