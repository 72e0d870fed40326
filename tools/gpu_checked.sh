# The checked build (device bound checks, DASS_CHECKED; compute-sanitizer is closed on this
# pool) under the whole GPU test suite, the sanitizer-driver pass and smoke.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-chk}
cp paper_2411_14847_b200/libdass.so /tmp/libdass_product.so
cp paper_2411_14847_b200/libdass_checked.so paper_2411_14847_b200/libdass.so
touch paper_2411_14847_b200/libdass.so
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/checked_pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/checked_pytest_$TAG.log
timeout 300 python tools/sanitize.py > gpurun_out/checked_sanitize_$TAG.log 2>&1; echo "sanitize rc=$?" >> gpurun_out/checked_sanitize_$TAG.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/checked_smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/checked_smoke_$TAG.log
grep -h "DASS_CHECK failed" gpurun_out/checked_*_$TAG.log | sort | uniq -c | head
tail -2 gpurun_out/checked_pytest_$TAG.log; tail -2 gpurun_out/checked_sanitize_$TAG.log; tail -1 gpurun_out/checked_smoke_$TAG.log
cp /tmp/libdass_product.so paper_2411_14847_b200/libdass.so
