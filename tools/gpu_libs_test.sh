# Run a pytest selection against several prebuilt libdass builds (under gpurun):
#   bash tools/gpu_libs_test.sh "<pytest -k expr>" A v1 v2 ...   (tools/ab/libdass_<name>.so)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
K="$1"; shift
for v in "$@"; do
  cp tools/ab/libdass_$v.so paper_2411_14847_b200/libdass.so
  echo "== $v"
  timeout 600 python -m pytest tests -m gpu -q -k "$K" 2>&1 | grep -E "^E   .*Error|passed|failed" | head -6
done
