# Pair passes on a fixed looping grid: interleaved A/B/C of tools/ab libraries built with different
# pair grids (blocks/SM then PAIR_GRID blocks; first run: A = one block per capacity tile, B = 4/SM, C = 2/SM;
# second: A = 2/SM, B = 1/SM, C = 3/SM; third: A = 148, B = 74, C = 104 blocks; fourth, with 74: A = HEAD,
# B = finalize on 148 blocks in the shared sort, C = finalize and emission on 148).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-pg}
for v in B C; do
  cp tools/ab/libdass_$v.so paper_2411_14847_b200/libdass.so
  timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_step.py -q -m gpu > gpurun_out/pytest_${TAG}_$v.log 2>&1; echo "$v pytest rc=$?"; tail -n 1 gpurun_out/pytest_${TAG}_$v.log
done
bash tools/gpu_ab_libs3.sh
