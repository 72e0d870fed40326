# ncu --set full of the two list-path raster kernels on one C3 view (under gpurun, 1 GPU):
#   bash tools/gpu_ncu_raster.sh <tag>
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-r}
CMD2="python bench.py --views 2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-graph --streams 1"
$CMD2 > gpurun_out/plain2_$TAG.log 2>&1 || { echo "plain run failed"; tail gpurun_out/plain2_$TAG.log; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:"render_bwd_(list|tw)" -s 2 -c 1 -o gpurun_out/prof_bwd_$TAG -f $CMD2 > gpurun_out/ncu_bwd_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"render_fwd" -s 2 -c 1 -o gpurun_out/prof_fwd_$TAG -f $CMD2 > gpurun_out/ncu_fwd_$TAG.log 2>&1
ls -la gpurun_out | grep $TAG
