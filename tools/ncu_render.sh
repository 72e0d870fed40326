# usage: bash tools/ncu_render.sh <tag>   (under gpurun; 1 GPU)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-r}
CMD="python bench.py --views 2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain run failed"; cat gpurun_out/plain_$TAG.log; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:render_bwd_raster -s 2 -c 1 -o gpurun_out/prof_bwd_$TAG -f $CMD > gpurun_out/ncu_bwd_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:render_fwd -s 2 -c 1 -o gpurun_out/prof_fwd_$TAG -f $CMD > gpurun_out/ncu_fwd_$TAG.log 2>&1
ls gpurun_out | grep $TAG
