# usage: bash tools/ncu_profile.sh <tag>   (run under gpurun; one GPU)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-r01}
CMD="python bench.py --views 2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:render_bwd_raster -s 2 -c 1 -o gpurun_out/prof_bwd_$TAG -f $CMD > gpurun_out/ncu_bwd_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:render_fwd -s 2 -c 1 -o gpurun_out/prof_fwd_$TAG -f $CMD > gpurun_out/ncu_fwd_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:onesweep -s 12 -c 2 -o gpurun_out/prof_sort_$TAG -f $CMD > gpurun_out/ncu_sort_$TAG.log 2>&1
CMD20="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
$CMD20 > gpurun_out/plain20_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD20 > gpurun_out/ncu_launch_$TAG.log 2>&1
ls -la gpurun_out
