# Profiles for profiles/ (under gpurun, 1 GPU): plain bench, then the launch
# list of the same command, then ncu --set full of the two raster kernels.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-r}
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-graph --lean"
$CMD > gpurun_out/plainL_$TAG.json 2> gpurun_out/plainL_$TAG.err || { echo "plain failed"; tail gpurun_out/plainL_$TAG.err; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
CMD2="python bench.py --views 2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-graph --streams 1"
$CMD2 > gpurun_out/plain2_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:render_bwd_list -s 2 -c 1 -o gpurun_out/prof_bwd_$TAG -f $CMD2 > gpurun_out/ncu_bwd_$TAG.log 2>&1; ncu --set full --clock-control none --import-source on -k regex:render_fwd -s 2 -c 1 -o gpurun_out/prof_fwd_$TAG -f $CMD2 > gpurun_out/ncu_fwd_$TAG.log 2>&1
ls -la gpurun_out | grep $TAG
timeout 300 python tools/deform_timing.py > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:deform_fwd_tc -c 1 -o gpurun_out/prof_deformtc_$TAG -f python tools/deform_timing.py > gpurun_out/ncu_deformtc_$TAG.log 2>&1
ls -la gpurun_out | grep $TAG
