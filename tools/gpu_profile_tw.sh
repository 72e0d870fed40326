# Profiles for profiles/ (under gpurun, 1 GPU): the launch list of the lean bench,
# then ncu --set full of the two TW raster kernels on one view.  bash tools/gpu_profile_tw.sh <tag>
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-r}
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-graph --lean"
$CMD > gpurun_out/plainL_$TAG.json 2> gpurun_out/plainL_$TAG.err || { echo "plain failed"; tail gpurun_out/plainL_$TAG.err; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
bash tools/gpu_ncu_raster.sh $TAG
