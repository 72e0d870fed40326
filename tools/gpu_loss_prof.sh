# usage: bash tools/gpu_loss_prof.sh <tag>   (under gpurun; one GPU): time + ncu the loss kernels
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-loss}
python -m paper_2411_14847_b200.build > /dev/null || exit 1
python tools/loss_timing.py 100 > gpurun_out/loss_time_$TAG.json || exit 1
cat gpurun_out/loss_time_$TAG.json
ncu --set full --clock-control none --import-source on -k regex:ssim -s 6 -c 2 -o gpurun_out/prof_loss_$TAG -f \
    python tools/loss_timing.py 1 > gpurun_out/ncu_loss_$TAG.log 2>&1
echo ncu rc=$?
