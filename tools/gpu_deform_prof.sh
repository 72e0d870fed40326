# usage: bash tools/gpu_deform_prof.sh   (under gpurun): f2 timing + one ncu --set full of each bwd kernel
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -m paper_2411_14847_b200.build > /dev/null || exit 1
timeout 300 python tools/deform_timing.py || exit 1
ncu --set full --clock-control none --import-source on -k regex:"^deform_bwd_kernel" -c 1 \
    -o gpurun_out/prof_deform_bwd -f python tools/deform_timing.py > gpurun_out/ncu_deform.log 2>&1
echo ncu rc=$?
