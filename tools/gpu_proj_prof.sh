# usage: bash tools/gpu_proj_prof.sh   (under gpurun): ncu --set full of project_views + preprocess_views on C3
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -m paper_2411_14847_b200.build > /dev/null || exit 1
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-graph --lean"
$CMD > gpurun_out/pp_plain.json 2> gpurun_out/pp_plain.err || { tail gpurun_out/pp_plain.err; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:"project|preprocess" -c 4 \
    -o gpurun_out/prof_pp -f $CMD > gpurun_out/ncu_pp.log 2>&1
echo ncu rc=$?
