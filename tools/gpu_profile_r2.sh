# Round-2 profile set: bench line, launch list of the same command, ncu --set full of
# the raster kernels (one C3 view), summaries written with tools/profile_txt.py.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-r02}
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --lean"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
CMD2="python bench.py --views 2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-graph --streams 1 --lean"
for k in render_fwd render_bwd onesweep project preprocess; do
  case $k in
    render_fwd) RX="render_fwd_tw";; render_bwd) RX="render_bwd_tw";; onesweep) RX="onesweep";; project) RX="project_kernel";; preprocess) RX="preprocess_views_kernel";;
  esac
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$RX -s 2 -c 1 -o gpurun_out/prof_${k}_$TAG -f $CMD2 > gpurun_out/ncu_${k}_$TAG.log 2>&1
  python tools/profile_txt.py gpurun_out/prof_${k}_$TAG.ncu-rep "--set full --clock-control none --import-source on -k regex:$RX -s 2 -c 1" "$CMD2" > gpurun_out/${TAG}_ncu_${k}.txt 2>/dev/null
done
timeout 900 python bench.py --nccl-single --emulate 0/8 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_emul8_$TAG.json 2> gpurun_out/bench_emul8_$TAG.err
ls gpurun_out | grep $TAG
