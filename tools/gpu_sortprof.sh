cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-s}
CMD2="python bench.py --views 2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-graph --streams 1 --lean"
timeout 600 ncu --metrics gpu__time_duration.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes.sum,launch__grid_size --clock-control none --csv -k regex:"tile_|onesweep|presort|emit|finalize|scan" $CMD2 > gpurun_out/sortprof_$TAG.csv 2> gpurun_out/sortprof_$TAG.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"tile_segsort|tile_scatter|tile_count" -s 3 -c 3 -o gpurun_out/prof_sort_$TAG -f $CMD2 > gpurun_out/ncu_sort_$TAG.log 2>&1
