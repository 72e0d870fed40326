cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
cp tools/ab/libdass_B.so paper_2411_14847_b200/libdass.so
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bucket.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --lean --no-graph > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_bucket.csv | head -30
