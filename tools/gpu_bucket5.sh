cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
cp tools/ab/libdass_B.so paper_2411_14847_b200/libdass.so
CMD2="python bench.py --views 2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-graph --streams 1 --lean"
for k in seg_sort_small bucket_count; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:${k}_kernel -s 2 -c 1 -o gpurun_out/prof_${k} -f $CMD2 > /dev/null 2>&1
python tools/profile_txt.py gpurun_out/prof_${k}.ncu-rep "x" "$CMD2" > gpurun_out/b5_ncu_${k}.txt 2>/dev/null
done
head -45 gpurun_out/b5_ncu_seg_sort_small.txt
