cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-f2}
CMD2="python bench.py --views 2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-graph --streams 1 --lean"
for k in preprocess preprocess2; do
  case $k in preprocess) SK=2;; preprocess2) SK=3;; esac
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:preprocess_views_kernel -s $SK -c 1 -o gpurun_out/prof_${k}_$TAG -f $CMD2 > /dev/null 2>&1
  python tools/profile_txt.py gpurun_out/prof_${k}_$TAG.ncu-rep "--set full --clock-control none --import-source on -k regex:preprocess_views_kernel -s $SK -c 1" "$CMD2" "2 1352x1014 views of the C3 scene (300k Gaussians)" > gpurun_out/${TAG}_ncu_${k}.txt 2>/dev/null
  grep -E "^kernel|Duration|Registers Per|Executed Instructions|Issue Slots|DRAM Throughput|dram_bytes|Achieved Occ" gpurun_out/${TAG}_ncu_${k}.txt
done
