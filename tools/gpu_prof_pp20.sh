# ncu --set full of the projection and preprocess launches at the C3 size (one launch = all
# 20 views), for bench.py's hot_path_roofline issue views.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-r02}
CMD3="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-graph --streams 1 --lean"
for k in project_keys project_records preprocess preprocess2; do
  case $k in
    project_keys) RX="project_keys_kernel"; SK=2;; project_records) RX="project_records_kernel"; SK=2;;
    preprocess) RX="preprocess_views_kernel"; SK=2;; preprocess2) RX="preprocess_views_kernel"; SK=3;;
  esac
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$RX -s $SK -c 1 -o gpurun_out/prof_${k}_20v_$TAG -f $CMD3 > /dev/null 2>&1
  python tools/profile_txt.py gpurun_out/prof_${k}_20v_$TAG.ncu-rep "--set full --clock-control none --import-source on -k regex:$RX -s $SK -c 1" "$CMD3" "all 20 1352x1014 views of the C3 scene (300k Gaussians)" > gpurun_out/${TAG}_ncu_${k}_20v.txt 2>/dev/null
  grep -E "^kernel|Duration|Executed Instructions|Issue Slots|Achieved Occ|DRAM Through" gpurun_out/${TAG}_ncu_${k}_20v.txt
done
