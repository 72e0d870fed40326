# ncu --set full of the projection parts and the preprocess parts (one C3 view pair)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-pp}
CMD2="python bench.py --views 2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-graph --streams 1 --lean"
for k in project_keys project_records preprocess1 preprocess2; do
  case $k in
    project_keys) RX="project_keys_kernel";; project_records) RX="project_records_kernel";;
    preprocess1) RX="preprocess_views_kernel<3, 1>";; preprocess2) RX="preprocess_views_kernel<3, 2>";;
  esac
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$RX" -s 2 -c 1 -o gpurun_out/prof_${k}_$TAG -f $CMD2 > /dev/null 2>&1
  python tools/profile_txt.py gpurun_out/prof_${k}_$TAG.ncu-rep "--set full --clock-control none --import-source on -k regex:$RX -s 2 -c 1" "$CMD2" > gpurun_out/${TAG}_ncu_${k}.txt 2>/dev/null
  grep -E "Duration|Registers|Achieved Occ|Issue Slots|DRAM Through|Executed Ins|dram_bytes" gpurun_out/${TAG}_ncu_${k}.txt
done
