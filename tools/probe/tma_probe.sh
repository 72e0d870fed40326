nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/tma_probe tools/probe/tma_probe.cu || exit 1
for a in "32 32 1 -4 0 3" "32 32 1 3 0 3" "32 32 1 0 -5 3" "52 50 3 -8 -5 3" "52 50 3 24 30 0" "32 32 1 1 0 0" "32 32 1 -1 0 0" "32 32 1 4 4 0"; do
  timeout 20 /tmp/tma_probe $a
done
