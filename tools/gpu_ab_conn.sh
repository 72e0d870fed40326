# A/B: CUDA_DEVICE_MAX_CONNECTIONS (hardware work queues shared by the 20 view streams)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2 3; do
  for c in 8 32 16; do
    CUDA_DEVICE_MAX_CONNECTIONS=$c timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/conn_${c}_${rep}.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/conn_${c}_${rep}.json').read().strip().splitlines()[-1]);print('$rep conn=$c', d['ms_per_step'], d['roofline']['in_step']['phases_ms'])"
  done
done
