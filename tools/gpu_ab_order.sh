# A/B: node creation order of the step graph (PassOptions.phase_major)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernel_variants.py -q -x > gpurun_out/order_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/order_pytest.log; tail -2 gpurun_out/order_pytest.log
for rep in 1 2 3; do
  for f in "" "--phase-major --fwd-join"; do
    timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e $f > gpurun_out/order_${rep}.json 2>/dev/null
    python -c "
import json;d=json.loads(open('gpurun_out/order_${rep}.json').read().strip().splitlines()[-1]);p=d['roofline']['in_step']['phases_ms'];e=p.pop('per_view_ends_ms');print('$rep [$f]', d['ms_per_step'], p)
if $rep==1: print('   ends', e)"
  done
done
