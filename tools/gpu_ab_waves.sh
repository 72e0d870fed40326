# A/B: backward waves with per-wave preprocess chunks (PassOptions.bwd_waves)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernel_variants.py -q -x > gpurun_out/waves_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/waves_pytest.log; tail -2 gpurun_out/waves_pytest.log
for rep in 1 2; do
  for w in 1 2 4 5; do
    timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --bwd-waves $w > gpurun_out/waves_${w}.json 2>/dev/null
    python -c "
import json;d=json.loads(open('gpurun_out/waves_${w}.json').read().strip().splitlines()[-1]);p=d['roofline']['in_step']['phases_ms'];e=p.pop('per_view_ends_ms');print('$rep waves=$w', d['ms_per_step'], p, 'last bwd end', max(x[2] for x in e))"
  done
done
