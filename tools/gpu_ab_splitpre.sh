cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernel_variants.py tests/test_gpu_step.py -q -x > gpurun_out/sp_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/sp_pytest.log; tail -2 gpurun_out/sp_pytest.log
for rep in 1 2 3; do for f in "" "--split-preprocess"; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e $f > gpurun_out/sp.json 2>/dev/null
python -c "
import json;d=json.loads(open('gpurun_out/sp.json').read().strip().splitlines()[-1]);print('$rep [$f]', d['ms_per_step'])"
done; done
