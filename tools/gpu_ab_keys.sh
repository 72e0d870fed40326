cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
cp tools/ab/libdass_B.so paper_2411_14847_b200/libdass.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_binsort_views.py tests/test_gpu_step.py -q -x > gpurun_out/keys_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/keys_pytest.log; tail -2 gpurun_out/keys_pytest.log
grep -q "rc=0" gpurun_out/keys_pytest.log || exit 1
for rep in 1 2 3; do for v in A B; do
cp tools/ab/libdass_$v.so paper_2411_14847_b200/libdass.so
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/k.json 2>/dev/null
python -c "
import json;d=json.loads(open('gpurun_out/k.json').read().strip().splitlines()[-1]);o=d['ops_ms_per_step_rank0'];print('$rep $v', d['ms_per_step'], 'proj', o['project_views'])"
done; done
