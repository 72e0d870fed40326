cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
cp tools/ab/libdass_B.so paper_2411_14847_b200/libdass.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_binsort_views.py tests/test_gpu_step.py tests/test_gpu_kernel_variants.py -q -x > gpurun_out/emit_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/emit_pytest.log; tail -2 gpurun_out/emit_pytest.log
grep -q "rc=0" gpurun_out/emit_pytest.log || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_emit.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --lean --no-graph > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_emit.csv | grep -E "emit|onesweep|presort|tile_scan|finalize"
for rep in 1 2 3; do for v in A B; do
cp tools/ab/libdass_$v.so paper_2411_14847_b200/libdass.so
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/k.json 2>/dev/null
python -c "
import json;d=json.loads(open('gpurun_out/k.json').read().strip().splitlines()[-1]);o=d['ops_ms_per_step_rank0'];p=d['roofline']['in_step']['phases_ms'];print('$rep $v', d['ms_per_step'], 'sort', o['bin_sort'], 'phase', p['sort'])"
done; done
