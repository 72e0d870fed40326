# A/B of two libdass builds on the step and its serial ends (under gpurun):
# A = in-tree .so, B = tools/ab/libdass_B.so; then the parity tests on B
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
cp paper_2411_14847_b200/libdass.so tools/ab/libdass_A.so
for v in A B A B A B; do
  cp tools/ab/libdass_$v.so paper_2411_14847_b200/libdass.so
  python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab.json')); o=d['ops_ms_per_step_rank0']
print('$v', d['ms_per_step'], 'proj', o['project_views'], 'pre', o['render_bwd_preprocess_views'])"
done
cp tools/ab/libdass_B.so paper_2411_14847_b200/libdass.so
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
