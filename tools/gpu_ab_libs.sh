# Interleaved A/B of tools/ab/libdass_{A,B}.so on the C3 step (under gpurun), then the
# parity tests with B in place.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in A B A B A B; do
  cp tools/ab/libdass_$v.so paper_2411_14847_b200/libdass.so
  timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab.json')); o=d['ops_ms_per_step_rank0']
print('$v', d['ms_per_step'], 'fwd', o['render_fwd'], 'bwd', o['render_bwd_raster'], 'sort', o['bin_sort'], 'proj', o['project_views'], 'pre', o['render_bwd_preprocess_views'])"
done
cp tools/ab/libdass_B.so paper_2411_14847_b200/libdass.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_step.py -q -x -m gpu 2>&1 | tail -1
