# Interleaved A/B/C of tools/ab/libdass_{A,B,C}.so on the C3 step (under gpurun).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in A B C A B C A B C; do
  cp tools/ab/libdass_$v.so paper_2411_14847_b200/libdass.so
  timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab.json')); o=d['ops_ms_per_step_rank0']
print('$v', d['ms_per_step'], 'fwd', o['render_fwd'], 'bwd', o['render_bwd_raster'], 'sort', o['bin_sort'], 'proj', o['project_views'], 'pre', o['render_bwd_preprocess_views'], 'phase', d['roofline']['in_step']['phases_ms']['sort'])"
done
