# A/B/C… of prebuilt libdass builds (under gpurun), interleaved, on the 10-step bench:
#   bash tools/gpu_ab_multi.sh A v2 v3     (tools/ab/libdass_<name>.so)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2 3; do
  for v in "$@"; do
    cp tools/ab/libdass_$v.so paper_2411_14847_b200/libdass.so
    python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/ab.json')); o=d['ops_ms_per_step_rank0']
print('$v', d['ms_per_step'], 'fwd', o['render_fwd'], 'bwd', o['render_bwd_raster'], 'bin', o['bin_sort'], 'proj', o['project_views'], 'pre', o['render_bwd_preprocess_views'])"
  done
done
