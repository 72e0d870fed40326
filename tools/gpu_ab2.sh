# A/B of two prebuilt libdass builds (under gpurun): tools/ab/libdass_A.so vs
# tools/ab/libdass_B.so, alternating, on the 10-step bench; B stays in-tree and
# the GPU parity tests run against it.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in A B A B A B; do
  cp tools/ab/libdass_$v.so paper_2411_14847_b200/libdass.so
  python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab.json')); o=d['ops_ms_per_step_rank0']
print('$v', d['ms_per_step'], 'fwd', o['render_fwd'], 'bwd', o['render_bwd_raster'])"
done
cp tools/ab/libdass_B.so paper_2411_14847_b200/libdass.so
touch paper_2411_14847_b200/libdass.so
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
