# A/B of two builds (full bench, op timings): A = in-tree, B = tools/ab/libdass_B.so
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
cp paper_2411_14847_b200/libdass.so tools/ab/libdass_A.so
for v in A B A B; do
  cp tools/ab/libdass_$v.so paper_2411_14847_b200/libdass.so
  python bench.py --no-e2e --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab.json')); o=d['ops_ms_per_step_rank0']
print('$v', d['ms_per_step'], {k: round(v, 3) for k, v in o.items()})"
done
cp tools/ab/libdass_B.so paper_2411_14847_b200/libdass.so
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
