# dass_bin_sort_shared in the multi-view step (B, working tree) against HEAD (A): parity with B,
# then interleaved A/B of the C3 step and of C2 (one view: plain dass_bin_sort in both).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-sh}
cp tools/ab/libdass_B.so paper_2411_14847_b200/libdass.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_step.py tests/test_gpu_kernel_variants.py -q -m gpu > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -n 3 gpurun_out/pytest_$TAG.log
for v in A B A B A B; do
  cp tools/ab/libdass_$v.so paper_2411_14847_b200/libdass.so
  timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_$TAG.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab_$TAG.json')); o=d['ops_ms_per_step_rank0']; ph=d['roofline']['in_step']['phases_ms']
print('$v c3', d['ms_per_step'], 'sort', o['bin_sort'], 'sort_phase', ph['sort'])"
done
for v in A B A B; do
  cp tools/ab/libdass_$v.so paper_2411_14847_b200/libdass.so
  timeout 600 python bench.py --config c2 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_$TAG.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab_$TAG.json')); print('$v c2', d['ms_per_step'])"
done
cp tools/ab/libdass_B.so paper_2411_14847_b200/libdass.so
