# The shift payload's collective issued before the preprocess SH part joins:
# its GPU tests, the step test, and the emulated 8-GPU rank (one-rank NCCL group) A/B
# against the collective-after-join schedule (--payload full would change the bytes,
# so the A/B toggles bench.py --late-collective).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-ec}
python -m paper_2411_14847_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_kernel_variants.py -m gpu -q -rs > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -3 gpurun_out/pytest_$TAG.log
for r in 1 2; do
for late in 0 1; do
  LATE=""; [ $late = 1 ] && LATE=--late-collective
  timeout 600 python bench.py $LATE --nccl-single --emulate 0/8 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/emul8_${TAG}_late${late}_$r.json 2> gpurun_out/emul8_${TAG}_late${late}_$r.err
  python -c "
import json;d=json.loads(open('gpurun_out/emul8_${TAG}_late${late}_$r.json').read().strip().splitlines()[-1]);print('late=$late', d['ms_per_step'], d.get('allreduce',{}).get('ms'))"
done
done
