# Full GPU test suite + smoke + one default bench line (tag in $1)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-v}
python -m paper_2411_14847_b200.build > /dev/null 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log; tail -2 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log; tail -2 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_c3_$TAG.json 2> gpurun_out/bench_c3_$TAG.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_c3_$TAG.json').read().strip().splitlines()[-1]);print(d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks'], d['roofline']['frac'], d['roofline']['in_step']['frac'])"
