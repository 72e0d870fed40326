cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -m paper_2411_14847_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_step.py tests/test_abi.py -q -x > gpurun_out/q2_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q2_pytest.log; tail -2 gpurun_out/q2_pytest.log
timeout 900 python bench.py > gpurun_out/q2_bench.json 2> gpurun_out/q2_bench.err; tail -3 gpurun_out/q2_bench.err
python - <<'P'
import json
d=json.loads(open("gpurun_out/q2_bench.json").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d["clocks"], json.dumps(d["roofline"]["in_step"]))
P
