# f2 GPU check (under gpurun): parity tests + timing of the deformation kernels.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-d}
timeout 900 python -m pytest tests/test_gpu_deform.py -q -x > gpurun_out/pytest_deform_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_deform_$TAG.log
tail -30 gpurun_out/pytest_deform_$TAG.log
timeout 300 python tools/deform_timing.py > gpurun_out/deform_timing_$TAG.json 2>&1; cat gpurun_out/deform_timing_$TAG.json
