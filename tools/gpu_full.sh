# Full round check (under gpurun): all GPU tests incl. full-size C2, smoke, the
# default bench line, the reference arm, launch list + one ncu capture.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-full}
timeout 1500 python -m pytest tests -m gpu -q --maxfail=20 > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -3 gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
tail -2 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
cat gpurun_out/bench_$TAG.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?" >> gpurun_out/bench_ref_$TAG.err
cat gpurun_out/bench_ref_$TAG.json
