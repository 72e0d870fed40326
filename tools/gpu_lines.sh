# Bench lines of every BASELINE.json config (C3 is the default line).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-l}
for c in c1 c2 c4 c5; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_${c}_$TAG.json 2> gpurun_out/bench_${c}_$TAG.err; echo "$c rc=$?" >> gpurun_out/bench_${c}_$TAG.err
  tail -1 gpurun_out/bench_${c}_$TAG.err
done
timeout 600 python bench.py --impl reference --config c1 --steps 5 --warmup 2 > gpurun_out/bench_ref_c1_$TAG.json 2>/dev/null
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_c3_$TAG.json 2>/dev/null
