cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for L in 0 1; do
  DASS_NO_LISTS=$L timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_ab$L.json 2> gpurun_out/bench_ab$L.err
  python -c "import json; d=json.load(open('gpurun_out/bench_ab$L.json')); print('NO_LISTS=$L', d['value'], d['ops_ms_per_step_rank0'])"
done
CMD2="python bench.py --views 2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-graph --streams 1"
$CMD2 > gpurun_out/plain2_ab.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:render_fwd -s 2 -c 1 -o gpurun_out/prof_fwd_lists -f $CMD2 > gpurun_out/ncu_fwd_lists.log 2>&1; \
ncu --set full --clock-control none --import-source on -k regex:render_bwd_list -s 2 -c 1 -o gpurun_out/prof_bwd_lists -f $CMD2 > gpurun_out/ncu_bwd_lists.log 2>&1
ls gpurun_out | grep lists
