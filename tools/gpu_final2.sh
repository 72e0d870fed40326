# Round-2 evidence set under gpurun (after the split projection / emit / preprocess work):
# GPU tests (+ parity stats), smoke, every config's bench line, the emulated 8-GPU rank,
# the oracle reference arm, the launch list and ncu --set full summaries.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-fin}
python -m paper_2411_14847_b200.build > /dev/null 2>&1
DASS_PARITY_STATS=gpurun_out/parity_stats_$TAG.json timeout 1800 python -m pytest tests -m gpu -q -rs > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_c3_$TAG.json 2> gpurun_out/bench_c3_$TAG.err
for c in c1 c2 c4 c5; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_${c}_$TAG.json 2> gpurun_out/bench_${c}_$TAG.err
done
timeout 900 python bench.py --nccl-single --emulate 0/8 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_emul8_$TAG.json 2> gpurun_out/bench_emul8_$TAG.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2>/dev/null
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --lean"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > /dev/null 2>&1
CMD2="python bench.py --views 2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-graph --streams 1 --lean"
for k in render_fwd render_bwd onesweep project_keys project_records emit presort_init; do
  case $k in
    render_fwd) RX="render_fwd_tw";; render_bwd) RX="render_bwd_tw";; onesweep) RX="onesweep";;
    project_keys) RX="project_keys_kernel";; project_records) RX="project_records_kernel";;
    preprocess) RX="preprocess_views_kernel<3, 1>";; preprocess2) RX="preprocess_views_kernel<3, 2>";;
    emit) RX="emit_kernel";; presort_init) RX="presort_init_kernel";;
  esac
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$RX" -s 2 -c 1 -o gpurun_out/prof_${k}_$TAG -f $CMD2 > /dev/null 2>&1
  python tools/profile_txt.py gpurun_out/prof_${k}_$TAG.ncu-rep "--set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:$RX' -s 2 -c 1" "$CMD2" > gpurun_out/${TAG}_ncu_${k}.txt 2>/dev/null
done
tail -2 gpurun_out/pytest_gpu_$TAG.log; tail -2 gpurun_out/smoke_$TAG.log
python -c "
import json;d=json.loads(open('gpurun_out/bench_c3_$TAG.json').read().strip().splitlines()[-1]);print(d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks'])"
bash tools/gpu_prof_pre.sh $TAG
bash tools/gpu_prof_pp20.sh $TAG
bash tools/gpu_checked.sh $TAG
