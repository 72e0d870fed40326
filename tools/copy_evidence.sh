# Copy one tools/gpu_final2.sh run (gpurun_out/*_TAG*) into the committed profiles/r02_* names.
# usage: bash tools/copy_evidence.sh TAG
set -e
T=$1; G=gpurun_out; P=profiles
for c in c1 c2 c3 c4 c5; do cp $G/bench_${c}_$T.json $P/r02_bench_$c.json; done
cp $G/bench_emul8_$T.json $P/r02_bench_c3_emulate_0of8_nccl1.json
cp $G/bench_ref_$T.json $P/r02_bench_reference_c3.json
cp $G/checked_pytest_$T.log $P/r02_checked_pytest_gpu.log
cp $G/checked_sanitize_$T.log $P/r02_checked_sanitize.log
cp $G/checked_smoke_$T.log $P/r02_checked_smoke.log
cp $G/pytest_gpu_$T.log $P/r02_pytest_gpu.log
cp $G/smoke_$T.log $P/r02_smoke.log
cp $G/parity_stats_$T.json $P/r02_parity_stats.json
python tools/launch_summary.py $G/launches_$T.csv > $P/r02_launches.txt
for f in $G/${T}_ncu_*.txt; do cp $f $P/r02_ncu_${f#$G/${T}_ncu_}; done
git -C "$(dirname "$0")/.." status --short profiles | head -40
