# usage: bash tools/gpu_loss_ab.sh   (under gpurun): loss parity + timing per DASS_LOSS_VS / DASS_LOSS_TMA
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -m paper_2411_14847_b200.build > /dev/null || exit 1
python -m pytest tests/test_gpu_parity.py -q -k fidelity 2>&1 | tail -2
DASS_LOSS_TMA=0 python -m pytest tests/test_gpu_parity.py -q -k fidelity 2>&1 | tail -2
for rep in 1 2; do
  for tma in 1 0; do
    for vs in 4 5 6; do
      echo "TMA=$tma VS=$vs $(DASS_LOSS_TMA=$tma DASS_LOSS_VS=$vs python tools/loss_timing.py 200)"
    done
  done
done
if [ -n "$PROF" ]; then
  DASS_LOSS_VS=$PROF ncu --set full --clock-control none --import-source on -k regex:ssim -s 6 -c 2 \
    -o gpurun_out/prof_loss_$PROF -f python tools/loss_timing.py 1 > gpurun_out/ncu_loss.log 2>&1
  echo ncu rc=$?
fi
