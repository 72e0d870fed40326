# dass_bin_sort_shared against dass_bin_sort on the emulated ranks of 2-, 4- and 8-GPU view
# plans (10, 5 and 2-3 concurrent views): bench.py --shared-sort-min-views 1 (shared) / 99 (plain).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -m paper_2411_14847_b200.build > /dev/null 2>&1
for w in 2 4 8; do
  for m in 1 99 1 99; do
    timeout 600 python bench.py --emulate 0/$w --shared-sort-min-views $m --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/thr.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/thr.json')); print('rank 0 of $w', 'shared' if $m == 1 else 'plain', d['ms_per_step'])"
  done
done
