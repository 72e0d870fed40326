# Bucket sort (B) with the sorts on high-priority streams vs the onesweep sort (A)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2 3; do
  for cfg in "A:" "B:" "B:--sort-chains 20" "A:--sort-chains 20"; do
    v=${cfg%%:*}; f=${cfg#*:}
    cp tools/ab/libdass_$v.so paper_2411_14847_b200/libdass.so
    timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e $f > gpurun_out/b2.json 2>/dev/null
    python -c "
import json;d=json.loads(open('gpurun_out/b2.json').read().strip().splitlines()[-1]);p=d['roofline']['in_step']['phases_ms'];e=p.pop('per_view_ends_ms');print('$rep $v [$f]', d['ms_per_step'], p, 'sort ends', round(min(x[0] for x in e),3), round(max(x[0] for x in e),3))"
  done
done
