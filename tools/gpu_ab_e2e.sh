# Interleaved A/B of the full C3 bench line (device value and e2e) for tools/ab/libdass_{A,B}.so.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-e2e}
for v in A B A B; do
  cp tools/ab/libdass_$v.so paper_2411_14847_b200/libdass.so
  timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ab_$TAG.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab_$TAG.json'))
print('$v', d['value'], d['ms_per_step'], 'e2e', round(d['e2e']['value'], 1), d['e2e']['ms_per_step'])"
done
