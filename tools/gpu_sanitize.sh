# compute-sanitizer over tools/sanitize.py, one tool after another.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-san}
timeout 300 python tools/sanitize.py > gpurun_out/sanitize_plain_$TAG.log 2>&1; echo "plain rc=$?" >> gpurun_out/sanitize_plain_$TAG.log
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 python tools/sanitize.py > gpurun_out/sanitize_${tool}_$TAG.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_${tool}_$TAG.log
  tail -4 gpurun_out/sanitize_${tool}_$TAG.log
done
