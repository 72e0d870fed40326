# Build libdass of a git revision into tools/ab/libdass_A.so (the working tree's
# build goes to tools/ab/libdass_B.so) for tools/gpu_ab_libs.sh.
# usage: bash tools/ab_build.sh [REV=HEAD]
set -e
REV=${1:-HEAD}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
mkdir -p "$ROOT/tools/ab"
rm -rf /tmp/dass_ab_wt && git -C "$ROOT" worktree prune && git -C "$ROOT" worktree add -f /tmp/dass_ab_wt "$REV" >/dev/null
(cd /tmp/dass_ab_wt && python -m paper_2411_14847_b200.build >/dev/null)
cp /tmp/dass_ab_wt/paper_2411_14847_b200/libdass.so "$ROOT/tools/ab/libdass_A.so"
git -C "$ROOT" worktree remove --force /tmp/dass_ab_wt
(cd "$ROOT" && python -m paper_2411_14847_b200.build >/dev/null)
cp "$ROOT/paper_2411_14847_b200/libdass.so" "$ROOT/tools/ab/libdass_B.so"
ls -la "$ROOT/tools/ab"
