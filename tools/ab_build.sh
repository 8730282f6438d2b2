#!/bin/bash
# Build libbm_b200.so of a git revision into abtmp/lib_<name>.so (same-box A/B
# with BM_LIB_PATH): tools/ab_build.sh <rev> <name>
set -e
REV=$1; NAME=$2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
WT=/tmp/bm_ab_$NAME
rm -rf "$WT"; git -C "$ROOT" worktree add -f --detach "$WT" "$REV" >/dev/null 2>&1
(cd "$WT" && python -m paper_2601_01405_b200.build >/dev/null)
mkdir -p "$ROOT/abtmp"; cp "$WT/paper_2601_01405_b200/libbm_b200.so" "$ROOT/abtmp/lib_$NAME.so"
git -C "$ROOT" worktree remove --force "$WT"
echo "abtmp/lib_$NAME.so"
