#!/bin/bash
# Build libhszg.so of git revision $1 into ab/lib_$1.so (A/B timing: HSZG_LIB=ab/lib_$1.so python bench.py ...)
set -e
REV=$1
ROOT=$(cd "$(dirname "$0")/.." && pwd)
WT=/tmp/hszg_ab_$REV
rm -rf "$WT"; git -C "$ROOT" worktree prune
git -C "$ROOT" worktree add -f --detach "$WT" "$REV" > /dev/null
mkdir -p "$ROOT/ab"
make -s -j7 -C "$WT/paper_2603_25206_b200/csrc" OUT="$ROOT/ab/lib_$REV.so" BUILD="$WT/build"
git -C "$ROOT" worktree remove --force "$WT"
echo "$ROOT/ab/lib_$REV.so"
