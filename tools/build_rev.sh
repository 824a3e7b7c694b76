#!/bin/bash
# Builds libcommdet_cuda.so of git revision $1 into build/lib_$2.so (for A/B runs:
# COMMDET_CUDA_LIB=build/lib_$2.so python tools/ab_time.py ...).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
WT=/tmp/wt_$2
rm -rf $WT
git -C $ROOT worktree prune
git -C $ROOT worktree add -f --detach $WT $1 > /dev/null
make -C $WT -j8 lib > /tmp/build_$2.log 2>&1
mkdir -p $ROOT/build
cp $WT/paper_1304_4453_b200/libcommdet_cuda.so $ROOT/build/lib_$2.so
git -C $ROOT worktree remove --force $WT
echo "built build/lib_$2.so from $1"
