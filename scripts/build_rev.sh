#!/bin/bash
# Build libplx.so from the csrc/ + include/ of a git revision, for an A/B on
# the GPU box:  scripts/build_rev.sh HEAD~1 old  -> paper_2112_05131_b200/libplx_old.so
# (select with PLX_LIB=<path>; the Python side must be ABI-compatible).
set -e
REV=$1; NAME=$2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
T=$(mktemp -d)
git -C "$ROOT" archive "$REV" paper_2112_05131_b200/csrc include | tar -x -C "$T"
make -s -C "$T/paper_2112_05131_b200/csrc" > /dev/null
cp "$T/paper_2112_05131_b200/libplx.so" "$ROOT/paper_2112_05131_b200/libplx_$NAME.so"
rm -rf "$T"
echo "built paper_2112_05131_b200/libplx_$NAME.so from $REV"
