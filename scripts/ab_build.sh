#!/bin/bash
# Build libsmcsd.so of git revision $1 as paper_2604_15672_b200/libsmcsd_ab.so (A/B timing in
# one GPU call: SMCSD_LIB_OVERRIDE=<that .so> python scripts/time_k1.py).  The ABI of both
# revisions must match what the current Python binding expects.
set -e
REV=${1:-HEAD}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d)
git -C "$ROOT" archive "$REV" paper_2604_15672_b200/csrc include | tar -x -C "$TMP"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
    -shared -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -I "$TMP/include" \
    -I "$TMP/paper_2604_15672_b200/csrc" "$TMP/paper_2604_15672_b200/csrc/smcsd_api.cu" \
    -o "$ROOT/paper_2604_15672_b200/libsmcsd_ab.so"
rm -rf "$TMP"
echo "built libsmcsd_ab.so from $REV"
