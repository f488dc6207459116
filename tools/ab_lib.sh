#!/bin/bash
# Build the committed csrc of <rev> (default HEAD) into _lib_base/libsrk.so for A/B
# timing against the working tree's _lib/libsrk.so (SRK_LIB_PATH selects a build).
set -e
REV=${1:-HEAD}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d)
git -C "$ROOT" archive "$REV" paper_1810_10197_b200/csrc include | tar -x -C "$TMP"
make -C "$TMP/paper_1810_10197_b200/csrc" -j16 OUTDIR="$ROOT/_lib_base" OBJDIR="$TMP/build" > /dev/null
rm -rf "$TMP"
ls -la "$ROOT/_lib_base/libsrk.so"
