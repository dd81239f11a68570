#!/bin/bash
# Build the committed (HEAD) library into paper_2506_20350_b200/csrc/build_prev/libtoepcuda_prev.so for
# same-box A/B runs against the working tree (tools/ab.sh default paper_.../build_prev/libtoepcuda_prev.so).
set -e
R=$(cd "$(dirname "$0")/.." && pwd)
T=$(mktemp -d)
git -C "$R" archive HEAD paper_2506_20350_b200/csrc include | tar -x -C "$T"
make -C "$T/paper_2506_20350_b200/csrc" -j8 > /dev/null
mkdir -p "$R/paper_2506_20350_b200/csrc/build_prev"
cp "$T/paper_2506_20350_b200/libtoepcuda.so" "$R/paper_2506_20350_b200/csrc/build_prev/libtoepcuda_prev.so"
rm -rf "$T"
