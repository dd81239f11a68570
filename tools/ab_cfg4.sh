#!/bin/bash
# same-box A/B of cfg4 (and cfg2) GMRES between the in-tree library and the committed one (tools/build_head.sh)
for lib in default paper_2506_20350_b200/csrc/build_prev/libtoepcuda_prev.so default paper_2506_20350_b200/csrc/build_prev/libtoepcuda_prev.so; do
  if [ "$lib" = default ]; then unset TOEPCUDA_LIB; else export TOEPCUDA_LIB=$PWD/$lib; fi
  echo "== $lib"; python tools/bench_configs.py cfg4 2>&1 | grep -o '"ms": [0-9.]*' | tr '\n' ' '; echo
done
