#!/bin/bash
# A/B timing of library variants: tools/ab.sh lib1.so lib2.so ...  ("default" = the in-tree library)
for lib in "$@"; do
  echo "== $lib"
  if [ "$lib" = default ]; then unset TOEPCUDA_LIB; else export TOEPCUDA_LIB=$PWD/$lib; fi
  case "$lib" in *probe*) timeout 200 python tools/fused_probe.py 2>&1 | head -4;; esac
  for r in 1 2; do timeout 200 python tools/mv_time.py; done
  timeout 200 python tools/gmres_time.py 2>&1 | grep -v orth-gram
done
