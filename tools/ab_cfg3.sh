for lib in default paper_2506_20350_b200/csrc/build_prev/libtoepcuda_prev.so default paper_2506_20350_b200/csrc/build_prev/libtoepcuda_prev.so; do
  if [ "$lib" = default ]; then unset TOEPCUDA_LIB; else export TOEPCUDA_LIB=$PWD/$lib; fi
  echo "== $lib"; python tools/bench_configs.py cfg3 2>&1 | tail -1 | grep -o '"solve_ms": [0-9.]*' | tr '\n' ' '; echo
done
