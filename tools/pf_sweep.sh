for v in build_probe build_pf32 build_pf64 build_pf80; do
  echo "== $v"
  TOEPCUDA_LIB=$PWD/paper_2506_20350_b200/csrc/$v/libtoepcuda_probe.so timeout 200 python tools/fused_probe.py
  TOEPCUDA_LIB=$PWD/paper_2506_20350_b200/csrc/$v/libtoepcuda_probe.so timeout 200 python tools/mv_time.py
  TOEPCUDA_LIB=$PWD/paper_2506_20350_b200/csrc/$v/libtoepcuda_probe.so timeout 200 python tools/gmres_time.py
done
