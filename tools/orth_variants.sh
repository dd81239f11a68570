# GMRES cfg2 solve times under orthogonalisation variants (L2 persisting window sizes)
for mb in 0 32 64 96; do
  echo "== persist $mb MB"
  if [ $mb = 0 ]; then python tools/gmres_time.py 2>&1 | tail -2; else TOEP_ORTH_PERSIST_MB=$mb python tools/gmres_time.py 2>&1 | tail -2; fi
done
