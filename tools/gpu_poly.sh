O=gpurun_out/poly; mkdir -p $O
for v in base poly2 poly4 poly6 poly8; do
  if [ $v = base ]; then L=""; else L=tools/variants/$v/libkgp.so; fi
  echo "== $v"
  for r in 1 2; do KGP_LIB=$L timeout 120 python tools/tc_probe.py 65536 32 2 fast gaussian 8 30 2>&1 | tail -1; done
  KGP_LIB=$L timeout 120 python tools/variant_err.py 16384 32 2>&1 | tail -1
done
