for v in ord1 ord3; do
  L=tools/variants/$v/libkgp.so
  echo "== $v"
  for r in 1 2; do KGP_LIB=$L timeout 40 python tools/tc_probe.py 65536 32 2 fast gaussian 8 30 2>&1 | tail -1; done
  KGP_LIB=$L timeout 40 python tools/tc_probe.py 65536 33 1 fast gaussian 8 30 2>&1 | tail -1
  KGP_LIB=$L timeout 40 python tools/variant_err.py 16384 32 2>&1 | tail -1
done
