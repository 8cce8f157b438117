for v in base dmin2 dmin0; do
  if [ $v = base ]; then L=""; else L=tools/variants/$v/libkgp.so; fi
  echo "== $v"
  KGP_LIB=$L timeout 40 python tools/tc_probe.py 65536 33 1 fast matern32 4 30 2>&1 | tail -1
  KGP_LIB=$L timeout 40 python tools/tc_probe.py 65536 33 2 fast matern32 4 30 2>&1 | tail -1
  KGP_LIB=$L timeout 40 python tools/tc_probe.py 65536 64 1 fast matern52 2 30 2>&1 | tail -1
  KGP_LIB=$L timeout 40 python tools/tc_probe.py 65536 17 1 fast gaussian 3 30 2>&1 | tail -1
  KGP_LIB=$L timeout 40 python tools/tc_probe.py 65536 17 2 fast gaussian 3 30 2>&1 | tail -1
  KGP_LIB=$L timeout 60 python tools/variant_err.py 16384 33 matern32 4 2>&1 | tail -1
  KGP_LIB=$L timeout 60 python tools/variant_err.py 16384 64 matern52 2 2>&1 | tail -1
  KGP_LIB=$L timeout 60 python tools/variant_err.py 16384 17 gaussian 3 2>&1 | tail -1
done
