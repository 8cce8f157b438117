for v in head base rtmma rtxf; do
  if [ $v = base ]; then L=""; else L=tools/variants/$v/libkgp.so; fi
  echo "== $v"
  for r in 1 2; do KGP_LIB=$L timeout 120 python tools/tc_probe.py 65536 33 1 fast matern32 4 30 2>&1 | tail -1; done
  KGP_LIB=$L timeout 120 python tools/tc_probe.py 65536 16 1 fast matern32 4 30 2>&1 | tail -1
  KGP_LIB=$L timeout 120 python tools/tc_probe.py 65536 33 2 fast gaussian 3 30 2>&1 | tail -1
  KGP_LIB=$L timeout 120 python tools/tc_probe.py 65536 64 1 fast matern52 2 30 2>&1 | tail -1
done
echo "== LB knobs (base)"
KGP_TC_LB=2 timeout 120 python tools/tc_probe.py 65536 32 2 fast gaussian 8 30 2>&1 | tail -1
KGP_TC_LB3=1 timeout 120 python tools/tc_probe.py 65536 32 2 fast gaussian 8 30 2>&1 | tail -1
KGP_TC_LB=0 timeout 120 python tools/tc_probe.py 65536 64 2 fast gaussian 8 30 2>&1 | tail -1
timeout 120 python tools/tc_probe.py 65536 64 2 fast gaussian 8 30 2>&1 | tail -1
