O=gpurun_out/direct; mkdir -p $O
for v in base leanx rtdx0 leanx_rtdx0; do
  if [ $v = base ]; then L=""; else L=tools/variants/$v/libkgp.so; fi
  echo "== $v"
  KGP_LIB=$L timeout 40 python tools/tc_probe.py 65536 33 1 fast matern32 4 30 2>&1 | tail -1
  KGP_LIB=$L timeout 40 python tools/tc_probe.py 65536 64 1 fast matern52 2 30 2>&1 | tail -1
  KGP_LIB=$L timeout 40 python tools/tc_probe.py 65536 17 1 fast gaussian 3 30 2>&1 | tail -1
  KGP_LIB=$L timeout 40 python tools/tc_probe.py 65536 33 2 fast matern32 4 30 2>&1 | tail -1
done
for c in "33 1 fast matern32 4" "64 1 fast matern52 2"; do
  rm -f $O/tr.bin
  KGP_LIB=tools/variants/instr/libkgp.so KGP_TC_TRACE=$O/tr.bin timeout 40 python tools/tc_probe.py 65536 $c 2 > /dev/null 2>&1
  echo "trace $c"; python tools/tc_trace.py $O/tr.bin 2>&1 | tail -4
done
