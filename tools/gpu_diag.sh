O=gpurun_out/diag; mkdir -p $O
L=tools/variants/instr/libkgp.so
for dbg in 0 16 32 48 4 1 2; do
  echo "== KGP_TC_DEBUG=$dbg"
  KGP_LIB=$L KGP_TC_DEBUG=$dbg timeout 120 python tools/tc_probe.py 65536 32 2 fast gaussian 8 20 2>&1 | tail -1
  rm -f $O/tr$dbg.bin
  KGP_LIB=$L KGP_TC_DEBUG=$dbg KGP_TC_TRACE=$O/tr$dbg.bin timeout 120 python tools/tc_probe.py 65536 32 2 fast gaussian 8 2 > /dev/null 2>&1
  python tools/tc_trace.py $O/tr$dbg.bin 2>&1 | tail -3
done
