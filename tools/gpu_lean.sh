O=gpurun_out/lean; mkdir -p $O
for v in base nolean base; do
  if [ $v = base ]; then L=""; else L=tools/variants/$v/libkgp.so; fi
  echo "== $v"
  for r in 1 2; do KGP_LIB=$L timeout 120 python tools/tc_probe.py 65536 32 2 fast gaussian 8 30 2>&1 | tail -1; done
  KGP_LIB=$L timeout 120 python tools/tc_probe.py 65536 33 1 fast matern32 4 30 2>&1 | tail -1
done
timeout 120 python tools/variant_err.py 16384 32 2>&1 | tail -1
echo "== trace (instr build)"
KGP_LIB=tools/variants/instr/libkgp.so KGP_TC_TRACE=$O/tr.bin timeout 120 python tools/tc_probe.py 65536 32 2 fast gaussian 8 3 2>&1 | tail -1
python tools/tc_trace.py $O/tr.bin 2>&1 | tail -4
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guard.py tests/test_gpu_configs.py -q -x -p no:cacheprovider 2>&1 | tail -3
