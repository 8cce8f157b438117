for v in base nodist4 base; do
  if [ $v = base ]; then L=""; else L=tools/variants/$v/libkgp.so; fi
  echo "== $v"
  for r in 1 2; do KGP_LIB=$L timeout 40 python tools/tc_probe.py 65536 32 2 fast gaussian 8 30 2>&1 | tail -1; done
  KGP_LIB=$L timeout 40 python tools/tc_probe.py 65536 51 1 fast gaussian 8 30 2>&1 | tail -1
  KGP_LIB=$L timeout 40 python tools/tc_probe.py 65536 32 2 bf16x3 gaussian 8 30 2>&1 | tail -1
  KGP_LIB=$L timeout 40 python tools/tc_probe.py 65536 32 2 tf32 gaussian 8 30 2>&1 | tail -1
  KGP_LIB=$L timeout 60 python tools/variant_err.py 16384 32 2>&1 | tail -1
  KGP_LIB=$L timeout 60 python tools/variant_err.py 65536 32 2>&1 | tail -1
done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guard.py tests/test_gpu_configs.py tests/test_gpu_gpc.py -q -x -p no:cacheprovider 2>&1 | tail -2
