for v in base cap32; do
  if [ $v = base ]; then L=""; else L=tools/variants/$v/libkgp.so; fi
  echo "== $v"
  KGP_LIB=$L timeout 90 python tools/f64_one.py 65536 32 2 gaussian 8 2>&1 | tail -1
  KGP_LIB=$L timeout 60 python tools/f64_one.py 16384 51 2 gaussian 8 2>&1 | tail -1
  KGP_LIB=$L timeout 60 python tools/f64_one.py 16384 33 2 matern32 4 2>&1 | tail -1
  KGP_LIB=$L timeout 60 python tools/f64_one.py 16384 28 2 matern52 2 2>&1 | tail -1
done
KGP_LIB=tools/variants/cap32/libkgp.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -p no:cacheprovider -k "fp64 or f64 or golden or cfg" 2>&1 | tail -2
