for v in base unr2 gexp unr2gexp; do
  if [ $v = base ]; then L=""; else L=tools/variants/$v/libkgp.so; fi
  echo "== $v"
  KGP_LIB=$L timeout 60 python tools/f64_one.py 4096 17 1 gaussian 3 2>&1 | tail -1
  KGP_LIB=$L timeout 60 python tools/f64_one.py 4096 1 1 gaussian 3 2>&1 | tail -1
  KGP_LIB=$L timeout 60 python tools/f64_one.py 4096 17 2 gaussian 3 2>&1 | tail -1
  KGP_LIB=$L timeout 90 python tools/f64_one.py 65536 32 2 gaussian 8 2>&1 | tail -1
  KGP_LIB=$L timeout 60 python tools/f64_one.py 16384 33 1 matern32 4 2>&1 | tail -1
  KGP_LIB=$L timeout 60 python tools/nlml_time.py fp64 otf 20 2>&1 | tail -1
done
KGP_LIB=tools/variants/unr2gexp/libkgp.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "fp64 or f64 or cfg1 or symmetric or golden" 2>&1 | tail -2
