for v in base symfg; do
  if [ $v = base ]; then L=""; else L=tools/variants/$v/libkgp.so; fi
  echo "== $v"
  for r in 1 2; do KGP_LIB=$L timeout 60 python tools/f64_one.py 4096 1 1 gaussian 3 2>&1 | tail -1; done
  KGP_LIB=$L timeout 60 python tools/f64_one.py 16384 2 1 gaussian 3 2>&1 | tail -1
  KGP_LIB=$L timeout 120 python tools/nlml_time.py fp64 otf 30 2>&1 | tail -1
done
KGP_LIB=tools/variants/symfg/libkgp.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "symmetric or cfg1 or fixed or nlml" 2>&1 | tail -2
