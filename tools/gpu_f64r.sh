timeout 120 python tools/nlml_time.py fp64 otf 20 2>&1 | tail -1
timeout 60 python tools/f64_one.py 4096 17 1 gaussian 3 2>&1 | tail -1
timeout 60 python tools/f64_one.py 4096 1 1 gaussian 3 2>&1 | tail -1
timeout 60 python tools/f64_one.py 16384 33 1 matern32 4 2>&1 | tail -1
timeout 90 python tools/f64_one.py 65536 32 2 gaussian 8 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "fp64 or f64 or golden or cfg or nlml or symmetric or dense or pcg or host" 2>&1 | tail -2
