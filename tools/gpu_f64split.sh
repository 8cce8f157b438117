# Variants first: tools/build_variant.sh notab "-DKGP_F64_TABEXP=0" (the exponential before exp_neg64t)
# A/B of the fp64 operator: table exp (exp_neg64t) and the lane-split wide-k kernels
O=gpurun_out/f64split; mkdir -p $O
run() {
  echo "== $1"
  timeout 60 python tools/f64_one.py 4096 17 1 gaussian 3 2>&1 | tail -1
  timeout 60 python tools/f64_one.py 4096 1 1 gaussian 3 2>&1 | tail -1
  timeout 60 python tools/f64_one.py 4096 17 2 gaussian 3 2>&1 | tail -1
  timeout 90 python tools/f64_one.py 65536 32 2 gaussian 8 2>&1 | tail -1
  timeout 90 python tools/f64_one.py 32768 32 1 gaussian 8 2>&1 | tail -1
  timeout 60 python tools/f64_one.py 16384 33 1 matern32 4 2>&1 | tail -1
  timeout 60 python tools/f64_one.py 16384 33 2 matern32 4 2>&1 | tail -1
  timeout 60 python tools/f64_one.py 16384 51 2 gaussian 8 2>&1 | tail -1
  timeout 60 python tools/f64_one.py 16384 64 1 matern52 2 2>&1 | tail -1
  timeout 60 python tools/nlml_time.py fp64 otf 20 2>&1 | tail -1
}
(
KGP_LIB=tools/variants/notab/libkgp.so KGP_F64_SPLIT=0 run "old: no table, no split"
KGP_F64_SPLIT=0 run "table, no split"
run "table + split"
) 2>&1 | tee $O/ab.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "fp64 or f64 or cfg1 or symmetric or golden or lane_split or determ" 2>&1 | tail -3 | tee $O/tests.log
