# Variant first: tools/build_variant.sh fmadist "-DKGP_F64_FMADIST=1"
O=gpurun_out/f64split; mkdir -p $O
run() {
  timeout 120 python tools/f64_grid.py 65536 gaussian 8 2 32 2>&1 | tail -1
  timeout 120 python tools/f64_grid.py 16384 gaussian 8 1 16,17,32,33,51,64 2>&1 | tail -1
  timeout 120 python tools/f64_grid.py 16384 matern32 4 1 17,33 2>&1 | tail -1
  timeout 120 python tools/f64_grid.py 4096 gaussian 3 1 1,17 2>&1 | tail -1
  timeout 60 python tools/nlml_time.py fp64 otf 20 2>&1 | tail -1
}
( echo "== base"; run; echo "== fmadist"; KGP_LIB=tools/variants/fmadist/libkgp.so run ) 2>&1 | tee $O/fmadist.log
