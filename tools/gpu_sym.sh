# Variants first: tools/build_variant.sh <name> "-DKGP_F64_SYM_Q=<chunk> -DKGP_F64_SYM_MINB=<CTAs per SM>" (sym8: 8/16, s4_16: 4/16, s8_20: 8/20, s8_24: 8/24, s4_24: 4/24)
O=gpurun_out/f64split; mkdir -p $O
run() {
  timeout 120 python tools/f64_grid.py 4096 gaussian 3 1 1,2,4 2>&1 | tail -1
  timeout 120 python tools/f64_grid.py 16384 matern32 4 1 1,4 2>&1 | tail -1
  timeout 60 python tools/nlml_time.py fp64 otf 20 2>&1 | tail -1
}
( echo "== base"; run; for v in sym8 s4_16 s8_20 s8_24 s4_24; do echo "== $v"; KGP_LIB=tools/variants/$v/libkgp.so run; done ) 2>&1 | tee $O/sym.log
