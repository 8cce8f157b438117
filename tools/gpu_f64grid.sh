O=gpurun_out/f64split; mkdir -p $O
grid() {
  for d in 3 8; do for nout in 1 2; do
    timeout 120 python tools/f64_grid.py 16384 gaussian $d $nout 4,8,12,16,17,20,24,28,32,33,40,48,51,64 2>&1 | tail -1
  done; done
  timeout 120 python tools/f64_grid.py 16384 matern32 4 1 16,17,24,28,32,33,48,64 2>&1 | tail -1
  timeout 120 python tools/f64_grid.py 16384 matern32 4 2 16,17,24,28,32,33,48,64 2>&1 | tail -1
  timeout 120 python tools/f64_grid.py 16384 matern52 2 1 16,33,64 2>&1 | tail -1
  timeout 120 python tools/f64_grid.py 4096 gaussian 3 1 1,16,17 2>&1 | tail -1
  timeout 120 python tools/f64_grid.py 4096 gaussian 3 2 17 2>&1 | tail -1
  timeout 120 python tools/f64_grid.py 65536 gaussian 8 2 32 2>&1 | tail -1
  timeout 60 python tools/nlml_time.py fp64 otf 20 2>&1 | tail -1
}
( echo "== ${TAG:-default}"; grid ) 2>&1 | tee $O/grid_${TAG:-default}.log
