O=gpurun_out/f64split; mkdir -p $O
run() {
  timeout 120 python tools/f64_grid.py 16384 matern32 4 1 33,34,36 2>&1 | tail -1
  timeout 120 python tools/f64_grid.py 16384 gaussian 8 1 33,36 2>&1 | tail -1
  timeout 120 python tools/f64_grid.py 16384 gaussian 3 1 33,36 2>&1 | tail -1
  timeout 120 python tools/f64_grid.py 16384 matern52 2 1 33 2>&1 | tail -1
  timeout 120 python tools/f64_grid.py 65536 matern32 4 1 33 2>&1 | tail -1
}
( echo "== one-lane (KGP_F64_SPLIT_MIN1=99)"; KGP_F64_SPLIT_MIN1=99 run; echo "== 2 x 18"; run ) 2>&1 | tee $O/k33.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "lane_split or fp64" 2>&1 | tail -2
