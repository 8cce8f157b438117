O=gpurun_out/w2; mkdir -p $O
for w in 1 0 1; do
  echo "== W2=$w"
  for r in 1 2; do KGP_TC_W2=$w timeout 120 python tools/tc_probe.py 65536 32 2 fast gaussian 8 30 2>&1 | tail -1; done
  KGP_TC_W2=$w timeout 120 python tools/tc_probe.py 65536 16 2 fast gaussian 8 30 2>&1 | tail -1
  KGP_TC_W2=$w timeout 120 python tools/tc_probe.py 65536 32 2 tf32 gaussian 8 30 2>&1 | tail -1
  KGP_TC_W2=$w timeout 120 python tools/tc_probe.py 65536 16 2 fast matern32 4 30 2>&1 | tail -1
  KGP_TC_W2=$w timeout 120 python tools/variant_err.py 16384 32 2>&1 | tail -1
  KGP_TC_W2=$w timeout 120 python tools/variant_err.py 65536 32 2>&1 | tail -1
done
KGP_TC_W2FLUSH=16 timeout 120 python tools/tc_probe.py 65536 32 2 fast gaussian 8 30 2>&1 | tail -1
KGP_TC_W2FLUSH=16 timeout 120 python tools/variant_err.py 65536 32 2>&1 | tail -1
timeout 300 python tools/op_matrix.py 65536 fast > $O/opm.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guard.py tests/test_gpu_configs.py -q -x -p no:cacheprovider 2>&1 | tail -3
