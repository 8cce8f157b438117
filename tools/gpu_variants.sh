for a in "4096 17 2 fp64 gaussian 3 20" "16384 33 1 fp64 matern32 4 10" "16384 33 2 fp64 matern52 2 10" "65536 32 2 fp64 gaussian 8 5"; do timeout 100 python tools/tc_probe.py $a; done
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
