O=gpurun_out/lrx; mkdir -p $O
timeout 300 python tools/op_matrix.py 65536 fast gaussian:8,gaussian:3,matern32:2,matern32:4,matern52:2,matern52:4 > $O/opm.txt 2>&1; cat $O/opm.txt | awk '{print $1,$2,$3,$4,$5,$6}'
timeout 60 python tools/tc_probe.py 65536 17 1 fast gaussian 3 30 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo tests rc=$?; tail -2 $O/gpu_tests.log
