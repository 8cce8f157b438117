O=gpurun_out/r02h; mkdir -p $O
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $O/smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?; tail -1 $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo tests rc=$?; tail -2 $O/gpu_tests.log
timeout 900 python bench.py > $O/bench.log 2>&1; echo bench rc=$?; tail -c 3000 $O/bench.log
