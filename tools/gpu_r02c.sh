# re-entry check of HEAD on a fresh box: gpu tests, bench, smoke, reference arm
O=gpurun_out/r02c; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x -s -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo tests rc=$?; grep -E "passed|failed|error" $O/gpu_tests.log | tail -5
timeout 900 python bench.py > $O/bench.log 2>&1; echo bench rc=$?; tail -c 600 $O/bench.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?; tail -1 $O/smoke.log
timeout 600 python bench.py --impl reference > $O/ref.log 2>&1; echo ref rc=$?; tail -c 300 $O/ref.log
