O=gpurun_out/r02full; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x -s > $O/gpu_tests.log 2>&1; echo tests rc=$?; grep -E "passed|failed|fast:|fp64:|cfg3-generator|w-solve" $O/gpu_tests.log | tail -20
timeout 600 python bench.py > $O/bench.log 2>&1; echo bench rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?; tail -1 $O/smoke.log
