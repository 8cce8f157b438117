O=gpurun_out/${RUN_TAG:-r02full3}; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -s > $O/gpu_tests.log 2>&1; echo tests rc=$?; grep -E "passed|failed|cfg3-generator|w-solve|local-variance" $O/gpu_tests.log | tail -8
timeout 900 python bench.py > $O/bench.log 2>&1; echo bench rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?; tail -1 $O/smoke.log
timeout 600 python bench.py --impl reference > $O/ref.log 2>&1; echo ref rc=$?; tail -c 300 $O/ref.log
