set -x
mkdir -p gpurun_out/r02a
O=gpurun_out/r02a
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $O/smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; tail -3 $O/gpu_tests.log
timeout 300 python tools/sanitize.py > $O/san_plain.log 2>&1; echo plain rc=$?; tail -2 $O/san_plain.log
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $CS --tool memcheck --leak-check no --print-limit 50 python tools/sanitize.py > $O/san_memcheck.log 2>&1; echo memcheck rc=$?; tail -4 $O/san_memcheck.log
timeout 900 $CS --tool synccheck --print-limit 50 python tools/sanitize.py > $O/san_synccheck.log 2>&1; echo synccheck rc=$?; tail -4 $O/san_synccheck.log
timeout 1200 $CS --tool racecheck --racecheck-report hazard --print-limit 50 python tools/sanitize.py nlml64 dense afn gpc local > $O/san_racecheck.log 2>&1; echo racecheck rc=$?; tail -4 $O/san_racecheck.log
timeout 900 $CS --tool racecheck --racecheck-report hazard --print-limit 50 python tools/sanitize.py fast peer > $O/san_racecheck_tc.log 2>&1; echo racecheck_tc rc=$?; tail -4 $O/san_racecheck_tc.log
timeout 900 $CS --tool initcheck --print-limit 50 python tools/sanitize.py nlml64 dense afn > $O/san_initcheck.log 2>&1; echo initcheck rc=$?; tail -4 $O/san_initcheck.log
timeout 600 python bench.py > $O/bench.log 2>&1; echo bench rc=$?; tail -c 3000 $O/bench.log
