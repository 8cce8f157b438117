set -x
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,temperature.gpu --format=csv > gpurun_out/smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --skip-nlml > gpurun_out/ncu_ll.log 2>&1; echo ll rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kmm_tc_kernel -s 3 -c 1 -f -o gpurun_out/prof_r01_cfg2_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --skip-nlml > gpurun_out/ncu_full.log 2>&1; echo full rc=$?
