# round 2 (second session): full GPU tests, bench, smoke; then ncu launch list + full capture of the headline kernel
O=gpurun_out/${R02:-r02d}; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo tests rc=$?; tail -2 $O/gpu_tests.log
timeout 900 python bench.py > $O/bench.log 2>&1; echo bench rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?; tail -1 $O/smoke.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --skip-nlml --skip-secondary > $O/ncu_ll.log 2>&1; echo ll rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kmm_tc_kernel -s 3 -c 1 -f -o $O/prof_cfg2_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --skip-nlml --skip-secondary > $O/ncu_full.log 2>&1; echo full rc=$?
