#!/bin/bash
# round-2 evidence: launch lists + one full capture of the headline kernel (each command ran
# without ncu first: the bench in tools/gpu_r02_full.sh, nlml_once below)
O=gpurun_out/r02prof; mkdir -p $O
timeout 300 python tools/nlml_once.py fp64 otf > $O/nlml_once.log 2>&1; echo nlml_once rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --skip-nlml --skip-secondary > $O/ncu_ll.log 2>&1; echo ll rc=$?
timeout 600 ncu --nvtx --nvtx-include "eval/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_nlml_cfg1_otf.csv python tools/nlml_once.py fp64 otf > $O/ncu_nlml.log 2>&1; echo nlml rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kmm_tc_kernel -s 3 -c 1 -f -o $O/prof_cfg2_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --skip-nlml --skip-secondary > $O/ncu_full.log 2>&1; echo full rc=$?
