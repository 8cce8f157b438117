#!/bin/bash
# round-2 final: full verification (tests, bench, smoke, reference arm), then the launch lists of the
# bench command and of one configs[0] OTF eval under ncu (each after it ran clean without ncu)
RUN_TAG=r02final bash tools/gpu_r02_full.sh
O=gpurun_out/r02final; mkdir -p $O
timeout 300 python tools/nlml_once.py fp64 otf > $O/nlml_once.log 2>&1; echo nlml_once rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --skip-nlml --skip-secondary > $O/ncu_ll.log 2>&1; echo ll rc=$?
timeout 600 ncu --nvtx --nvtx-include "eval/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_nlml_cfg1_otf.csv python tools/nlml_once.py fp64 otf > $O/ncu_nlml.log 2>&1; echo nlml rc=$?
