#!/bin/bash
# round-end evidence: launch lists of the bench command and of one cfg1 NLML evaluation
set -x
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --skip-nlml > gpurun_out/ncu_ll.log 2>&1; echo ll rc=$?
timeout 600 ncu --nvtx --nvtx-include "eval/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/nlml_launches.csv python tools/nlml_once.py > gpurun_out/ncu_nlml.log 2>&1; echo nlml rc=$?
