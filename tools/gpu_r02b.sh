O=gpurun_out/r02b; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_boundary.py tests/test_gpu_configs.py -k "not cfg3_generator" -x -q -s > $O/tests.log 2>&1; echo tests rc=$?; tail -30 $O/tests.log
for dbg in 0 1 2 4 5 6 3 7; do KGP_TC_DEBUG=$dbg timeout 120 python tools/tc_probe.py 65536 32 2 fast; done > $O/probe_debug.log 2>&1; cat $O/probe_debug.log
for fl in 8 16 32; do KGP_TC_FLUSH=$fl timeout 120 python tools/tc_probe.py 65536 32 2 fast; done > $O/probe_flush.log 2>&1; cat $O/probe_flush.log
for ms in 1 2 4; do KGP_TC_MAXSPLIT=$ms timeout 120 python tools/tc_probe.py 65536 32 2 fast; done > $O/probe_split.log 2>&1; cat $O/probe_split.log
timeout 120 python tools/tc_probe.py 65536 32 1 fast >> $O/probe_misc.log 2>&1
timeout 120 python tools/tc_probe.py 65536 32 2 tf32 >> $O/probe_misc.log 2>&1
timeout 120 python tools/tc_probe.py 65536 32 1 tf32 >> $O/probe_misc.log 2>&1
timeout 120 python tools/tc_probe.py 65536 16 2 fast >> $O/probe_misc.log 2>&1
timeout 120 python tools/tc_probe.py 65536 64 2 fast >> $O/probe_misc.log 2>&1
cat $O/probe_misc.log
