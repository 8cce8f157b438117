O=gpurun_out/r02f; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo tests rc=$?; tail -2 $O/gpu_tests.log
timeout 900 python bench.py > $O/bench.log 2>&1; echo bench rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?; tail -1 $O/smoke.log
timeout 300 python tools/nlml_time.py fp64 otf 20 > $O/nlml_time.log 2>&1; cat $O/nlml_time.log | tail -1
timeout 600 ncu --nvtx --nvtx-include "eval/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_nlml_cfg1_otf.csv python tools/nlml_once.py fp64 otf > $O/ncu_nlml.log 2>&1; echo nlml ll rc=$?
