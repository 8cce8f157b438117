O=gpurun_out/wg; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_afn.py -q -x -p no:cacheprovider > $O/tests.log 2>&1; echo tests rc=$?; tail -1 $O/tests.log
for n in 65536 262144; do for e in 0 1; do KGP_AFN_WGEMM=$e timeout 300 python tools/nlml_cfg3_once.py $n 2>&1 | tail -1 | cut -c1-60 | sed "s/^/n=$n wg=$e /"; done; done
