O=gpurun_out/wg; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_afn.py -q -x -p no:cacheprovider > $O/tests.log 2>&1; echo tests rc=$?; tail -3 $O/tests.log
for nmk in "65536 1024 33" "262144 1024 33" "131072 512 51" "262144 2048 64"; do
  for e in 0 1; do KGP_AFN_WGEMM=$e timeout 300 python tools/precond_apply_bench.py $nmk 2>&1 | grep afn | sed "s/^/wg=$e /"; done
done | tee $O/apply.log
KGP_AFN_WGEMM=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ll1.csv python tools/precond_apply_bench.py 65536 1024 33 > /dev/null 2>&1; echo ll1 rc=$?
KGP_AFN_WGEMM=0 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ll0.csv python tools/precond_apply_bench.py 65536 1024 33 > /dev/null 2>&1; echo ll0 rc=$?
