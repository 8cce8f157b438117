O=gpurun_out/wg; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_afn.py -q -x -p no:cacheprovider -k wide > $O/tests.log 2>&1; echo tests rc=$?; tail -1 $O/tests.log
KGP_AFN_WGEMM=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"wy_k|wtu_k|d884" --log-file $O/q1.csv python tools/precond_apply_bench.py 65536 1024 33 > /dev/null 2>&1; echo q1 rc=$?
python tools/launch_summary.py $O/q1.csv 8
if [ "$FULL" = 1 ]; then KGP_AFN_WGEMM=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"wy_kernel|wtu_kernel" -s 4 -c 2 -f -o $O/wg_full python tools/precond_apply_bench.py 65536 1024 33 > $O/ncu_full.log 2>&1; echo full rc=$?; fi
