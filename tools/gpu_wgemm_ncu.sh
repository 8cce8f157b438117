O=gpurun_out/wg; mkdir -p $O
KGP_AFN_WGEMM=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"wy_kernel|wtu_kernel" -s 4 -c 2 -f -o $O/wg_full python tools/precond_apply_bench.py 65536 1024 33 > $O/ncu_full.log 2>&1; echo full rc=$?
