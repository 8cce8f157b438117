for k in 12 17 24 32 40; do
  for e in 0 1; do KGP_AFN_WGEMM=$e timeout 300 python tools/precond_apply_bench.py 65536 1024 $k 2>&1 | grep afn | sed "s/^/wg=$e /"; done
done
