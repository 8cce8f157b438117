for p in bf16x3 fast; do for dbg in 0 16 32 48 1 17 49; do KGP_TC_DEBUG=$dbg timeout 100 python tools/tc_probe.py 65536 32 2 $p; done; done
