for v in default bfns2; do L=paper_2503_02259_b200/libkgp.so; [ $v != default ] && L=tools/variants/$v/libkgp.so; for fl in 8 16; do for p in fast bf16x3; do echo -n "$v "; KGP_TC_FLUSH=$fl KGP_LIB=$L timeout 100 python tools/tc_probe.py 65536 32 2 $p; done; done; done
KGP_TC_FLUSH=16 timeout 100 python tools/op_err2.py 65536 32 fast bf16x3
