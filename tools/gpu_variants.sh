for v in default roles; do L=paper_2503_02259_b200/libkgp.so; [ $v != default ] && L=tools/variants/$v/libkgp.so; for a in "65536 32 2 fast" "65536 32 2 fast" "65536 33 1 fast matern32 4" "65536 32 2 bf16x3"; do echo -n "$v "; KGP_LIB=$L timeout 100 python tools/tc_probe.py $a; done; done
KGP_LIB=tools/variants/roles/libkgp.so timeout 100 python tools/op_err2.py 65536 32 fast
