for v in default one1 one2 one3; do L=paper_2503_02259_b200/libkgp.so; [ $v != default ] && L=tools/variants/$v/libkgp.so; for i in 1 2; do echo -n "$v "; KGP_LIB=$L timeout 100 python tools/tc_probe.py 65536 32 2 fast; done; done
for v in one1 one2; do KGP_LIB=tools/variants/$v/libkgp.so timeout 100 python tools/op_err2.py 65536 32 fast; done
