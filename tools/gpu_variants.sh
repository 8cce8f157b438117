for v in st8 st4 st8sc; do L=tools/variants/$v/libkgp.so; for i in 1 2; do echo -n "$v "; KGP_LIB=$L timeout 100 python tools/tc_probe.py 65536 32 2 fast; done; done
for v in st8 st4; do echo -n "$v "; KGP_LIB=tools/variants/$v/libkgp.so timeout 100 python tools/tc_probe.py 65536 33 1 fast matern32 4; done
timeout 100 python tools/tc_probe.py 65536 33 1 fast matern32 4
