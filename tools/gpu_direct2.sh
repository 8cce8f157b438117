O=gpurun_out/direct2; mkdir -p $O
KD=gaussian:3,gaussian:4,matern32:2,matern32:4,matern52:2,matern52:4
timeout 300 python tools/op_matrix.py 65536 fast $KD > $O/base.txt 2>&1
KGP_LIB=tools/variants/leanx_rtdx0/libkgp.so timeout 300 python tools/op_matrix.py 65536 fast $KD > $O/lr.txt 2>&1
paste $O/base.txt $O/lr.txt | awk -F'\t' '{split($1,a," ms"); split($2,b," ms"); n=split(a[1],x," "); m=split(b[1],y," "); printf "%-32s base %8s lr %8s\n", substr($1,1,30), x[n], y[m]}'
