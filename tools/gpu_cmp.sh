O=gpurun_out/cmp; mkdir -p $O
for v in head base; do
  if [ $v = base ]; then L=""; else L=tools/variants/$v/libkgp.so; fi
  echo "== $v"
  KGP_LIB=$L timeout 300 python tools/op_matrix.py 65536 fast > $O/opm_$v.txt 2>&1
  for p in fast bf16x3 tf32; do KGP_LIB=$L timeout 120 python tools/tc_probe.py 65536 32 2 $p gaussian 8 30 2>&1 | tail -1; done
done
paste $O/opm_head.txt $O/opm_base.txt | awk -F'\t' '{split($1,a," ms"); split($2,b," ms"); n=split(a[1],x," "); m=split(b[1],y," "); printf "%-40s head %8s new %8s\n", substr($1,1,30), x[n], y[m]}'
