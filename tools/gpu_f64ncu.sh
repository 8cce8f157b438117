# ncu --set full of a slow / fast neighbour pair of the one-lane fp64 kernel (n = 16384, d = 8, one output,
# k = 16 vs 20), raw metrics exported as CSV on the box (the .ncu-rep files are too large to bring back)
O=gpurun_out/f64split; mkdir -p $O; T=/tmp/f64ncu; mkdir -p $T
for k in 16 20; do
KGP_F64_SPLIT=0 ncu --set full --clock-control none -k regex:kmm_f64_kernel -s 2 -c 1 -o $T/k$k -f python tools/f64_one.py 16384 $k 1 gaussian 8 > $O/ncu_k$k.log 2>&1
ncu -i $T/k$k.ncu-rep --page raw --csv > $O/k$k.raw.csv 2>/dev/null
done
ls -la $O | tail -5
