# Round 2, fourth session: ncu captures of the fp64 operator kernels (after the same commands ran clean
# in tools/gpu_f64grid.sh / tools/gpu_r02_full.sh). CSV exports only (the .ncu-rep files stay on the box).
O=gpurun_out/r02d_prof; mkdir -p $O; T=/tmp/r02d; mkdir -p $T
cap() {  # name regex args...
  name=$1; rx=$2; shift 2
  ncu --set full --clock-control none --import-source on -k regex:$rx -s 2 -c 1 -o $T/$name -f python tools/f64_one.py "$@" > $O/$name.log 2>&1
  ncu -i $T/$name.ncu-rep --page raw --csv > $O/$name.raw.csv 2>/dev/null
  ncu -i $T/$name.ncu-rep --page details --csv > $O/$name.details.csv 2>/dev/null
}
cap f64_split_cfg2 kmm_f64_split_kernel 65536 32 2 gaussian 8
cap f64_cfg1_k17 'kmm_f64_kernel' 4096 17 1 gaussian 3
cap f64_cfg1_k1 kmm_f64_sym_kernel 4096 1 1 gaussian 3
cap f64_cfg3_k33 'kmm_f64_kernel' 16384 33 1 matern32 4
ls -la $O
