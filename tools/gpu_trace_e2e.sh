for q in 45 50 55; do echo "q$q waves"; KGP_HOST_RRATIO=$q KGP_HOST_TRACE=1 timeout 60 python tools/e2e_trace.py 2>&1 | tail -1; done
echo "q50 nowaves"; KGP_HOST_WAVES=0 KGP_HOST_TRACE=1 timeout 60 python tools/e2e_trace.py 2>&1 | tail -1
for c in 2 4; do echo "rows$c"; KGP_HOST_CHUNKS=$c KGP_HOST_TRACE=1 timeout 60 python tools/e2e_trace.py 2>&1 | tail -1; done
run() { timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --skip-nlml --skip-secondary 2>/dev/null \
    | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', 'e2e ms', round(d['e2e']['ms_per_step'], 3), 'step ms', round(d['ms_per_step'], 3))"; }
run default; KGP_HOST_CHUNKS=4 run rows4; KGP_HOST_RRATIO=45 run q45
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "host" 2>&1 | tail -2
