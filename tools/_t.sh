timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_fast_path.py tests/test_config_parity.py tests/test_scan_path.py -q -x -p no:cacheprovider 2>&1 | tail -2
b() { echo -n "$* : "; env $1 timeout 600 python bench.py --config $2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('%.4g'%d['value'], d['ms_per_step'], d.get('price',{}).get('rel_err_vs_reference'))"; }
for i in 1 2; do b QT_X_HIST1=1 c1; b QT_X_HIST1=0 c1; b QT_X_HIST1=1 c2; b QT_X_HIST1=0 c2; done
