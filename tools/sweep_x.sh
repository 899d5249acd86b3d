# k_paths_x configuration sweep on the C2 shape (2e8 paths): bench value per setting
run() { echo -n "$* : "; env "$@" python bench.py --paths 2e8 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('%.4g'%d['value'], '%.2f ms'%d['ms_per_step'], d['conservation_ok'])"; }
for v in "$@"; do run $v; done
