# bench value / ms / e2e per config (no CPU baseline); extra env via arguments: VAR=val ...
for c in ${CONFIGS:-c3 c4 c5}; do
  echo -n "$c $* : "
  env "$@" python bench.py --config $c --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('%.4g'%d['value'], '%.2f ms'%d['ms_per_step'], 'e2e %.4g'%d['e2e']['value'], 'cons', d.get('conservation_ok'))"
done
