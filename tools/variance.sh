# run-to-run variance of the selection pass and the step (env A/B): bash tools/variance.sh "ENV=.." ...
for cfg in "$@"; do
  echo "== $cfg"
  for i in 1 2 3 4; do
    env $cfg python bench.py --steps 60 --warmup 5 --no-extras --no-cpu-baseline --no-clocks 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.readline()); print('  sel', d['selection']['ms'], 'value', d['value'], 'p50/max', d['step_ms_p10_p50_p90_max'][1], d['step_ms_p10_p50_p90_max'][3], 'e2e', d['e2e']['value'])"
  done
done
