# quick env A/B of the C3 step: each line "<env assignments>" -> value, ms/step, stage ms
for cfg in "$@"; do
  for i in 1 2; do
    env $cfg timeout 600 python bench.py --steps 60 --warmup 5 --no-cpu-baseline --no-extras --no-clocks > gpurun_out/x.log 2>gpurun_out/x.err
    echo "[$cfg] $(tail -1 gpurun_out/x.log | python3 -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['ms_per_step'], d['stages_ms'])" 2>&1 | tail -1)"
  done
done
