# A/B of environment settings on the C3 bench step: bash tools/ab_env.sh "VAR=a VAR2=b" "VAR=c" ...
for cfg in "$@"; do
  for rep in 1 2; do
    env $cfg python bench.py --steps 100 --warmup 5 --no-extras --no-cpu-baseline --no-clocks > gpurun_out/abe.json 2> gpurun_out/abe.err
    echo "[$cfg] $(tail -1 gpurun_out/abe.json | python3 -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['ms_per_step'], d['step_ms_p10_p50_p90_max'], d['e2e']['value'])")"
  done
done
