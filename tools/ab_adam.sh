# A/B of library variants on the isolated (ncu, serialised) fused Adam with the
# next view's colour epilogue, plus the pipelined bench: bash tools/ab_adam.sh v1 v2 ...
# (v = default | name of paper_2511_18441_b200/_lib/ab/librcgs_<name>.so)
mkdir -p gpurun_out/ab
for v in "$@"; do
  if [ "$v" = default ]; then L=""; else L="paper_2511_18441_b200/_lib/ab/librcgs_$v.so"; fi
  RCGS_LIB_PATH=$L ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -k regex:"adam_fused|color_kernel" --csv \
      --log-file gpurun_out/ab/adam_$v.csv python tools/step_probe.py --config c3 --steps 3 --warmup 12 --prefetch 2 > /dev/null 2>&1
  for i in 1 2; do RCGS_LIB_PATH=$L python bench.py --no-extras --no-cpu-baseline --no-clocks 2>/dev/null | tail -1 | \
      python3 -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$v', d['value'], d['stages_ms'])"; done
  python3 - gpurun_out/ab/adam_$v.csv <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
t = [float(r[h.index('Metric Value')].replace(',', '')) for r in rows[1:]]
print(sys.argv[1], 'adam us', [round(x / 1e3, 1) for x in t])
PY
done
