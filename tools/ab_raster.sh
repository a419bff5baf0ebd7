# A/B of library variants on the recording raster (kernel_times, prefetch 0) and
# the pipelined bench: bash tools/ab_raster.sh v1 v2 ... (v = default | ab/librcgs_<v>.so)
for v in "$@"; do
  if [ "$v" = default ]; then L=""; else L="paper_2511_18441_b200/_lib/ab/librcgs_$v.so"; fi
  RCGS_LIB_PATH=$L python tools/kernel_times.py --config c3 --steps 20 --prefetch 0 2>/dev/null | grep -E "raster_kernel|rec_bwd|total" | sed "s/^/$v /"
  for i in 1 2; do RCGS_LIB_PATH=$L python bench.py --no-extras --no-cpu-baseline --no-clocks 2>/dev/null | tail -1 | \
      python3 -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$v', d['value'], d['stages_ms'])"; done
done
