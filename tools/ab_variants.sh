# A/B of in-tree library builds: for each RCGS_LIB_PATH given (default: the
# main build), N bench runs of the C3 step (step ms, stage ms, fwd warp iterations)
N=${N:-2}
for lib in "$@"; do
  for i in $(seq $N); do
    RCGS_LIB_PATH=$lib timeout 600 python bench.py --config c3 --steps 100 --warmup 5 --no-cpu-baseline --no-extras --no-clocks > gpurun_out/x.log 2>gpurun_out/x.err
    echo "$lib $(tail -1 gpurun_out/x.log | python3 -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['ms_per_step'], d['stages_ms'], d['raster_work_per_launch']['fwd'])" 2>&1 | tail -1)"
  done
done
