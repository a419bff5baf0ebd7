# GPU check: parity tests, then N bench runs of the C3 step (prints step ms, stage ms, Mpix/s, warp iterations)
N=${1:-2}
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log
for i in $(seq $N); do timeout 600 python bench.py --config c3 --steps 100 --warmup 5 --no-cpu-baseline --no-extras --no-clocks > gpurun_out/x.log 2>gpurun_out/x.err; echo "$(tail -1 gpurun_out/x.log | python3 -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d[\"ms_per_step\"], d[\"stages_ms\"], d[\"rendered_mpix_s\"], d[\"raster_work_per_launch\"][\"fwd\"][\"warp_iterations\"])")"; done
