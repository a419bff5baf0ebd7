# Round profile set (run on the GPU box from the repo root):
#  1. bench.py once without ncu (must exit 0)
#  2. ncu launch list (gpu__time_duration, clocks uncontrolled) of the same bench command
#  3. ncu --set full of every kernel of one steady-state optimizer step (tools/step_probe.py)
# Summaries land in gpurun_out/prof/ (copy to profiles/).
set -e
B="python bench.py --steps 5 --warmup 3 --no-extras --no-cpu-baseline --no-clocks"
$B > gpurun_out/prof_bench.json 2> gpurun_out/prof_bench.err
# the timed steps only (bench.py brackets them with cudaProfilerStart/Stop)
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
python tools/step_probe.py --config c3 --steps 1 --warmup 12 > gpurun_out/sp.log 2>&1
ncu --set full --import-source on --clock-control none --profile-from-start off -o gpurun_out/step_full -f \
    python tools/step_probe.py --config c3 --steps 1 --warmup 12 > gpurun_out/ncu_full.log 2>&1
# summaries on the box (the full capture is too large to bring back), plus a
# smaller full capture of the two rasteriser kernels to keep
python tools/profile_summarize.py ${TAG:-r01} gpurun_out/prof > gpurun_out/prof_summary.log 2>&1
rm -f gpurun_out/step_full.ncu-rep
ncu --set full --import-source on --clock-control none --profile-from-start off --kernel-name-base demangled \
    -k "regex:raster_kernel" -c 2 -o gpurun_out/prof/${TAG:-r01}_raster -f \
    python tools/step_probe.py --config c3 --steps 1 --warmup 12 > gpurun_out/ncu_raster.log 2>&1
echo profile-done
