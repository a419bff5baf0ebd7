# Isolated (ncu, serialised) durations of the fused Adam with (prefetch 2) and
# without (prefetch 0) the next view's colour epilogue, and the build kernels.
set -e
mkdir -p gpurun_out/adam
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/adam/pf2.csv python tools/step_probe.py --config c3 --steps 3 --warmup 12 --prefetch 2 > gpurun_out/adam/pf2.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/adam/pf0.csv python tools/step_probe.py --config c3 --steps 3 --warmup 12 --prefetch 0 > gpurun_out/adam/pf0.log 2>&1
echo adam-done
