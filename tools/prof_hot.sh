# Focused ncu captures of the hot kernels (run on the GPU box from the repo root):
# loss passes (standalone 1080p pair), the fused Adam with and without the next
# view's colour epilogue, and the recording raster, each with source.
set -e
mkdir -p gpurun_out/hot
python tools/loss_bench.py > gpurun_out/hot/loss_bench.json 2>&1
ncu --set full --import-source on --clock-control none -k regex:loss_ -s 15 -c 3 -o gpurun_out/hot/loss -f \
    python tools/loss_bench.py > gpurun_out/hot/ncu_loss.log 2>&1
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"adam_fused|raster_kernel" -c 2 \
    -o gpurun_out/hot/step_pf2 -f python tools/step_probe.py --config c3 --steps 1 --warmup 12 --prefetch 2 > gpurun_out/hot/ncu_pf2.log 2>&1
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"adam_fused|color_kernel" -c 2 \
    -o gpurun_out/hot/step_pf0 -f python tools/step_probe.py --config c3 --steps 1 --warmup 12 --prefetch 0 > gpurun_out/hot/ncu_pf0.log 2>&1
echo hot-done
