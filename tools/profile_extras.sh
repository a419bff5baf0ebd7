# ncu --set full of the 8(f) row kernels (stereo matcher, PLY decode/encode) on
# one C3 view; the program is run once without ncu first.  Run on the GPU box
# from the repo root; the summary lands in gpurun_out/prof/.
set -e
mkdir -p gpurun_out/prof
python tools/extras_probe.py > gpurun_out/extras_probe.log 2>&1
ncu --set full --import-source on --clock-control none --profile-from-start off --kernel-name-base demangled \
    -k "regex:stereo_|ply_" -o gpurun_out/extras_full -f python tools/extras_probe.py > gpurun_out/ncu_extras.log 2>&1
ncu -i gpurun_out/extras_full.ncu-rep --page raw --csv > gpurun_out/extras_raw.csv
python tools/profile_extras_summary.py gpurun_out/extras_raw.csv ${TAG:-r01} > gpurun_out/prof/${TAG:-r01}_ncu_extras.md
rm -f gpurun_out/extras_full.ncu-rep
echo extras-done
