# A/B of library variants by in-pipeline kernel times: bash tools/ab_kt.sh <pattern> v1 v2 ...
# (each vN is paper_2511_18441_b200/_lib/librcgs_vN.so, copied over librcgs.so in turn)
L=paper_2511_18441_b200/_lib
PAT=$1; shift
for v in "$@"; do cp $L/librcgs_$v.so $L/librcgs.so; python tools/kernel_times.py --config c3 --steps 20 --prefetch 0 > gpurun_out/kt_$v.txt 2>&1; echo "== $v"; grep -E "$PAT|total" gpurun_out/kt_$v.txt; done
