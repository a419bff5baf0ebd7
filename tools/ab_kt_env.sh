# A/B of library variants x env by in-pipeline kernel times (prefetch 0) and bench:
#   bash tools/ab_kt_env.sh <pattern> "lib:ENV=..." ...   (lib = librcgs_<lib>.so)
L=paper_2511_18441_b200/_lib
PAT=$1; shift
for spec in "$@"; do
  v=${spec%%:*}; e=${spec#*:}
  cp $L/librcgs_$v.so $L/librcgs.so
  env $e python tools/kernel_times.py --config c3 --steps 20 --prefetch 0 > gpurun_out/kt_$v.txt 2>&1
  b=$(env $e python bench.py --steps 100 --warmup 5 --no-extras --no-cpu-baseline --no-clocks 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['e2e']['value'])")
  echo "== $spec  bench: $b"; grep -E "$PAT" gpurun_out/kt_$v.txt
done
