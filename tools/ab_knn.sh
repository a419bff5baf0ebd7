L=paper_2511_18441_b200/_lib
cp $L/librcgs.so /tmp/librcgs_keep.so
for v in "$@"; do cp $L/librcgs_$v.so $L/librcgs.so; echo "== $v"; timeout 120 python tools/knn_probe.py --points 1400000; done
cp /tmp/librcgs_keep.so $L/librcgs.so
