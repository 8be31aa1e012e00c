# dev: hook time vs buffer placement (FSV_EPAD: ecol start offset in entries,
# FSV_HPAD: hub accumulator offset in ints)
L=${1:-paper_1910_05971_b200/libfastsv.so}
for e in ${EPADS:-0 262144}; do
for h in ${HPADS:-0 32 256 1024 4096 16384 65536}; do
  echo "epad $e hpad $h: $(FSV_EPAD=$e FSV_HPAD=$h python tools/layout_check.py $L 2 | sed 's/labels.*//')"
done; done
