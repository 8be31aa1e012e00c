# dev: solve/hook time vs buffer placement
#   FSV_EPAD: layout start offset in entries, FSV_HPAD: hub accumulator offset in ints
#   usage: CFG=2 EPADS="0 262144" HPADS="0 4096" bash tools/padsweep.sh [lib]
L=${1:-paper_1910_05971_b200/libfastsv.so}
for e in ${EPADS:-0 262144}; do
for h in ${HPADS:-0}; do
  echo "cfg ${CFG:-2} epad $e hpad $h: $(FSV_EPAD=$e FSV_HPAD=$h python tools/layout_check.py $L ${CFG:-2} | sed 's/labels.*//')"
done; done
