# dev: solve time vs vertex-array (X, G) and hub-accumulator placement
#   usage: CFG=2 VPADS="0 1024" HPADS="0 12288" bash tools/vpadsweep.sh [lib]
L=${1:-paper_1910_05971_b200/libfastsv.so}
for v in ${VPADS:-0}; do
for h in ${HPADS:-0}; do
  echo "cfg ${CFG:-2} vpad $v hpad $h: $(FSV_VPAD=$v FSV_HPAD=$h python tools/layout_check.py $L ${CFG:-2} | sed 's/labels.*//')"
done; done
