# Shifting-window inverse kernel variants against the dispatched kernels (tools/inv_bench).
cd tools
run() { m=$1; nb=$2; shift; shift; NEGF_INV_FORCE_LEGACY=1 ./inv_bench $m $nb 256 0; for s in "$@"; do echo -n "  $s: "; RG_SHAPE=$s ./inv_bench $m $nb 256 0; done; }
run 6 500 sw:32x1x8x16 sw:32x1x12x16
run 11 500 sw:32x1x12x16 sw:32x1x16x16 sw:32x1x16x12
run 14 500 sw:32x1x16x16 sw:32x1x16x12
