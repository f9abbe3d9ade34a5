# Shifting-window inverse kernel variants against the dispatched kernels (tools/inv_bench).
cd tools
run() { m=$1; shift; ./inv_bench $m 200 256 0; for s in "$@"; do echo -n "  $s: "; RG_SHAPE=$s ./inv_bench $m 200 256 0; done; }
run 27 sw:32x2x14x8 swl:32x2x14x10 swl:32x1x28x10
run 32 sw:32x1x32x10 swl:32x1x32x10 swl:32x2x16x10
run 35 sw:48x2x20x4 swl:48x2x18x4
run 40 sw:48x2x20x4 swl:48x2x20x4
run 48 sw:48x2x24x4 swl:48x2x24x4
run 52 sw:64x2x28x2 swl:64x2x26x3
run 56 sw:64x2x28x2 swl:64x2x28x3
run 60 sw:64x2x32x3 swl:64x2x30x3
run 64 sw:64x2x32x3 swl:64x2x32x3 swl:64x2x32x2
run 100 sw:104x4x25x1 swl:104x4x25x1
