# real window inverse kernel shapes on real blocks (tools/inv_bench)
cd tools
for m in 52 56 60 64; do INV_REAL=1 ./inv_bench $m 326 256 0; done
for s in sw:64x2x32x3 sw:64x2x32x2 sw:64x4x16x3 sw:64x4x16x4 sw:64x4x16x2 sw:64x1x48x3; do echo -n "$s real: "; SW_REAL=1 INV_REAL=1 RG_SHAPE=$s ./inv_bench 64 326 256 0; done
for s in sw:48x2x24x4 sw:48x2x24x5 sw:48x4x12x4 sw:48x4x12x5; do echo -n "$s real: "; SW_REAL=1 INV_REAL=1 RG_SHAPE=$s ./inv_bench 48 200 256 0; done
for s in sw:32x1x32x10 sw:32x2x16x10 sw:32x2x16x8 sw:32x4x8x12; do echo -n "$s real: "; SW_REAL=1 INV_REAL=1 RG_SHAPE=$s ./inv_bench 32 200 256 0; done
