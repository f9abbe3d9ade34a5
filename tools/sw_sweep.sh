cd tools
for s in sw:64x1x64x5 sw:64x1x64x6 sw:64x1x64x7; do echo -n "$s real: "; SW_REAL=1 INV_REAL=1 RG_SHAPE=$s ./inv_bench 64 326 256 0; done
for s in sw:64x2x30x3 sw:64x1x60x5 sw:64x1x60x6; do echo -n "$s real: "; SW_REAL=1 INV_REAL=1 RG_SHAPE=$s ./inv_bench 60 326 256 0; done
for s in sw:64x2x26x3 sw:64x1x52x5 sw:64x1x52x6; do echo -n "$s real: "; SW_REAL=1 INV_REAL=1 RG_SHAPE=$s ./inv_bench 52 326 256 0; done
for s in sw:48x2x24x4 sw:64x1x48x6; do echo -n "$s real: "; SW_REAL=1 INV_REAL=1 RG_SHAPE=$s ./inv_bench 48 200 256 0; done
for s in sw:48x2x20x4 sw:64x1x40x6 sw:64x1x40x8; do echo -n "$s real: "; SW_REAL=1 INV_REAL=1 RG_SHAPE=$s ./inv_bench 40 200 256 0; done
for s in sw:48x2x20x4 sw:64x1x40x6 sw:64x1x40x8; do echo -n "$s real: "; SW_REAL=1 INV_REAL=1 RG_SHAPE=$s ./inv_bench 34 200 256 0; done
