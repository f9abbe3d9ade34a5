cd tools
for m in 64 60 56 52; do
  INV_REAL=1 ./inv_bench $m 326 256 0
  for s in sw2r:64x2x$((m/2))x3 ; do echo -n "  $s: "; INV_REAL=1 RG_SHAPE=$s ./inv_bench $m 326 256 0; done
done
echo -n "  sw2r:64x2x32x2: "; INV_REAL=1 RG_SHAPE=sw2r:64x2x32x2 ./inv_bench 64 326 256 0
echo -n "  sw2r:64x4x16x2: "; INV_REAL=1 RG_SHAPE=sw2r:64x4x16x2 ./inv_bench 64 326 256 0
echo -n "  odd nE sw2r:64x2x32x3: "; INV_REAL=1 RG_SHAPE=sw2r:64x2x32x3 ./inv_bench 64 326 255 0
INV_REAL=1 ./inv_bench 48 200 256 0
for s in sw2r:48x2x24x4 sw2r:48x2x24x5; do echo -n "  $s: "; INV_REAL=1 RG_SHAPE=$s ./inv_bench 48 200 256 0; done
INV_REAL=1 ./inv_bench 40 200 256 0
echo -n "  sw2r:48x2x20x5: "; INV_REAL=1 RG_SHAPE=sw2r:48x2x20x5 ./inv_bench 40 200 256 0
INV_REAL=1 ./inv_bench 32 200 256 0
for s in sw2r:32x1x32x8 sw2r:32x1x32x10 sw2r:32x2x16x12; do echo -n "  $s: "; INV_REAL=1 RG_SHAPE=$s ./inv_bench 32 200 256 0; done
