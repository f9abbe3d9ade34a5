# Batched inverse kernels on config-2 leaf sizes (tools/inv_bench): the
# dispatched kernel per size class, plus the register shapes for comparison.
cd tools
for m in 28 32; do ./inv_bench $m 200 256 0; RG_SHAPE=32x2 ./inv_bench $m 200 256 0; done
for m in 40 48; do ./inv_bench $m 200 256 0; done
for m in 50 56 64; do ./inv_bench $m 326 256 0; RG_SHAPE=64x4 ./inv_bench $m 326 256 0; done
