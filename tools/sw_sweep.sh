# real vs complex window inverse kernels on real blocks (tools/inv_bench)
cd tools
for m in 27 32 40 48 56 64; do INV_REAL=1 INV_REAL_COMPLEX_KERNEL=1 ./inv_bench $m 200 256 0; INV_REAL=1 ./inv_bench $m 200 256 0; done
