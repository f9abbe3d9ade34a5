# Window inverse kernels (tools/inv_bench): the dispatched kernel per size on complex
# and on real blocks (INV_REAL=1: real data, real kernel; INV_REAL_COMPLEX_KERNEL=1: the
# complex kernel on the same real data), plus forced shapes (RG_SHAPE=sw:ROWSxHxSxMINB,
# SW_REAL=1 for the double instantiation).  Results: profiles/inverse_experiments_r02.txt
cd tools
for m in 27 32 40 48 52 56 60 64 74 100; do
  nb=200; [ $m -ge 49 ] && [ $m -le 64 ] && nb=326
  ./inv_bench $m $nb 256 0
  INV_REAL=1 INV_REAL_COMPLEX_KERNEL=1 ./inv_bench $m $nb 256 0
  INV_REAL=1 ./inv_bench $m $nb 256 0
done
