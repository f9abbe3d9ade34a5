# A/B of the warp-tile bounds (plan-time env switches)
B="python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-rgf --extra-configs="
P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), round(d["ms_per_step"],2), {k:round(v["ms_per_step"],2) for k,v in d["roofline"]["kernels"].items() if k in ("gemm","inverse")}, {k.split(":")[1][:22]:round(v["ms_per_step"],2) for k,v in d["roofline"]["by_level"].items() if k.startswith("gemm")})'
for wm in 16 32 48; do for wk in 128 256 1024; do
  echo "warp_m $wm warp_k $wk"; NEGF_WARP_TILE_M=$wm NEGF_WARP_TILE_K=$wk $B 2>/dev/null | python -c "$P"
done; done
