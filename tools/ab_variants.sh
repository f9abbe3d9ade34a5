# A/B of variant builds (tools/variant.sh -> build/variants/*.so, loaded through NEGF_LIB)
B="python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-rgf --extra-configs="
P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), round(d["ms_per_step"],2), {k:round(v["ms_per_step"],2) for k,v in d["roofline"]["kernels"].items() if k in ("gemm","inverse")}, {k.split(":")[1][:22]:round(v["ms_per_step"],2) for k,v in d["roofline"]["by_level"].items() if k.startswith("gemm")})'
echo default; $B 2>/dev/null | python -c "$P"
for v in "$@"; do echo $v; NEGF_LIB=build/variants/$v.so $B 2>/dev/null | python -c "$P"; done
