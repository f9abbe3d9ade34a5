B="python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-rgf --extra-configs="
P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), round(d["ms_per_step"],2), {k:round(v["ms_per_step"],2) for k,v in d["roofline"]["kernels"].items()}, {k.split(":")[1][:18]:round(v["ms_per_step"],2) for k,v in d["roofline"]["by_level"].items()})'
echo default; $B 2>/dev/null | python -c "$P"
echo adaptive; NEGF_GEMM_EG=-1 $B 2>/dev/null | python -c "$P"
echo default; $B 2>/dev/null | python -c "$P"
echo adaptive; NEGF_GEMM_EG=-1 $B 2>/dev/null | python -c "$P"
EGS="default -1" bash tools/gemm_traffic.sh 2>&1 | grep -A6 "^== eg"
