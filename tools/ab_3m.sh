B="python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-rgf --extra-configs="
P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), round(d["ms_per_step"],2), {k:round(v["ms_per_step"],2) for k,v in d["roofline"]["kernels"].items()})'
echo default; $B 2>/dev/null | python -c "$P"
echo 3m-fold+G; NEGF_GEMM_3M_PHASES=3 $B 2>/dev/null | python -c "$P"
echo 3m-fold; NEGF_GEMM_3M_PHASES=1 $B 2>/dev/null | python -c "$P"
python tools/resid_margin.py --ref 2>&1 | tail -4
NEGF_GEMM_3M_PHASES=3 python tools/resid_margin.py --ref 2>&1 | tail -4
NEGF_GEMM_3M_PHASES=1 python tools/resid_margin.py --ref 2>&1 | tail -4
