# A/B of the k_gemm item order: all energies in one group (default) vs wave-sized groups (NEGF_GEMM_EG=-1) vs fixed groups
B="python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-rgf --extra-configs="
P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), round(d["ms_per_step"],2), {k:round(v["ms_per_step"],2) for k,v in d["roofline"]["kernels"].items()})'
for eg in default -1 4 16; do
  if [ "$eg" = default ]; then unset NEGF_GEMM_EG; else export NEGF_GEMM_EG=$eg; fi
  echo "eg $eg"; $B 2>/dev/null | python -c "$P"
done
