# A/B of the k_gemm item order on the config-2 bench: "DYN:EG" pairs
# (NEGF_GEMM_DYN, NEGF_GEMM_EG; EG 0 = compiled-in default).
mkdir -p gpurun_out/ab
for v in ${VARIANTS:-1:0 0:0 0:256}; do
  dyn=${v%%:*}; eg=${v##*:}
  if [ "$eg" = 0 ]; then unset NEGF_GEMM_EG; else export NEGF_GEMM_EG=$eg; fi
  NEGF_GEMM_DYN=$dyn python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-rgf --extra-configs "" \
      > gpurun_out/ab/v_${dyn}_${eg}.json 2> gpurun_out/ab/v_${dyn}_${eg}.err
  python -c "
import json; d = json.loads(open('gpurun_out/ab/v_${dyn}_${eg}.json').read().strip().splitlines()[-1])
bl = d['roofline'].get('by_level', {})
print('dyn $dyn eg $eg', round(d['value'], 1), round(d['roofline']['achieved'], 2),
      {k.split(':')[1].strip()[:14] if 'gemm' in k else k[:14]: round(v['ms_per_step'], 2) for k, v in bl.items()})"
done
