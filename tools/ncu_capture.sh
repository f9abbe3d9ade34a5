# ncu evidence for one config-2 batch (256 energies): launch list + --set full
# captures of the kernels DESIGN.md §3 lists, summarised on the box
# (tools/ncu_summary.py; raw CSV pages kept, large reports dropped so the
# merge-back stays small).  Run after the bench itself exited 0 without ncu.
set -x
mkdir -p gpurun_out/ncu
B="python tools/launch_map.py batch 1"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu/launches.csv $B > gpurun_out/ncu/launches.log 2>&1
python tools/launch_map.py ops gpurun_out/ncu/ops.json
python tools/launch_map.py map gpurun_out/ncu/launches.csv gpurun_out/ncu/ops.json > gpurun_out/ncu/launch_map.txt 2>&1
F="ncu -f --set full --clock-control none --import-source on"
# k_gemm launch index of (phase, level, arrangement) in plan order
gidx() { python -c "
import json; g=[o for o in json.load(open('gpurun_out/ncu/ops.json')) if o['kind']==1]
print([i for i,o in enumerate(g) if (o['phase'],o['level'],o['arr'])==($1,$2,$3)][0])"; }
cap() {  # name, ncu filter args...
  local name=$1; shift
  rm -f /tmp/ncu_$name.ncu-rep
  $F "$@" -o /tmp/ncu_$name $B > /dev/null 2>&1
  ncu -i /tmp/ncu_$name.ncu-rep --page raw --csv > gpurun_out/ncu/$name.raw.csv 2>/dev/null
  python tools/ncu_summary.py /tmp/ncu_$name.ncu-rep > gpurun_out/ncu/$name.summary.txt 2>&1
}
cap gemm_lv9_fold -k regex:k_gemm --launch-skip $(gidx 0 9 0) -c 1
cap gemm_lv2_grows_warp -k regex:k_gemm --launch-skip $(gidx 1 2 3) -c 1
cap gemm_lv5_grows -k regex:k_gemm --launch-skip $(gidx 1 5 0) -c 1
cap gemm_lv1_compact -k regex:k_gemm --launch-skip $(gidx 1 1 0) -c 1
cap inverse_sw -k regex:k_inverse_sw -c 12
cap inverse_la -k regex:k_inverse_la -c 1
cap bigpanel -k regex:k_bigpanel -c 1
cap sschur -k regex:k_sschur -c 1
cap spsi -k regex:k_spsi -c 1
cap mgather -k regex:k_mgather -c 1
# launch list of the bench command itself (kernel shares of the step)
ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/ncu/bench_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-rgf --extra-configs= > gpurun_out/ncu/bench_under_ncu.log 2>&1
python tools/launch_map.py shares gpurun_out/ncu/bench_launches.csv > gpurun_out/ncu/bench_launch_shares.txt 2>&1
du -sh gpurun_out/ncu; ls -la gpurun_out/ncu
