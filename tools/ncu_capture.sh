# ncu evidence for one config-2 batch (256 energies): launch list + --set full
# captures of the kernels DESIGN.md §3 lists.  Run on the GPU box after the
# bench itself has exited 0 without ncu.  Outputs under gpurun_out/ncu/.
set -x
mkdir -p gpurun_out/ncu
B="python tools/launch_map.py batch 1"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu/launches.csv $B > gpurun_out/ncu/launches.log 2>&1
F="ncu --set full --clock-control none --import-source on"
$F -k regex:k_gemm --launch-skip 26 -c 1 -o gpurun_out/ncu/gemm_lv9_fold $B > /dev/null 2>&1
$F -k regex:k_gemm --launch-skip 101 -c 1 -o gpurun_out/ncu/gemm_lv2_grows $B > /dev/null 2>&1
$F -k regex:k_gemm --launch-skip 103 -c 1 -o gpurun_out/ncu/gemm_lv1_compact $B > /dev/null 2>&1
$F -k regex:k_inverse_blocked -c 1 -o gpurun_out/ncu/inverse_blocked $B > /dev/null 2>&1
$F -k regex:k_inverse_rg -c 2 -o gpurun_out/ncu/inverse_rg $B > /dev/null 2>&1
$F -k regex:k_inverse_la -c 1 -o gpurun_out/ncu/inverse_la $B > /dev/null 2>&1
$F -k regex:k_bigpanel -c 1 -o gpurun_out/ncu/bigpanel $B > /dev/null 2>&1
$F -k regex:k_sschur -c 1 -o gpurun_out/ncu/sschur $B > /dev/null 2>&1
$F -k regex:k_spsi -c 1 -o gpurun_out/ncu/spsi $B > /dev/null 2>&1
$F -k regex:k_mgather -c 1 -o gpurun_out/ncu/mgather $B > /dev/null 2>&1
ls -la gpurun_out/ncu
