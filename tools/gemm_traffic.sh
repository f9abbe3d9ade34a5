# k_gemm DRAM traffic of one config-2 batch against the algorithmic bytes, per
# item-order energy group (NEGF_GEMM_EG; default = the compiled-in groups).
mkdir -p gpurun_out/traffic
python tools/launch_map.py ops gpurun_out/traffic/ops.json
for eg in ${EGS:-default 256}; do
  if [ "$eg" = default ]; then unset NEGF_GEMM_EG; else export NEGF_GEMM_EG=$eg; fi
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:k_gemm \
      --clock-control none --csv --log-file gpurun_out/traffic/dram_$eg.csv python tools/launch_map.py batch \
      > gpurun_out/traffic/ncu_$eg.log 2>&1
  python tools/launch_map.py traffic gpurun_out/traffic/dram_$eg.csv gpurun_out/traffic/ops.json \
      > gpurun_out/traffic/traffic_$eg.txt 2>&1
  echo "== eg $eg"; cat gpurun_out/traffic/traffic_$eg.txt
done
