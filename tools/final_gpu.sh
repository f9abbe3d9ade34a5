# Round-end evidence on one B200: GPU tests, both bench arms, ncu captures, k_gemm DRAM traffic.
mkdir -p gpurun_out/final
python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/final/gputest.log
python bench.py --impl reference > gpurun_out/final/bench_ref.json 2> gpurun_out/final/bench_ref.err
python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err
python tools/real_check.py > gpurun_out/final/real_check.txt 2>&1
python tools/resid_margin.py --ref > gpurun_out/final/resid_margin.txt 2>&1
bash tools/ncu_capture.sh > gpurun_out/final/ncu_capture.log 2>&1
EGS="default" bash tools/gemm_traffic.sh > gpurun_out/final/gemm_traffic.log 2>&1
cat gpurun_out/final/gputest.log; tail -1 gpurun_out/final/bench.err; cat gpurun_out/final/real_check.txt; tail -3 gpurun_out/final/resid_margin.txt; cat gpurun_out/traffic/traffic_default.txt | head -6
