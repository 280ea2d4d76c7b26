python -m pytest tests/test_gpu_solve_kernels.py tests/test_gpu_fds.py tests/test_gpu_configs.py tests/test_gpu_sources.py -q -x 2>&1 | tail -3 > gpurun_out/ab3.log
for v in 1 0; do
  echo "== EBEM_GEMM_MMA=$v" >> gpurun_out/ab3.log
  EBEM_GEMM_MMA=$v python tools/repeat_probe.py 262144 2 --prof >> gpurun_out/ab3.log 2>&1
done
ncu --query-metrics 2>/dev/null | grep -i "dmma\|fp64\|tensor_op" > gpurun_out/metrics_fp64.txt
ncu --set full --import-source on --clock-control none -k regex:k_gemm_mma -s 6 -c 1 -o gpurun_out/gemm_mma python tools/repeat_probe.py 262144 1 > gpurun_out/ncu_gemm.log 2>&1
