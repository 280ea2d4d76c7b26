python -m pytest tests/test_gpu_solve_kernels.py tests/test_gpu_fds.py tests/test_gpu_sources.py -q -x 2>&1 | tail -2 > gpurun_out/ab4.log
for v in 1 0; do
  echo "== EBEM_GEMM_MMA=$v" >> gpurun_out/ab4.log
  EBEM_GEMM_MMA=$v python tools/kernel_table.py 262144 2 >> gpurun_out/ab4.log 2>&1
done
EBEM_GEMM_MMA=1 python tools/kernel_table.py 65536 2 180 >> gpurun_out/ab4.log 2>&1
ncu --metrics gpu__time_duration.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,smsp__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed_pipe_fp64.sum --clock-control none -k regex:k_gemm --csv python tools/kernel_table.py 262144 1 > gpurun_out/ncu_gemm_metrics.csv 2>&1
