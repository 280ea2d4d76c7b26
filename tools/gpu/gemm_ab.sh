python -m pytest tests/test_gpu_solve_kernels.py tests/test_gpu_fds.py -q -x 2>&1 | tail -n 2
for v in 0 1; do echo "== EBEM_GEMM_CELL=$v"; EBEM_GEMM_CELL=$v python tools/kernel_table.py 262144 2 2>&1 | grep -E "factorize|k_gemm"; done
python -m pytest tests/test_gpu_configs.py -q -x 2>&1 | tail -n 2; cat gpurun_out/solution_*.json
ncu --set full --import-source on --clock-control none -k regex:k_gemm_cell -s 0 -c 3 -o gpurun_out/gemm_cell python tools/repeat_probe.py 262144 1 > /dev/null 2>&1
