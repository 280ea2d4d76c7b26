python -m pytest tests/test_gpu_tsqr.py tests/test_gpu_basis.py -q -x 2>&1 | tail -n 3
for v in 0 1; do echo "== WY=$v"; EBEM_TSQR_WY=$v python tools/kernel_table.py 262144 2 2>&1 | grep -E "factorize|k_qr|k_cpqr"; done
python -m pytest tests/test_gpu_configs.py tests/test_gpu_fds.py -q -x 2>&1 | tail -n 3; cat gpurun_out/solution_*.json
