python -m pytest tests/test_gpu_tsqr.py tests/test_gpu_basis.py -q -x > gpurun_out/panel_tests.log 2>&1; tail -n 15 gpurun_out/panel_tests.log
for v in 0 1; do echo "== EBEM_TSQR_PANEL=$v"; EBEM_TSQR_PANEL=$v python tools/kernel_table.py 262144 2 2>&1 | grep -E "factorize|k_qr|k_cpqr"; done
python -m pytest tests/test_gpu_configs.py -q -x > gpurun_out/panel_cfg.log 2>&1; tail -n 5 gpurun_out/panel_cfg.log; cat gpurun_out/solution_*.json
