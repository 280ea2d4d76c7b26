python -m pytest tests/test_gpu_fds.py tests/test_gpu_solve_kernels.py tests/test_gpu_conv.py "tests/test_gpu_configs.py::test_config3_multi_rhs_vs_reference" -q -x 2>&1 | tail -2 > gpurun_out/solve_ab.log
for cfg in "new 1 1 4096" "nomin 1 1 0" "oldtrsv 1 0 4096" "old 0 0 4096"; do
  set -- $cfg
  echo "== $1" >> gpurun_out/solve_ab.log
  EBEM_GEMV_WARP=$2 EBEM_TRSV_BLK=$3 EBEM_GEMV_WARP_MIN=$4 python tools/solve_profile.py 262144 1 >> gpurun_out/solve_ab.log 2>&1
done
ncu --profile-from-start off --metrics gpu__time_duration.sum,launch__grid_size,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python tools/solve_profile.py 262144 1 > gpurun_out/solve_ncu3.csv 2>&1
