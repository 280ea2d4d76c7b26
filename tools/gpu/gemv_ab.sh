python -m pytest tests/test_gpu_fds.py tests/test_gpu_solve_kernels.py -q -x 2>&1 | tail -2 > gpurun_out/gemv_ab.log
for v in 1 0; do
  echo "== EBEM_GEMV_WARP=$v" >> gpurun_out/gemv_ab.log
  EBEM_GEMV_WARP=$v python tools/solve_profile.py 262144 1 >> gpurun_out/gemv_ab.log 2>&1
  EBEM_GEMV_WARP=$v python tools/solve_profile.py 262144 4 >> gpurun_out/gemv_ab.log 2>&1
done
ncu --profile-from-start off --metrics gpu__time_duration.sum,launch__grid_size,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python tools/solve_profile.py 262144 1 > gpurun_out/solve_ncu2.csv 2>&1
