for cfg in "def 1 " "old 0 " "oldnocs 0 abx/nocs.so" "ptsnocs 1 abx/nocs.so"; do
  set -- $cfg
  echo "== $1" >> gpurun_out/ab2.log
  EBEM_FILL_PTS=$2 EBEM_GPU_LIB=$3 python tools/repeat_probe.py 262144 2 --prof >> gpurun_out/ab2.log 2>&1
done
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_configs.py -q -x 2>&1 | tail -3 >> gpurun_out/ab2.log
