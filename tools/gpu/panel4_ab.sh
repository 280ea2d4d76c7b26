# wavefront TSQR: 4-reflector panel consumption, with the ring depth caps
set -x
python -m pytest tests/test_gpu_tsqr.py tests/test_gpu_basis.py -x -q 2>&1 | tail -2
for d in 128 512; do
  EBEM_TSQR_SLOTS=$d python tools/repeat_probe.py 262144 3 --prof 2>&1 | tail -2
done
python -m pytest tests/test_gpu_configs.py tests/test_gpu_fds.py -x -q 2>&1 | tail -2
