# TSQR reflector ring depth A/B (EBEM_TSQR_SLOTS caps the slots: 128 = before)
set -x
for d in 128 256 512; do
  EBEM_TSQR_SLOTS=$d python tools/repeat_probe.py 262144 3 --prof 2>&1 | tail -2
done
python -m pytest tests/test_gpu_tsqr.py tests/test_gpu_basis.py -x -q 2>&1 | tail -2
