# blocked single-RHS CTA LU solve: parity, bitwise A/B of the solution, timing
set -x
python -m pytest tests/test_gpu_solve_kernels.py -x -q 2>&1 | tail -2
for n in 16384 65536; do
  EBEM_GETRS_CTA_BLK=0 python tools/bitcmp.py $n gpurun_out/g0_$n.npy
  EBEM_GETRS_CTA_BLK=1 python tools/bitcmp.py $n gpurun_out/g1_$n.npy
  python tools/bitcmp.py --cmp gpurun_out/g0_$n.npy gpurun_out/g1_$n.npy
done
rm -f gpurun_out/g?_*.npy
EBEM_GETRS_CTA_BLK=0 python tools/solve_profile.py 262144 1 | tail -1
EBEM_GETRS_CTA_BLK=1 python tools/solve_profile.py 262144 1 | tail -1
EBEM_GETRS_CTA_BLK=1 python tools/solve_profile.py 262144 4 | tail -1
