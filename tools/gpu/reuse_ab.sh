# cross-level reuse A/B: EBEM_REUSE=0 (none) / 1 (bitwise-safe copies) /
# 2 (default: also the other-orientation sibling entries) at several N
# (circle), then timing at 2N = 2^19
set -x
for n in 1024 4096 16384 65536; do
  EBEM_REUSE=0 python tools/bitcmp.py $n gpurun_out/r0_$n.npy
  EBEM_REUSE=1 python tools/bitcmp.py $n gpurun_out/r1_$n.npy
  EBEM_REUSE=2 python tools/bitcmp.py $n gpurun_out/r2_$n.npy
  python tools/bitcmp.py --cmp gpurun_out/r0_$n.npy gpurun_out/r1_$n.npy
  python tools/bitcmp.py --cmp gpurun_out/r0_$n.npy gpurun_out/r2_$n.npy
done
EBEM_REUSE=0 python tools/repeat_probe.py 262144 3 --prof
EBEM_REUSE=1 python tools/repeat_probe.py 262144 3 --prof
EBEM_REUSE=2 python tools/repeat_probe.py 262144 3 --prof
rm -f gpurun_out/r?_*.npy
