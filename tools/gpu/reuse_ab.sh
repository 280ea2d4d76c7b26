# cross-level reuse A/B: bitwise-equal solutions with EBEM_REUSE=0/1 at
# several N (circle) + the star config, then timing at 2N = 2^19
set -x
for n in 1024 4096 16384 65536; do
  EBEM_REUSE=0 python tools/bitcmp.py $n gpurun_out/r0_$n.npy
  EBEM_REUSE=1 python tools/bitcmp.py $n gpurun_out/r1_$n.npy
  python tools/bitcmp.py --cmp gpurun_out/r0_$n.npy gpurun_out/r1_$n.npy
done
EBEM_REUSE=0 python tools/repeat_probe.py 262144 3 --prof
EBEM_REUSE=1 python tools/repeat_probe.py 262144 3 --prof
rm -f gpurun_out/r0_*.npy gpurun_out/r1_*.npy
