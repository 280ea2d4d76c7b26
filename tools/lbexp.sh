# TSQR variant experiments (development aid; GPU box).  Each entry: EXTRA flags.
set -e
cd paper_2411_18026_b200/csrc
for v in "-DEBEM_TSQR_S_LANES=4 -DEBEM_TSQR_S_THREADS=256 -DEBEM_TSQR_M_LANES=4 -DEBEM_TSQR_M_THREADS=512" \
         "-DEBEM_TSQR_S_LANES=16 -DEBEM_TSQR_S_THREADS=1024 -DEBEM_TSQR_M_LANES=8 -DEBEM_TSQR_M_THREADS=1024"; do
  touch ebem_tsqr.cu; make -j8 EXTRA="$v" > /dev/null 2>&1
  echo "== $v"
  (cd ../.. && python tools/repeat_probe.py 262144 2 --prof 2>&1 | tail -1)
done
