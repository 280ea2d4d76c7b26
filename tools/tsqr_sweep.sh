# TSQR layout sweep (development aid; GPU box): ring depth, rows per lane,
# lanes per column, CTA size and register budget of the small (n <= 64) variant.
cd paper_2411_18026_b200/csrc
for v in "$@"; do
  touch ebem_tsqr.cu; make -j8 EXTRA="$v" > /dev/null 2>&1 || { echo "build failed $v"; continue; }
  echo "== $v"
  (cd ../.. && timeout 300 python tools/repeat_probe.py 262144 2 --prof 2>&1 | tail -1)
done
touch ebem_tsqr.cu; make -j8 > /dev/null 2>&1
