# Team-layout QR/CPQR build variants (development aid; GPU box).
cd paper_2411_18026_b200/csrc
for v in "$@"; do
  touch ebem_qr.cu; make -j8 EXTRA="$v" > /dev/null 2>&1 || { echo "build failed $v"; continue; }
  echo "== $v"
  (cd ../.. && timeout 120 python tools/prof_breakdown.py 2>&1 | tail -1)
done
touch ebem_qr.cu; make -j8 > /dev/null 2>&1
