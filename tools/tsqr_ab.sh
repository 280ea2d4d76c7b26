# single-pipeline TSQR timing for build variants (development aid; GPU box)
cd paper_2411_18026_b200/csrc
for v in "$@"; do
  touch ebem_tsqr.cu; make -j8 EXTRA="$v" > /dev/null 2>&1 || { echo "build failed $v"; continue; }
  echo "== $v"
  (cd ../.. && EBEM_TSQR_PIECES=1 timeout 120 python tools/tsqr_bench.py 2>&1 | tail -5)
done
touch ebem_tsqr.cu; make -j8 > /dev/null 2>&1
