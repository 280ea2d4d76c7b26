# Fill-kernel variant timing (development aid; GPU box): build with each
# EXTRA flag set and print the factorization's top kernels.
cd paper_2411_18026_b200/csrc
for v in "$@"; do
  touch ebem_fill.cu; make -j8 EXTRA="$v" > /dev/null 2>&1 || { echo "build failed $v"; continue; }
  echo "== $v"
  (cd ../.. && timeout 120 python tools/repeat_probe.py 262144 2 --prof 2>&1 | tail -1)
done
touch ebem_fill.cu; make -j8 > /dev/null 2>&1
