# Launch-bounds experiments for the fill kernels (development aid; GPU box).
set -e
cd paper_2411_18026_b200/csrc
for v in "-DEBEM_PROXY_MINB=1" "-DEBEM_PROXY_MINB=1 -DEBEM_PROXY_PAIRS_CAP=64" "-DEBEM_PROXY_MINB=2 -DEBEM_PROXY_PAIRS_CAP=64" ""; do
  touch ebem_fill.cu; make -j8 EXTRA="$v" > /dev/null 2>&1
  echo "== $v"
  (cd ../.. && python tools/repeat_probe.py 262144 2 --prof 2>&1 | tail -1)
done
