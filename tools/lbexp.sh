set -e
cd paper_2411_18026_b200/csrc
for v in "2 1" "3 2" "4 3"; do
  set -- $v
  touch ebem_fill.cu; make -j8 EXTRA="-DEBEM_NEAR_MINB=$1 -DEBEM_PROXY_MINB=$2" > /dev/null 2>&1
  echo "== near minb $1 proxy minb $2"
  (cd ../.. && python tools/scale_probe.py 65536 2>&1 | grep -E "N=|near_sep|proxy")
done
