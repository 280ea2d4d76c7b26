set -e
cd paper_2411_18026_b200/csrc
for v in "0 0" "1 0" "0 1" "1 1"; do
  set -- $v
  touch ebem_fill.cu; make -j8 EXTRA="-DEBEM_SERIES_PARAM=$1 -DEBEM_HANKEL_PAIR=$2" > /dev/null 2>&1
  echo "== series_param $1 hankel_pair $2"
  (cd ../.. && python tools/scale_probe.py 65536 2>&1 | grep -E "N=|near_sep|proxy")
done
