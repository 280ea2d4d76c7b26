set -e
cd paper_2411_18026_b200/csrc
for v in 2 3; do
  touch ebem_fill.cu; make -j8 EXTRA="-DEBEM_SYM_MINB=$v" > /dev/null 2>&1
  echo "== sym minb $v"
  (cd ../.. && python tools/scale_probe.py 262144 2>&1 | grep -E "N=|near_sym")
done
