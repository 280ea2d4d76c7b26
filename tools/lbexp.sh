set -e
cd paper_2411_18026_b200/csrc
for v in 256 512 1024; do
  touch ebem_dense.cu; make -j8 EXTRA="-DEBEM_QR_THREADS=$v" > /dev/null 2>&1
  echo "== qr threads $v"
  (cd ../.. && python tools/scale_probe.py 262144 2>&1 | grep -E "N=|qr_reduce|cpqr|getrf")
done
