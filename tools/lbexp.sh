# TSQR register-budget experiments (development aid; GPU box).
set -e
cd paper_2411_18026_b200/csrc
for v in "-DEBEM_TSQR_REGS=96" "-DEBEM_TSQR_REGS=128" "-DEBEM_TSQR_REGS=64"; do
  touch ebem_tsqr.cu; make -j8 EXTRA="$v" > /dev/null 2>&1
  echo "== $v"
  (cd ../.. && python tools/repeat_probe.py 262144 2 --prof 2>&1 | tail -1)
done
