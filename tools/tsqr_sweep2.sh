# TSQR piece-count sweep (development aid; GPU box): waves of row pieces per
# round for a build with the given flags.
cd paper_2411_18026_b200/csrc
touch ebem_tsqr.cu; make -j8 EXTRA="$1" > /dev/null 2>&1 || { echo "build failed $1"; exit 1; }
cd ../..
for w in 1 2 4 8; do
  echo "== $1 waves $w"
  EBEM_TSQR_WAVES=$w timeout 300 python tools/repeat_probe.py 262144 2 --prof 2>&1 | tail -1
done
