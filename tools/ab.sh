# A/B timing of the working tree against a reference tree in ab_old/ (dev aid)
for r in 1 2; do
  echo "== new"; python tools/repeat_probe.py 262144 3 2>&1 | tail -1
  echo "== old"; (cd ab_old && python tools/repeat_probe.py 262144 3 2>&1 | tail -1)
done
