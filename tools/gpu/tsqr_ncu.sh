# wavefront TSQR (medium variant): wall + gaps, then one full ncu capture
# of a mid-level launch with source-level stall samples
set -x
EBEM_VERBOSE=1 python tools/repeat_probe.py 262144 3 --prof 2>&1 | grep -v "^\[ebem\]   " | tail -4
python tools/repeat_probe.py 262144 3 | tail -1
ncu --set full --import-source on --clock-control none -k regex:k_tsqr -s 4 -c 1 -o gpurun_out/tsqr_panel python tools/repeat_probe.py 262144 1 > /dev/null 2>&1
ls -la gpurun_out/tsqr_panel.ncu-rep
