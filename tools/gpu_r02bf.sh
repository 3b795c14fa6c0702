# warp-parallel exact sequential sums in the B-side summary: parity + timeline
timeout 900 python -m pytest tests/ -m gpu -x -q -k "bside or parity or summary or config or calib" 2>&1 | tail -2
for f in bfloat16 float32; do VABFT_BSIDE_TRACE=1 timeout 120 python tools/bside_once.py $f 2>&1 | grep trace | tail -1; done
VABFT_BSIDE_DEBUG=3 VABFT_BSIDE_TRACE=1 timeout 120 python tools/bside_once.py 2>&1 | grep trace | tail -1
VABFT_BSIDE_TRACE=1 timeout 120 python tools/bside_once.py bfloat16 11008 4096 2>&1 | grep trace | tail -1
timeout 300 python tools/bside_probe.py 2>&1 | tail -4
