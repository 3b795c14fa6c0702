# B-side 16-bit: per-row atomic accumulators, ordered p1/p2 only in the combine
timeout 900 python -m pytest tests/ -m gpu -x -q -k "bside or parity or summary or config or calib or blockwise" 2>&1 | tail -2
for d in 0 1 2; do VABFT_BSIDE_DEBUG=$d VABFT_BSIDE_TRACE=1 timeout 120 python tools/bside_once.py 2>&1 | grep trace | tail -1; done
timeout 300 python tools/bside_probe.py 2>&1 | tail -4
VABFT_BSIDE_DEBUG=1 timeout 120 python tools/bside_probe.py 2>&1 | head -1
