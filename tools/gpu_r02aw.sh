# B-side TMA-ring kernel: trace, probe, parity tests
for f in bfloat16 float32; do VABFT_BSIDE_TRACE=1 timeout 120 python tools/bside_once.py $f 2>&1 | tail -2; done
VABFT_BSIDE_DEBUG=1 VABFT_BSIDE_TRACE=1 timeout 120 python tools/bside_once.py 2>&1 | tail -2
VABFT_BSIDE_TRACE=1 timeout 120 python tools/bside_once.py bfloat16 11008 4096 2>&1 | tail -2
timeout 300 python tools/bside_probe.py 2>&1 | tail -4
timeout 1200 python -m pytest tests/ -m gpu -x -q -k "bside or wide or fp32 or tf32 or config or parity" 2>&1 | tail -3
