# B-side timeline: unrolled chain batches; 1 vs 2 CTAs per SM
for p in 2 1; do echo "per_sm=$p"; VABFT_BSIDE_PERSM=$p VABFT_BSIDE_TRACE=1 timeout 300 python tools/bside_once.py 2>&1 | tail -2;
VABFT_BSIDE_DEBUG=3 VABFT_BSIDE_PERSM=$p VABFT_BSIDE_TRACE=1 timeout 300 python tools/bside_once.py 2>&1 | tail -2;
VABFT_BSIDE_PERSM=$p timeout 300 python tools/bside_probe.py 2>&1 | head -1; done
