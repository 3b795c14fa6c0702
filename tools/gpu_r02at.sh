# B-side timeline (globaltimer stamps)
for d in 0 1 3; do echo "debug=$d"; VABFT_BSIDE_DEBUG=$d VABFT_BSIDE_TRACE=1 timeout 300 python tools/bside_once.py 2>&1 | tail -2; done
VABFT_BSIDE_TRACE=1 timeout 300 python tools/bside_once.py float32 2>&1 | tail -2
VABFT_BSIDE_TRACE=1 timeout 300 python tools/bside_once.py bfloat16 11008 4096 2>&1 | tail -2
