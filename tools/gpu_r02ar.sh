# B-side pass ablations: full, no chains (1), chains alone (3)
for d in 0 1 3; do echo "debug=$d"; VABFT_BSIDE_DEBUG=$d timeout 300 python tools/bside_probe.py 2>&1 | tail -4; done
VABFT_BSIDE_DEBUG=3 timeout 300 python tools/bside_probe.py 11008 4096 2>&1 | head -1
