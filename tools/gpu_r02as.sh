# chain fetch via cp.async: chains alone and the full pass; B-side parity tests
for d in 0 3; do echo "debug=$d"; VABFT_BSIDE_DEBUG=$d timeout 300 python tools/bside_probe.py 2>&1 | tail -4; done
timeout 900 python -m pytest tests/ -m gpu -x -q -k "bside or parity or summary" 2>&1 | tail -3
