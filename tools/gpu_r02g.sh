./tools/micro/fp64_tput
for d in 0 2; do echo "debug=$d"; VABFT_BSIDE_DEBUG=$d timeout 300 python tools/bside_probe.py 4096 4096 2>&1 | cut -c1-110; done
timeout 900 python -m pytest tests/test_gpu_configs.py -x -q 2>&1 | tail -3
