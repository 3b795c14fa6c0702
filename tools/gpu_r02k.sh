for d in 3 4 5 6 7; do echo "debug=$d"; VABFT_BSIDE_DEBUG=$d timeout 300 python tools/bside_probe.py 4096 4096 2>&1 | head -1 | cut -c1-110; done
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_calibration.py -x -q > gpurun_out/t.log 2>&1; echo "rc=$?"; grep -E "passed|failed|Error|assert" gpurun_out/t.log | head -20
