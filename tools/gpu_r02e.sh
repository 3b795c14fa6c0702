for d in 0 1 2; do echo "debug=$d"; VABFT_BSIDE_DEBUG=$d timeout 300 python tools/bside_probe.py 4096 4096 2>&1 | cut -c1-120; done
timeout 600 python -m pytest tests/test_gpu_wide.py tests/test_gpu_configs.py -x -q 2>&1 | tail -3
timeout 300 python tools/formats_only.py > gpurun_out/formats.log 2>&1; tail -20 gpurun_out/formats.log
