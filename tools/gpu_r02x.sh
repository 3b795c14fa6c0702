timeout 900 python -m pytest tests/test_gpu_wide.py tests/test_gpu_configs.py -x -q > gpurun_out/t.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/t.log
python tools/wide_probe.py 4096 1
python tools/wide_probe.py 4096 3
python tools/wide_probe.py 2048 1 fp64
