timeout 300 python tools/wide_probe.py 2>&1 | tail -12
timeout 1200 python -m pytest tests/ -m gpu -x -q -k "wide or fp32 or fp64 or config or tf32" > gpurun_out/t.log 2>&1; echo "rc=$?"; tail -3 gpurun_out/t.log
timeout 600 python tools/formats_only.py 2>&1 | tail -5
