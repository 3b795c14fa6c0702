timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; rc=$?; echo "pytest rc=$rc"; tail -15 gpurun_out/gputest.log | grep -E "passed|failed|Error|assert"
for d in 0 1; do echo "debug=$d"; VABFT_BSIDE_DEBUG=$d timeout 300 python tools/bside_probe.py 4096 4096 2>&1 | cut -c1-100; done
python tools/wide_probe.py 4096 1
python tools/wide_probe.py 4096 3
