timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; rc=$?; echo "pytest rc=$rc"; tail -15 gpurun_out/gputest.log | grep -E "passed|failed|Error|assert"
for d in 0 1 4; do echo "debug=$d"; VABFT_BSIDE_DEBUG=$d timeout 300 python tools/bside_probe.py 4096 4096 2>&1 | cut -c1-110; done
timeout 300 python tools/bside_probe.py 11008 4096 2>&1 | cut -c1-110
if [ $rc -eq 0 ]; then
  timeout 1500 python tools/calib_run.py 100 > gpurun_out/calib_r02.jsonl 2> gpurun_out/calib_r02.err; echo "calib rc=$?"
  timeout 900 python tools/c5_oracle_parity.py > gpurun_out/c5_parity.jsonl 2> gpurun_out/c5_parity.err; echo "c5 rc=$?"; tail -1 gpurun_out/c5_parity.jsonl
fi
