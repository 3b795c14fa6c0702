timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/gputest.log
for d in 0 1 2; do echo "debug=$d"; VABFT_BSIDE_DEBUG=$d timeout 300 python tools/bside_probe.py 4096 4096 2>&1 | cut -c1-140; done
timeout 300 python tools/bside_probe.py 11008 4096 2>&1 | cut -c1-140
timeout 300 python tools/formats_only.py > gpurun_out/formats.log 2>&1; tail -3 gpurun_out/formats.log | cut -c1-900
