# round 2: GPU tests (incl. the BASELINE-config parity tests) + smoke
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -5 gpurun_out/smoke.log
