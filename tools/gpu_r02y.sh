timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; rc=$?; echo "pytest rc=$rc"; tail -15 gpurun_out/gputest.log | grep -E "passed|failed|Error|assert"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "c2 rc=$?"
