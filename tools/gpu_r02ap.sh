# HEAD check after the re-entry: full GPU suite, smoke, default bench, B-side probe
timeout 1500 python -m pytest tests/ -m gpu -x -q > gpurun_out/t_all.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench_default.json
timeout 300 python tools/bside_probe.py 2>&1 | tail -8
