# round-2 final evidence: full GPU suite, smoke, default bench (all lines), reference arm, bench launch list
timeout 1500 python -m pytest tests/ -m gpu -x -q > gpurun_out/t_all.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 1200 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-formats --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo "ncu rc=$?"
python tools/summarize_launches.py gpurun_out/launches_bench.csv "ncu --metrics gpu__time_duration.sum --clock-control none python bench.py --steps 2 --warmup 3 --no-formats --no-cpu-baseline" > gpurun_out/launches_bench.txt 2>&1; head -30 gpurun_out/launches_bench.txt
