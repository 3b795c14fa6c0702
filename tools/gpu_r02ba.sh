# integer exact sums for guard-failing 16-bit rows: timeline, parity tests, bench mixed-scale
MIXED=1 python tools/trace_probe.py 4096 2>&1 | head -9
timeout 1500 python -m pytest tests/ -m gpu -x -q > gpurun_out/t_all.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_all.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_r02ba.json 2> gpurun_out/bench_r02ba.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_r02ba.json').read().strip().splitlines()[-1])
print(d['value'], d['abft_overhead_pct'], d['roofline']['frac'])
print('mixed', d['mixed_scale'], 'bside_us', d['bside_update_us'])"
