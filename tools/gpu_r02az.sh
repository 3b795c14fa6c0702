# after the fused FP32 split + bench mixed-scale / bside fields: full GPU suite, smoke, bench
timeout 1500 python -m pytest tests/ -m gpu -x -q > gpurun_out/t_all.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02az.json 2> gpurun_out/bench_r02az.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_r02az.json').read().strip().splitlines()[-1])
print(d['value'], d['abft_overhead_pct'], d['roofline']['frac'], d['clocks'])
print('mixed', d['mixed_scale'], 'bside_us', d['bside_update_us'])
print({k:(round(v['fused_tflops'],1), round(v['abft_overhead_pct'],2)) for k,v in d['formats'].items()})
print('e2e', d['e2e']['value'])"
