python tools/trace_probe.py 4096
VABFT_PAIR=1 python tools/trace_probe.py 8192x4096x4096
timeout 600 python bench.py --steps 20 --warmup 5 --no-formats --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "c2 rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/bench_c2.json').read().strip().splitlines()[-1]); print(d['value'], d['fused_vs_plain'], d['clocks'])"
