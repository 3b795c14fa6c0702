# wide A pass: streaming without arrivals + staged combine kernel
VABFT_APART_TRACE=1 python tools/ap_trace.py 2>&1 | grep -v Warn | tail -8
python tools/wide_probe.py 2>&1 | tail -1
python tools/wide_probe.py 4096 3 2>&1 | tail -1
python tools/wide_probe.py 2048 3 fp64 2>&1 | tail -1
timeout 1200 python -m pytest tests/ -m gpu -x -q -k "wide or fp32 or fp64 or tf32 or config or operand or campaign or calib" 2>&1 | tail -2
timeout 600 python tools/formats_only.py 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); [print(k, round(v['fused_tflops'],1), round(v['plain_tflops'],1), round(v['abft_overhead_pct'],2)) for k,v in d.items()]"
