# FP32 B-side: sub-tile FP64 sums + fused transposed TF32 split
VABFT_BSIDE_TRACE=1 timeout 300 python tools/bside_once.py float32 2>&1 | tail -2
timeout 300 python tools/bside_probe.py 2>&1 | tail -4
timeout 1200 python -m pytest tests/ -m gpu -x -q -k "wide or fp32 or tf32 or bside or config" 2>&1 | tail -3
timeout 600 python tools/formats_only.py 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); [print(k, round(v['fused_tflops'],1), round(v['plain_tflops'],1), round(v['abft_overhead_pct'],2)) for k,v in d.items()]"
