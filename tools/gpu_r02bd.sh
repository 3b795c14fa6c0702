bash tools/gpu_r02bc.sh > /dev/null 2>&1; python tools/ncu_stats_summary.py gpurun_out/ncu_stats.csv gpurun_out/r02_ncu_stats_passes.json | python3 -c "
import json,sys; d=json.load(sys.stdin)
for k,v in d['kernels'].items(): print(k, round(v['us'],1), 'us', round(v['algorithmic_GBps']), 'GB/s alg', round(v['frac_of_hbm_peak'],3))"
python tools/wide_probe.py 2>&1 | tail -1
timeout 1200 python -m pytest tests/ -m gpu -x -q -k "wide or fp32 or fp64 or tf32 or config or operand" 2>&1 | tail -2
