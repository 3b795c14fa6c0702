# refresh C4 lines: LLaMA batch (224 GEMMs) and the N-split GEMM
timeout 1200 python bench.py --config llama --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_llama.json 2> gpurun_out/bench_llama.err; echo "llama rc=$?"
timeout 900 python bench.py --config nsplit --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_nsplit.json 2> gpurun_out/bench_nsplit.err; echo "nsplit rc=$?"
for f in llama nsplit; do python -c "
import json; d=json.loads(open('gpurun_out/bench_$f.json').read().strip().splitlines()[-1])
print('$f', round(d['value'],1), round(d['abft_overhead_pct'],2), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'], d['fpr'])"; done
