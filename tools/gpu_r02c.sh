# round 2: config parity + bench lines (c2, reference, llama, nsplit) + tensor-pipe ncu of the fused / plain kernels
timeout 600 python -m pytest tests/test_gpu_configs.py -x -q > gpurun_out/gputest_configs.log 2>&1; echo "configs rc=$?"; tail -3 gpurun_out/gputest_configs.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "c2 rc=$?"
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_c2.json 2> gpurun_out/bench_ref_c2.err; echo "ref rc=$?"
timeout 600 python bench.py --config llama --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_llama.json 2> gpurun_out/bench_llama.err; echo "llama rc=$?"
timeout 600 python bench.py --config nsplit --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_nsplit.json 2> gpurun_out/bench_nsplit.err; echo "nsplit rc=$?"
python tools/fused_once.py 4096 4096 4096 online > gpurun_out/fused_once.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.sum.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tensor_subpipe_hmma.sum,sm__cycles_elapsed.avg.per_second \
  --clock-control none -k regex:tc_gemm --csv --log-file gpurun_out/ncu_tensor_pipe_c2.csv python tools/fused_once.py 4096 4096 4096 online > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?"
