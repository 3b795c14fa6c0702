set -x
nvidia-smi -L; nproc; lscpu | grep -E 'Model name|^CPU\(s\)|Thread|Socket'
ncu --query-metrics --chip gb100 > gpurun_out/query_metrics.txt 2>&1
ncu --query-metrics-mode suffix --metrics sm__pipe_tensor_cycles_active,sm__inst_executed_pipe_uma --chip gb100 > gpurun_out/query_suffix.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/gputest.log
