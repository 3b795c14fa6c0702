# ncu metrics of the statistics passes (B-side BF16 / FP32, wide A pass, combine)
python tools/stats_once.py > /dev/null 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"bside_kernel|wide_apart|wide_combine" --csv python tools/stats_once.py > gpurun_out/ncu_stats.csv 2> gpurun_out/ncu_stats.err; echo rc=$?
python tools/ncu_stats_summary.py gpurun_out/ncu_stats.csv gpurun_out/r02_ncu_stats_passes.json | head -60
