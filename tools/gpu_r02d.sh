timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/gputest.log
timeout 300 python tools/bside_probe.py 4096 4096 > gpurun_out/bside_4096.jsonl 2>&1; echo "probe rc=$?"; cat gpurun_out/bside_4096.jsonl
timeout 300 python tools/bside_probe.py 11008 4096 > gpurun_out/bside_11008.jsonl 2>&1; cat gpurun_out/bside_11008.jsonl
timeout 300 python tools/bside_probe.py 4096 11008 >> gpurun_out/bside_11008.jsonl 2>&1; tail -4 gpurun_out/bside_11008.jsonl
python tools/bside_probe.py 4096 4096 > /dev/null 2>&1 && ncu --set full --import-source on --clock-control none -k regex:bside_kernel -s 2 -c 2 -o gpurun_out/bside_prof python tools/bside_probe.py 4096 4096 > gpurun_out/ncu_bside.log 2>&1; echo "ncu rc=$?"
