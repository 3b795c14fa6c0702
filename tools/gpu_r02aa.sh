python tools/l2_probe.py
K=8192 python tools/l2_probe.py
python tools/peaks_probe.py > gpurun_out/peaks.json; cat gpurun_out/peaks.json
