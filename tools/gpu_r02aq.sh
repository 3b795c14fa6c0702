# ncu --set full of the statistics passes: B-side (BF16, FP32), wide A pass (FP32)
python tools/bside_once.py > /dev/null 2>&1 || exit 1
python tools/aside_once.py > /dev/null 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:bside_kernel -s 1 -c 1 -o gpurun_out/bside_bf16 python tools/bside_once.py > gpurun_out/ncu_bs16.log 2>&1; echo rc=$?
ncu --set full --import-source on --clock-control none -k regex:bside_kernel -s 1 -c 1 -o gpurun_out/bside_fp32 python tools/bside_once.py float32 > gpurun_out/ncu_bs32.log 2>&1; echo rc=$?
ncu --set full --import-source on --clock-control none -k regex:wide_apart -c 1 -o gpurun_out/apart_fp32 python tools/aside_once.py > gpurun_out/ncu_ap.log 2>&1; echo rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/bside_once.py float32 > gpurun_out/launches_bs32.csv 2>&1
tail -3 gpurun_out/ncu_ap.log
