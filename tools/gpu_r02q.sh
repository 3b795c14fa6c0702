python tools/wide_probe.py 4096 1
python tools/wide_probe.py 4096 3
python tools/wide_probe.py 2048 1 fp64
python tools/wide_probe.py 4096 1 > /dev/null 2>&1 && ncu --set full --import-source on --clock-control none -k regex:wide_apart -s 1 -c 1 -o gpurun_out/apart_prof python tools/wide_probe.py 4096 1 > gpurun_out/ncu_apart.log 2>&1; echo "ncu rc=$?"
