python tools/fp32_once.py > /dev/null 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:wide_apart -s 2 -c 1 -o gpurun_out/apart_r02_cur python tools/fp32_once.py > gpurun_out/ncu_apart_cur.log 2>&1; echo rc=$?
