python tools/bside_once.py > /dev/null 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:bside_ring -s 1 -c 1 -o gpurun_out/ring_bf16 python tools/bside_once.py > gpurun_out/ncu_ring.log 2>&1; echo rc=$?
VABFT_BSIDE_DEBUG=1 ncu --set full --import-source on --clock-control none -k regex:bside_ring -s 1 -c 1 -o gpurun_out/ring_bf16_nochain python tools/bside_once.py > gpurun_out/ncu_ring2.log 2>&1; echo rc=$?
