for f in bfloat16 float32; do VABFT_BSIDE_TRACE=1 timeout 120 python tools/bside_once.py $f 2>&1 | tail -2; done
VABFT_BSIDE_DEBUG=1 VABFT_BSIDE_TRACE=1 timeout 120 python tools/bside_once.py 2>&1 | tail -2
VABFT_BSIDE_DEBUG=1 ncu --set full --import-source on --clock-control none -k regex:bside_ring -s 1 -c 1 -o gpurun_out/ring_bf16_nochain2 python tools/bside_once.py > gpurun_out/ncu_ring3.log 2>&1; echo rc=$?
