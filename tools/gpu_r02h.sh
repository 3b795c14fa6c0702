export VABFT_BSIDE_DEBUG=2
python tools/bside_probe.py 4096 4096 > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:bside_kernel -s 48 -c 1 -o gpurun_out/bside_fp32 python tools/bside_probe.py 4096 4096 > gpurun_out/ncu1.log 2>&1; echo "ncu rc=$?"
ncu --set full --import-source on --clock-control none -k regex:bside_kernel -s 2 -c 1 -o gpurun_out/bside_bf16 python tools/bside_probe.py 4096 4096 > gpurun_out/ncu2.log 2>&1; echo "ncu rc=$?"
