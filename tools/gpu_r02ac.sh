python tools/fused_once.py > /dev/null 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:tc_gemm_kernel -c 2 -o gpurun_out/c2_full python tools/fused_once.py > gpurun_out/ncu_c2_full.log 2>&1
echo ncu rc=$?
tail -3 gpurun_out/ncu_c2_full.log
