# FP32 (3xTF32), TF32 (one pass) device calibrations -> gpurun_out/
for f in fp32 tf32; do timeout 600 python tools/calib_run.py 4 $f > gpurun_out/calib_$f.json 2> gpurun_out/calib_$f.err; done
