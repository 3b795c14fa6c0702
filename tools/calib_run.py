"""Device e_max calibration of the fused paths (calibration.calibrate, the
reference protocol of calibration.cpp:88-150 on the B200 kernels) and print
one JSON object per (format, mode).

  python tools/calib_run.py [trials] [formats] > profiles/r02_calibration_device.jsonl
"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_08043_b200.calibration import calibrate  # noqa: E402
trials = int(sys.argv[1]) if len(sys.argv) > 1 else 100
fmts = (sys.argv[2] if len(sys.argv) > 2 else "bf16:online,bf16:offline,fp16:online,fp32:online,tf32:online,fp64:online").split(",")
sizes = (128, 256, 512, 1024, 2048, 4096, 8192, 16384)
for fm in fmts:
    fmt, mode = fm.split(":")
    t0 = time.time()
    r = calibrate(fmt, sizes=sizes, trials=trials, mode=mode)
    out = r.as_dict()
    out["e_max_at"] = {str(k): r.e_max_for(k) for k in (768, 1024, 3072, 4096, 11008, 16384)}
    out["seconds"] = round(time.time() - t0, 1)
    print(json.dumps(out), flush=True)
