"""Run the device e_max calibration (online + offline, BF16) and print JSON."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_08043_b200.calibration import calibrate  # noqa: E402
out = {}
fmt = sys.argv[2] if len(sys.argv) > 2 else "bf16"
for mode in ("online", "offline"):
    r = calibrate(fmt, sizes=(128, 256, 512, 1024, 2048, 4096, 8192, 16384), trials=int(sys.argv[1]) if len(sys.argv) > 1 else 8, mode=mode)
    out[mode] = r.as_dict()
    out[mode]["e_max_at"] = {str(k): r.e_max_for(k) for k in (768, 1024, 3072, 4096, 11008, 16384)}
print(json.dumps(out))
