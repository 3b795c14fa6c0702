"""bench.py's wide-format lines alone (FP32 3xTF32 / 1xTF32, FP64)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
dev = torch.device("cuda", 0)
flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)
print(json.dumps(bench.measure_formats(dev, flush, torch)))
