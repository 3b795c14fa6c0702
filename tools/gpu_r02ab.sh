python tools/ladder_probe.py 4096x4096x4096 4608x4096x4096 4608x4096x8192
PLAIN=1 python tools/trace_probe.py 4096
python tools/trace_probe.py 4096
PLAIN=1 python tools/trace_probe.py 4608x4096x4096
VABFT_SPLIT_LAST=1 python tools/trace_probe.py 4608x4096x4096
