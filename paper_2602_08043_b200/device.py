"""Device-memory plumbing for the Python layer (PyTorch is used only to own
device buffers and streams; all compute goes through libvabft_b200.so).

Host matrices follow vabft::Matrix (proj/include/vabft/precision.hpp:94-131):
FP64 storage holding values on the format's grid. On the device they live in
native storage: BF16/FP16 as 16-bit patterns, FP32 as float, FP64 as double.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _capi

TORCH_DTYPES = {"bf16": torch.bfloat16, "fp16": torch.float16, "fp32": torch.float32, "fp64": torch.float64}


def fmt_name(fmt) -> str:
    if isinstance(fmt, str):
        return fmt
    return {v: k for k, v in _capi.FORMAT_CODES.items()}[int(fmt)]


def to_device(x: np.ndarray, fmt, device="cuda") -> torch.Tensor:
    """Host FP64 values (on the format grid) -> native device storage."""
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
    return t.to(TORCH_DTYPES[fmt_name(fmt)]).to(device).contiguous()


def to_host(t: torch.Tensor) -> np.ndarray:
    return t.detach().to(torch.float64).cpu().numpy()


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def empty(shape, dtype, device="cuda"):
    return torch.empty(shape, dtype=dtype, device=device)


def zeros(shape, dtype, device="cuda"):
    return torch.zeros(shape, dtype=dtype, device=device)
