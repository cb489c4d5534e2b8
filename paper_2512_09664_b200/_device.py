"""Device plumbing: numpy/torch <-> CUDA tensors, current stream handles."""

from __future__ import annotations

import numpy as np
import torch


def cuda_device(device=None) -> torch.device:
    if not torch.cuda.is_available():
        from ._lib import BackendUnavailable

        raise BackendUnavailable("no CUDA device is available; this package has no CPU path")
    if device is None or device == "cpu" or device == "cuda":
        return torch.device("cuda", torch.cuda.current_device())
    dev = torch.device(device)
    if dev.type != "cuda":
        return torch.device("cuda", torch.cuda.current_device())
    if dev.index is None:
        return torch.device("cuda", torch.cuda.current_device())
    return dev


def stream_ptr(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def to_dev(arr, dtype: torch.dtype, device: torch.device) -> torch.Tensor:
    """Contiguous CUDA tensor of `dtype` (no copy when already conforming)."""
    if isinstance(arr, torch.Tensor):
        t = arr
    else:
        a = np.asarray(arr)
        if a.dtype == np.bool_:
            a = a.astype(np.uint8)
        t = torch.from_numpy(np.ascontiguousarray(a))
    if t.dtype == torch.bool:
        t = t.to(torch.uint8)
    return t.to(device=device, dtype=dtype).contiguous()


def like_input(result: torch.Tensor, template):
    """Return numpy when the caller passed numpy, else the CUDA tensor."""
    if isinstance(template, torch.Tensor):
        return result
    return result.cpu().numpy()
