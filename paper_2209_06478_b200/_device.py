"""Device plumbing: CUDA availability, streams, workspaces, int32 narrowing.

PyTorch is used only for device buffers and streams; all arithmetic on the
hot path runs in the sm_100a kernels of libdynsparse_b200.so.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native
from .errors import DeviceError, IndexOutOfRange

I32_MAX = 2**31 - 1
I32_MIN = -(2**31)

_WORKSPACES: dict[tuple[int, int], torch.Tensor] = {}


def require_cuda(device=None) -> torch.device:
    """Resolve the execution device; fail loudly when there is none."""
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device available: dynsparse-b200 has no CPU fallback")
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    dev = torch.device(device)
    if dev.type != "cuda":
        raise DeviceError(f"device {dev} is not a CUDA device")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


def stream(device: torch.device) -> int:
    """cudaStream_t of the current torch stream on ``device`` (as an int)."""
    return torch.cuda.current_stream(device).cuda_stream


def ptr(t: torch.Tensor | None) -> int | None:
    if t is None or t.numel() == 0:
        return None
    return t.data_ptr()


def new_workspace(device: torch.device) -> torch.Tensor:
    """A fresh zero-initialised reduction workspace (partials, tickets, the
    grid-barrier words) owned by the caller -- what a captured CUDA graph
    embeds, so two graphs never share one even when their capture streams'
    handles were recycled."""
    nbytes = int(_native.load().ds_cg_workspace_bytes())
    return torch.zeros(nbytes, dtype=torch.uint8, device=device)


def workspace(device: torch.device) -> torch.Tensor:
    """Zero-initialised reduction workspace for eager launches on (device,
    current stream): work on one stream is serialised, so it is shared."""
    key = (device.index, stream(device))
    ws = _WORKSPACES.get(key)
    if ws is None:
        ws = new_workspace(device)
        _WORKSPACES[key] = ws
    return ws


def to_index_tensor(values, device: torch.device) -> torch.Tensor:
    """int64 host indices -> int32 device tensor (range-checked, exact)."""
    if isinstance(values, torch.Tensor):
        t = values.detach()
        if t.numel():
            lo, hi = int(t.min()), int(t.max())
            if lo < I32_MIN or hi > I32_MAX:
                raise IndexOutOfRange("index values do not fit the int32 device layout")
        return t.to(device=device, dtype=torch.int32).contiguous()
    arr = np.ascontiguousarray(values, dtype=np.int64)
    if arr.size and (int(arr.min()) < I32_MIN or int(arr.max()) > I32_MAX):
        raise IndexOutOfRange("index values do not fit the int32 device layout")
    return torch.from_numpy(arr.astype(np.int32)).to(device).contiguous()


def to_value_tensor(values, device: torch.device) -> torch.Tensor:
    if isinstance(values, torch.Tensor):
        return values.detach().to(device=device, dtype=torch.float64).contiguous()
    arr = np.ascontiguousarray(values, dtype=np.float64)
    return torch.from_numpy(arr).to(device).contiguous()


def index_to_host(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy().astype(np.int64)


def value_to_host(t: torch.Tensor) -> np.ndarray:
    return np.ascontiguousarray(t.detach().cpu().numpy(), dtype=np.float64)


def check_dims(*dims: int) -> None:
    for d in dims:
        if d > I32_MAX:
            raise DeviceError(f"dimension {d} exceeds the int32 device index range")
