"""Device-tensor plumbing shared by the host modules: torch owns memory and
streams; the kernels only see raw pointers (include/minions.h)."""
from __future__ import annotations

import torch

_NATIVE_OK = None


def require_cuda() -> torch.device:
    """The product path runs only on a CUDA device with the native library loaded."""
    global _NATIVE_OK
    if _NATIVE_OK is None:
        from . import _native  # noqa: F401  (raises if the library is missing)
        _NATIVE_OK = True
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2402_15678_b200 needs a CUDA device (sm_100a); "
                           "there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(t: torch.Tensor | None, dtype: torch.dtype | None = None, name: str = "tensor") -> int | None:
    """Raw device pointer of a contiguous CUDA tensor (None -> NULL)."""
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if dtype is not None and t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t.data_ptr()


def as_dev(x, dtype: torch.dtype, device) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=dtype).contiguous()
    return torch.as_tensor(x, dtype=dtype).to(device).contiguous()


_PARTITIONS: dict = {}


def sm_partition_streams(draft_sms: int, device: torch.device, draft_priority: int = 0,
                         verify_priority: int = 0):
    """(draft stream, verify stream, draft SMs, verify SMs) on two green
    contexts splitting the device's SMs (ms_sm_partition) — created once per
    (device, split, priorities) per process and reused by every engine."""
    from . import _native
    import ctypes
    dev = device.index if device.index is not None else torch.cuda.current_device()
    key = (dev, draft_sms, draft_priority, verify_priority)
    if key not in _PARTITIONS:
        sd, sv = ctypes.c_void_p(), ctypes.c_void_p()
        nd, nv = ctypes.c_int(), ctypes.c_int()
        _native.call("ms_sm_partition", dev, draft_sms, draft_priority, verify_priority, ctypes.byref(sd),
                     ctypes.byref(sv), ctypes.byref(nd), ctypes.byref(nv))
        d = torch.device("cuda", dev)
        _PARTITIONS[key] = (torch.cuda.ExternalStream(sd.value, device=d),
                            torch.cuda.ExternalStream(sv.value, device=d), nd.value, nv.value)
    return _PARTITIONS[key]
