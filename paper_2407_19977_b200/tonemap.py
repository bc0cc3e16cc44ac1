"""Display transform on the GPU: Khronos PBR Neutral
tone map -> sRGB -> half-up 8-bit quantization, the reference's
`tonemap_to_u8` (tonemap.py:18-61), evaluated in float64 by `k_tonemap_u8`
behind lt_tonemap_u8.  A progressive render can then ship 3 bytes per pixel
to the host instead of a float64 frame."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib


def tonemap_device(linear, out=None, stream=None):
    """linear: CUDA float32 tensor (..., 3) of non-negative radiance ->
    uint8 tensor of the same shape on the same device."""
    import torch
    if linear.dtype != torch.float32 or not linear.is_cuda or linear.shape[-1] != 3:
        raise ValueError("expected a CUDA float32 tensor with a trailing channel axis of 3")
    lin = linear.contiguous()
    if out is None:
        out = torch.empty(lin.shape, dtype=torch.uint8, device=lin.device)
    st = stream if stream is not None else torch.cuda.current_stream(lin.device)
    _lib.check(_lib.lib().lt_tonemap_u8(C.c_void_p(lin.data_ptr()), lin.numel() // 3,
                                        C.c_void_p(out.data_ptr()), C.c_void_p(st.cuda_stream)))
    return out


def tonemap_to_u8(linear, device: int = 0) -> np.ndarray:
    """Host convenience with the reference's signature: (..., 3) float
    array -> uint8 array (computed on the GPU)."""
    import torch
    a = np.asarray(linear, dtype=np.float64)
    if a.shape[-1] != 3:
        raise ValueError(f"expected trailing channel axis of size 3, got {a.shape}")
    if np.any(a < 0.0):
        raise ValueError("tone map input must be non-negative")
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(f"cuda:{device}")
    return tonemap_device(t).cpu().numpy()


def accumulator_to_u8(acc, stream=None):
    """The display image of a device Accumulator: mean (sum / valid) then the
    tone map, all on the device; returns a (h, w, 3) uint8 CUDA tensor."""
    return tonemap_device(acc.mean().float().contiguous(), stream=stream)
