"""Display transform on the GPU: Khronos PBR Neutral
tone map -> sRGB -> half-up 8-bit quantization (tonemap.py:18-61), and the
PNG / raw-dump writers (tonemap.py:64-77).

* The reference's host API -- `pbr_neutral_tonemap`, `linear_to_srgb`,
  `srgb_to_linear`, `quantize_to_u8`, `tonemap_to_u8` -- takes float64
  arrays of any leading shape and evaluates them on the device in float64
  (lt_display_batch, csrc/lt_query64.cu), with the reference's validation.
* `tonemap_device` / `accumulator_to_u8` run the fused `k_tonemap_u8` on a
  device frame, so a progressive render ships 3 bytes per pixel to the host
  instead of a float64 frame.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib, query


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


def _rgb(color) -> np.ndarray:
    c = np.asarray(color, dtype=np.float64)
    if c.shape[-1] != 3:
        raise ValueError(f"expected trailing channel axis of size 3, got {c.shape}")
    if np.any(c < 0.0):
        raise ValueError("tone map input must be non-negative")
    return c


def pbr_neutral_tonemap(color) -> np.ndarray:
    """Khronos PBR Neutral (tonemap.py:18-41), float64 on the device."""
    return query.display(0, _rgb(color))


def linear_to_srgb(x) -> np.ndarray:
    """sRGB encode of clipped [0, 1] values (tonemap.py:44-47)."""
    return query.display(1, x)


def srgb_to_linear(x) -> np.ndarray:
    """tonemap.py:50-52."""
    return query.display(2, x)


def quantize_to_u8(x) -> np.ndarray:
    """floor(255 clip(v, 0, 1) + 0.5) (tonemap.py:55-58)."""
    return query.display(3, x)


def tonemap_to_u8(linear) -> np.ndarray:
    """The full display pipeline (tonemap.py:61-62): tone map, sRGB encode,
    quantize -- each stage float64 on the device."""
    return quantize_to_u8(linear_to_srgb(pbr_neutral_tonemap(linear)))


def write_png(path, pixels_u8) -> None:
    """8-bit RGB PNG, no alpha (tonemap.py:64-69)."""
    from PIL import Image
    arr = np.asarray(pixels_u8)
    if arr.dtype != np.uint8 or arr.ndim != 3 or arr.shape[2] != 3:
        raise ValueError(f"expected uint8 array of shape (h, w, 3), got {arr.dtype} {arr.shape}")
    Image.fromarray(arr, mode="RGB").save(path, format="PNG")


def write_linear_dump(path, linear) -> None:
    """Row-major little-endian float32 RGB triplets (tonemap.py:72-77)."""
    arr = np.asarray(linear, dtype=np.float64)
    if arr.ndim != 3 or arr.shape[2] != 3:
        raise ValueError(f"expected array of shape (h, w, 3), got {arr.shape}")
    np.ascontiguousarray(arr, dtype="<f4").tofile(path)


def accumulator_to_u8(acc, stream=None):
    """The display image of a device Accumulator: mean (sum / valid) then the
    tone map, all on the device; returns a (h, w, 3) uint8 CUDA tensor."""
    return tonemap_device(acc.mean().float().contiguous(), stream=stream)
