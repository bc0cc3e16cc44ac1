"""PCG32 stream API (rng.py:29-109 of the reference), host side.

The device kernels carry the same integer arithmetic (csrc/lt_device.cuh:
pcg_next, mix64, seed_stream); these Python-int versions serve the public
API and let callers build the (state, increment) pairs trace_radiance takes.
"""
from __future__ import annotations

from dataclasses import dataclass

_M64 = (1 << 64) - 1
_MULT = 6364136223846793005


@dataclass(frozen=True)
class PcgState:
    state: int
    increment: int


def _step(state: int, inc: int) -> tuple[int, int]:
    """XSH-RR output of `state`, and the successor state."""
    x = (((state >> 18) ^ state) >> 27) & 0xFFFFFFFF
    r = state >> 59
    out = ((x >> r) | (x << ((32 - r) & 31))) & 0xFFFFFFFF
    return out, (state * _MULT + inc) & _M64


def _mix64(x: int) -> int:
    z = (x + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def pcg_seed(init_state: int, init_seq: int) -> PcgState:
    inc = ((init_seq & _M64) << 1 | 1) & _M64
    _, s = _step(0, inc)
    s = (s + (init_state & _M64)) & _M64
    _, s = _step(s, inc)
    return PcgState(s, inc)


def pcg_next_u32(rng: PcgState) -> tuple[int, PcgState]:
    out, s = _step(rng.state, rng.increment)
    return out, PcgState(s, rng.increment)


def next_unit_real(rng: PcgState) -> tuple[float, PcgState]:
    out, rng = pcg_next_u32(rng)
    return out * (1.0 / 4294967296.0), rng


def seed_stream(pixel_index: int, sample_index: int, global_seed: int) -> PcgState:
    if pixel_index < 0 or sample_index < 0:
        raise ValueError("pixel_index and sample_index must be non-negative")
    return pcg_seed(_mix64((global_seed & _M64) ^ _mix64(sample_index)), _mix64(pixel_index))
