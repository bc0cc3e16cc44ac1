"""Worker-thread controls of the reference (_parallel.py:23-36).  The render
runs on the GPU, so the CPU thread count has no effect on results or speed;
the functions exist so callers of the reference keep working."""
from __future__ import annotations

import os

_workers = max(1, os.cpu_count() or 1)


def thread_cap() -> int:
    """Upper bound accepted by set_worker_count."""
    return max(1, os.cpu_count() or 1)


def set_worker_count(threads: int | None) -> int:
    """Record the requested host worker count (None = all cores), clamped
    to [1, cap] as the reference clamps it; returns the count in effect.
    GPU work is unaffected."""
    global _workers
    if threads is None:
        threads = os.cpu_count() or 1
    _workers = max(1, min(int(threads), thread_cap()))
    return _workers
