"""Host<->device copy rates on the GPU box: pinned vs pageable sources and
multi-threaded host memcpy into pinned memory (scene-upload design input)."""
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

n = 200 << 20
dev = torch.device("cuda", 0)
d = torch.empty(n, dtype=torch.uint8, device=dev)
pin = torch.empty(n, dtype=torch.uint8, pin_memory=True)
page = np.ones(n, np.uint8)
pin.numpy()[:] = 1


def timeit(f, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return n / best / 1e9


print("pinned H2D GB/s", timeit(lambda: d.copy_(pin, non_blocking=True)))
print("pageable H2D GB/s", timeit(lambda: d.copy_(torch.from_numpy(page))))
print("pinned D2H GB/s", timeit(lambda: pin.copy_(d, non_blocking=True)))
for th in (1, 2, 4, 8, 16):
    ex = ThreadPoolExecutor(th)
    dst = pin.numpy()

    def cp():
        step = n // th
        list(ex.map(lambda i: np.copyto(dst[i * step:(i + 1) * step],
                                        page[i * step:(i + 1) * step]), range(th)))
    print(f"host memcpy pageable->pinned {th} threads GB/s", timeit(cp))
