"""Host-path bounds of the e2e measurement: pinned H2D / D2H bandwidth alone and
concurrent (full duplex), and host float64 <-> fp32 conversion rates with N threads.
GPU only; one JSON line."""
import json
import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

GB = 1 << 30
n = 256 << 20  # fp32 elements: 1 GiB
h32 = torch.empty(n, dtype=torch.float32, pin_memory=True)
h64 = torch.empty(n, dtype=torch.float64, pin_memory=True)
d32 = torch.empty(n, dtype=torch.float32, device="cuda")
d64 = torch.empty(n, dtype=torch.float64, device="cuda")
h32.fill_(1.0)
h64.fill_(1.0)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


res = {}
res["h2d_fp32_GBs"] = 4 * n / timed(lambda: d32.copy_(h32, non_blocking=True)) / 1e9
res["d2h_fp32_GBs"] = 4 * n / timed(lambda: h32.copy_(d32, non_blocking=True)) / 1e9
res["d2h_fp64_GBs"] = 8 * n / timed(lambda: h64.copy_(d64, non_blocking=True)) / 1e9


def duplex():
    with torch.cuda.stream(s1):
        d32.copy_(h32, non_blocking=True)
    with torch.cuda.stream(s2):
        h64.copy_(d64, non_blocking=True)


t = timed(duplex)
res["duplex_h2d_fp32_plus_d2h_fp64_ms_per_GiB_in"] = 1e3 * t
res["duplex_total_GBs"] = 12 * n / t / 1e9
src64 = np.random.default_rng(0).standard_normal(n)  # 2 GiB float64, pageable
dst32 = h32.numpy()
out64 = np.empty(n)
out64[:] = 0.0  # fault in
for th in (1, 4, 8, 16, 32):
    if th > (os.cpu_count() or 1):
        continue
    pool = ThreadPoolExecutor(th)
    part = -(-n // th)

    def narrow():
        list(pool.map(lambda a: np.copyto(dst32[a:a + part], src64[a:a + part], "same_kind"),
                      range(0, n, part)))

    def widen():
        list(pool.map(lambda a: np.copyto(out64[a:a + part], dst32[a:a + part], "same_kind"),
                      range(0, n, part)))

    narrow()
    t0 = time.perf_counter()
    narrow()
    res[f"narrow64to32_{th}thr_GBs_of_input"] = 8 * n / (time.perf_counter() - t0) / 1e9
    widen()
    t0 = time.perf_counter()
    widen()
    res[f"widen32to64_{th}thr_GBs_of_output"] = 8 * n / (time.perf_counter() - t0) / 1e9
    pool.shutdown()
res["cpus"] = os.cpu_count()
print(json.dumps(res))
