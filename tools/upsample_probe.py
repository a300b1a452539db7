"""Lanczos level transfer at C4 scale: (Z/2, N/2, N/2) -> (Z, N, N) with K9f; GPU only."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_28756_b200.multires import upsample_stack  # noqa: E402

res = {}
for n, z in ((2048, 64), (2048, 512), (2048, 2048), (1024, 1024)):
    x = torch.randn((z // 2, n // 2, n // 2), device="cuda")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    y = upsample_stack(x, n, z)
    torch.cuda.synchronize()
    cold = time.perf_counter() - t0
    del y
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    y = upsample_stack(x, n, z)
    torch.cuda.synchronize()
    warm = time.perf_counter() - t0
    res[f"{z}x{n}^2"] = {"cold_ms": 1e3 * cold, "warm_ms": 1e3 * warm,
                         "GBs_at_4.5B_per_voxel": 4.5 * z * n * n / warm / 1e9}
    del x, y
    torch.cuda.empty_cache()
print(json.dumps(res))
