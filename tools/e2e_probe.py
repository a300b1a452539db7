"""Break down the host-buffer path of fidelity_grad (64 x 2048^2 float64). GPU only."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_28756_b200 import _device  # noqa: E402

f = np.random.default_rng(5).standard_normal((64, 2048, 2048))
res = {}
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x = _device.to_device(f)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    h = _device.to_host64(x)
    t2 = time.perf_counter()
    res = {"h2d_s": t1 - t0, "d2h_s": t2 - t1, "h2d_GBs": f.nbytes / (t1 - t0) / 1e9,
           "d2h_GBs": h.nbytes / (t2 - t1) / 1e9}
    del h
t0 = time.perf_counter()
g = np.empty_like(f)
np.copyto(g, f)
res["host_copy_1thread_GBs"] = f.nbytes / (time.perf_counter() - t0) / 1e9
res["cpus"] = os.cpu_count()
print(json.dumps(res))
