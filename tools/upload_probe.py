"""to_device (float64 host -> fp32 device) of a C4-sized sinogram (2048 x 128 x 2048):
first call and repeated call, 8 vs 16 staging threads.  GPU only."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_28756_b200 import _device  # noqa: E402

a = np.random.default_rng(0).standard_normal((2048, 128, 2048))
res = {}
for th in (8, 16, 8):
    _device._STAGE_THREADS = th
    if _device._stage_pool is not None:
        _device._stage_pool.shutdown()
        _device._stage_pool = None
    for rep in ("first", "second"):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        x = _device.to_device(a)
        torch.cuda.synchronize()
        res.setdefault(f"{th}thr_{rep}", []).append(round(time.perf_counter() - t0, 4))
        del x
print(json.dumps(res))
