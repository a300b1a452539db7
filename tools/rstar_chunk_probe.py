"""R*g (64 x 2048^2, 128 angles) vs the NUFFT workspace chunk (slices per spreading
launch) and the spreading tile order (heaviest first vs natural); GPU only."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28756_b200 as tf  # noqa: E402
from paper_2603_28756_b200 import nufft  # noqa: E402
from paper_2603_28756_b200.radon import back_project_stack  # noqa: E402

ang = np.linspace(0, np.pi, 128, endpoint=False)
geom = tf.ScanGeometry(angles=ang, detector_bins=2048, image_side=2048)
plan = tf.NufftPlan(2048, tf.polar_sampling(geom), 1e-6)
rows = torch.randn((64, 128, 2048), device="cuda")
res = {}
ref = None
t = plan.device_tables()
back_project_stack(plan, rows)
lpt = t["tile_order"]
natural = torch.arange(lpt.numel(), dtype=torch.int32, device=lpt.device)
for gb in (1, 2, 4, 1, 8, 13):
    for name, order in (("lpt", lpt), ("natural", natural)):
        nufft._WS_BYTES = gb << 30
        t["tile_order"] = order
        back_project_stack(plan, rows)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            out = back_project_stack(plan, rows)
        b.record()
        torch.cuda.synchronize()
        if ref is None:
            ref = out.clone()
        key = f"ws_{gb}GB_{(gb << 30) // 201326592}slices_{name}"
        res.setdefault(key, []).append(round(a.elapsed_time(b) / 3, 3))
        res.setdefault("bitwise_equal", []).append(bool(torch.equal(out, ref)))
t["tile_order"] = lpt
print(json.dumps(res))
