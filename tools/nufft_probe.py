"""One-time kernels at C3 scale: R*g / FBP (K8 + K7 + grid FFTs) over a 64-slice 2048^2
slab and a Lanczos level transfer (K9). GPU only; used for ncu captures."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28756_b200 as tf  # noqa: E402
from paper_2603_28756_b200.multires import upsample_stack  # noqa: E402
from paper_2603_28756_b200.radon import back_project_stack, fbp_stack  # noqa: E402

z = int(os.environ.get("PROBE_SLICES", "64"))
ang = np.linspace(0, np.pi, 128, endpoint=False)
geom = tf.ScanGeometry(angles=ang, detector_bins=2048, image_side=2048)
plan = tf.NufftPlan(2048, tf.polar_sampling(geom), 1e-6)
rows = torch.randn((z, 128, 2048), device="cuda")
coarse = torch.randn((z // 2, 1024, 1024), device="cuda")


def ev(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


res = {"slices": z,
       "rstar_ms": ev(lambda: back_project_stack(plan, rows)),
       "fbp_ms": ev(lambda: fbp_stack(plan, rows)),
       "lanczos_up2_ms": ev(lambda: upsample_stack(coarse, 2048, z))}
res["rstar_slices_per_s"] = z / res["rstar_ms"] * 1e3
print(json.dumps(res))
