"""HBM read / write / copy bandwidth with torch ops (CUDA events). GPU only."""
import json
import torch

n = 1 << 29  # 2 GiB of fp32
a = torch.empty(n, device="cuda")
b = torch.empty(n, device="cuda")
a.fill_(1.0)
b.fill_(2.0)


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


res = {}
res["write_GBs"] = 4 * n / t(lambda: a.fill_(3.0)) / 1e9
res["read_GBs"] = 4 * n / t(lambda: torch.sum(a)) / 1e9
res["copy_GBs"] = 8 * n / t(lambda: b.copy_(a)) / 1e9
h = n // 3
res["read2_write1_GBs"] = 12 * h / t(lambda: torch.add(a[:h], a[h:2 * h], out=b[:h])) / 1e9
print(json.dumps(res))
