import time, torch, json, os
res={}
torch.cuda.synchronize()
for gb in (1, 4, 34):
    n = gb * (1 << 30) // 4
    torch.cuda.synchronize(); t0=time.perf_counter()
    x = torch.empty(n, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize(); t1=time.perf_counter()
    x.zero_(); torch.cuda.synchronize(); t2=time.perf_counter()
    del x
    torch.cuda.empty_cache(); torch.cuda.synchronize(); t3=time.perf_counter()
    res[f"{gb}GB"]={"malloc_ms":1e3*(t1-t0),"first_touch_zero_ms":1e3*(t2-t1),"free_ms":1e3*(t3-t2)}
res["conf"]=os.environ.get("PYTORCH_CUDA_ALLOC_CONF")
print(json.dumps(res))
