"""Diagnostic: page-locked table upload time through the C ABI (sliced feeder) vs a raw copy.
   SOFG_UPLOAD_SLICE_MB=<mb> python tools/upload_probe.py"""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2603_00326_b200 as sofg

n, d = 1_000_000, 4096
A = sofg.Context(0)
hptr = A.L.sofg_host_alloc(n * d * 4)
Xh = np.ctypeslib.as_array((C.c_float * (n * d)).from_address(hptr)).reshape(d, n)
Xh[:] = 1.0
yh = np.zeros(n, np.int32)
for it in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    A.upload_ptr(hptr, yh, n, d, 2)
    A.train_forest(sofg.TrainConfig(n_trees=1, mode="dynamic", breakeven=512, seed=7, bootstrap_fraction=1e-5))
    torch.cuda.synchronize()
    print("slice_mb", os.environ.get("SOFG_UPLOAD_SLICE_MB", "32"), "upload+tiny train", round(time.perf_counter() - t, 3), flush=True)
src = torch.from_numpy(Xh.reshape(-1)[: 1 << 30])  # 4 GB view of the page-locked buffer
dst = torch.empty(src.numel(), dtype=torch.float32, device="cuda")
for it in range(2):
    torch.cuda.synchronize(); t = time.perf_counter(); dst.copy_(src, non_blocking=True); torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print("raw 4 GB copy", round(dt, 3), "s", round(4.295 / dt, 1), "GB/s", flush=True)
