"""Diagnostic: does a page-locked table upload on a second context overlap training on the first?"""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2603_00326_b200 as sofg

n, d = 1_000_000, 4096
A = sofg.Context(0)
A.generate_trunk(n, d, 2, seed=1)
hptr = A.L.sofg_host_alloc(n * d * 4)
Xh = np.ctypeslib.as_array((C.c_float * (n * d)).from_address(hptr)).reshape(d, n)
yh = np.zeros(n, np.int32)
A.download(Xh, yh)
B = sofg.Context(0)
cfg = lambda b: sofg.TrainConfig(n_trees=10000, mode="dynamic", breakeven=512, seed=7, tree_begin=b, tree_end=b + 100)
B.upload_ptr(hptr, yh, n, d, 2); B.train_forest(cfg(0)); A.train_forest(cfg(100))
torch.cuda.synchronize()
t = time.perf_counter(); A.train_forest(cfg(200)); torch.cuda.synchronize(); print("train A alone", time.perf_counter() - t)
t = time.perf_counter(); B.upload_ptr(hptr, yh, n, d, 2); t1 = time.perf_counter(); torch.cuda.synchronize(); print("upload B alone: call", t1 - t, "landed", time.perf_counter() - t)
t = time.perf_counter(); B.upload_ptr(hptr, yh, n, d, 2); t1 = time.perf_counter()
A.train_forest(cfg(300)); t2 = time.perf_counter(); torch.cuda.synchronize(); t3 = time.perf_counter()
print("upload B call", t1 - t, "train A", t2 - t1, "sync", t3 - t2)
t = time.perf_counter(); B.train_forest(cfg(400)); print("train B after", time.perf_counter() - t)
