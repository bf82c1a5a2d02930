import sys, time, ctypes as C
sys.path.insert(0, '.')
import numpy as np
import paper_2603_00326_b200 as sofg
n, d = 1_000_000, 4096
ctx = sofg.Context(0)
ctx.generate_trunk(n, d, 2, seed=1)
hptr = ctx.L.sofg_host_alloc(n * d * 4)
Xh = np.ctypeslib.as_array((C.c_float * (n * d)).from_address(hptr)).reshape(d, n)
yh = np.zeros(n, np.int32)
ctx.download(Xh, yh)
ctx.set_stats(1)
for s in range(4):
    cfg = sofg.TrainConfig(n_trees=1000, mode="dynamic", breakeven=512, seed=7, tree_begin=100 * s, tree_end=100 * s + 100)
    ctx.reset_stats()
    t0 = time.perf_counter(); ctx.upload_ptr(hptr, yh, n, d, 2); t1 = time.perf_counter()
    f = ctx.train_forest(cfg); t2 = time.perf_counter()
    st = ctx.stats()
    print(f"step {s}: upload {1e3*(t1-t0):.0f} ms train {1e3*(t2-t1):.0f} ms", {k: round(v, 1) for k, v in st.items() if k in ('ms_train_total','ms_waves_total','ms_host_bootstrap','ms_host_roots','ms_host_submit','ms_host_post','ms_host_prep','ms_host_final')}, flush=True)
