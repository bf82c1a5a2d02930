import sys, time, ctypes as C, os
sys.path.insert(0, '.')
import numpy as np
import paper_2603_00326_b200 as sofg
from paper_2603_00326_b200 import _export
ctx = sofg.Context(0)
ctx.generate_trunk(1_000_000, 4096, 2, seed=1)
NT = int(sys.argv[1]) if len(sys.argv) > 1 else 100
for groups in ("1",):
    os.environ["SOFG_GROUPS"] = groups
    for it in range(3):
        cfg = sofg.TrainConfig(n_trees=1000, mode="dynamic", breakeven=1024, seed=7, tree_begin=NT * it, tree_end=NT * it + NT)
        c = cfg.to_c(); h = C.c_void_p()
        t0 = time.perf_counter()
        rc = ctx.L.sofg_train_forest(ctx.h, C.byref(c), C.byref(h))
        t1 = time.perf_counter()
        f = _export(h)
        t2 = time.perf_counter()
        ctx.L.sofg_forest_free(h)
        t3 = time.perf_counter()
        st = ctx.stats()
        print(f"groups={groups} it={it} train {1e3*(t1-t0):.0f} ms export {1e3*(t2-t1):.0f} ms free {1e3*(t3-t2):.0f} ms nodes {len(f.left)}", flush=True)
