import sys, os; sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import numpy as np, oracle_lib, torch
torch.cuda.is_available()
import paper_2603_00326_b200 as sofg
from test_gpu_parity import _cfg
ref = oracle_lib.get("port")
X, y = ref.generate_trunk(9000, 20, 6)
Xq = np.round(X * 8) / 8
ctx = sofg.Context(0)
for mode, be in (("exact", None), ("dynamic", 5000)):
    for name, data in (("X", X), ("Xq", Xq)):
        ctx.upload(data, y, 2)
        gc, oc = _cfg(n_trees=3, mode=mode, breakeven=be, seed=21, n_workers=int(os.environ.get("NW", "0")))
        print("=== run", mode, name, flush=True)
        sys.stderr.flush()
        g = ctx.train_forest(gc)
