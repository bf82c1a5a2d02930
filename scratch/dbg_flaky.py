import sys, os; sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import numpy as np, oracle_lib
import torch
print('cuda', torch.cuda.is_available())
import paper_2603_00326_b200 as sofg
from test_gpu_parity import _cfg
ref = oracle_lib.get("reference") if oracle_lib.have_reference() else oracle_lib.get("port")
X, y = ref.generate_trunk(9000, 20, 6)
Xq = np.round(X * 8) / 8
ctx = sofg.Context(0)
def terms(f, i):
    return list(zip(f.feat[f.term_off[i]:f.term_off[i+1]].tolist(), f.weight[f.term_off[i]:f.term_off[i+1]].tolist()))
def walk(a, b, i, j, depth, path):
    if (a.left[i] < 0) != (b.left[j] < 0) or a.thr[i].tobytes() != b.thr[j].tobytes() or terms(a, i) != terms(b, j) or a.pred[i] != b.pred[j]:
        return (depth, path, repr(a.thr[i]), terms(a, i)[:4], repr(b.thr[j]), terms(b, j)[:4])
    if a.left[i] < 0: return None
    return walk(a, b, a.left[i], b.left[j], depth + 1, path + "L") or walk(a, b, a.right[i], b.right[j], depth + 1, path + "R")
for rep in range(4):
  for mode, be in (("exact", None), ("dynamic", 5000)):
    for name, data in (("X", X), ("Xq", Xq)):
        gc, oc = _cfg(n_trees=3, mode=mode, breakeven=be, seed=21)
        o = ref.train_forest(data, y, 2, oc)
        if True:
            ctx.upload(data, y, 2)
            g = ctx.train_forest(gc)
            gg = oracle_lib.FlatForest(g.tree_off, g.left, g.right, g.pred, g.thr, g.term_off, g.feat, g.weight)
            bad = [(t, walk(gg.tree(t), o.tree(t), 0, 0, 0, "")) for t in range(3) if not gg.tree_equal(o, t)]
            if bad: print(mode, name, rep, bad, flush=True)
print("done")
