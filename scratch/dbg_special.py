import sys; sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import numpy as np, oracle_lib
import paper_2603_00326_b200 as sofg
from test_gpu_parity import _cfg
ref = oracle_lib.get("reference") if oracle_lib.have_reference() else oracle_lib.get("port")
X, y = ref.generate_trunk(3000, 24, 8)
X = X.copy(); rng = np.random.default_rng(8); m = rng.random(X.shape)
X[m < 0.05] = 0.0; X[(m >= 0.05) & (m < 0.1)] = -0.0; X[(m >= 0.1) & (m < 0.15)] *= np.float32(1e-40); X[3, (m[3] > 0.9)] = np.float32(1e-45)
X = X.astype(np.float32)
ctx = sofg.Context(0); ctx.upload(X, y, 2)
gc, oc = _cfg(n_trees=3, mode="dynamic", breakeven=300, seed=17)
g = ctx.train_forest(gc); o = ref.train_forest(X, y, 2, oc)
gg = oracle_lib.FlatForest(g.tree_off, g.left, g.right, g.pred, g.thr, g.term_off, g.feat, g.weight)
def terms(f, i):
    return list(zip(f.feat[f.term_off[i]:f.term_off[i+1]].tolist(), f.weight[f.term_off[i]:f.term_off[i+1]].tolist()))
def walk(a, b, i, j, depth, path):
    if a.left[i] < 0 or b.left[j] < 0 or a.thr[i].tobytes() != b.thr[j].tobytes() or terms(a, i) != terms(b, j):
        if (a.left[i] < 0) != (b.left[j] < 0) or a.thr[i].tobytes() != b.thr[j].tobytes() or terms(a, i) != terms(b, j) or a.pred[i] != b.pred[j]:
            print(" diff at depth", depth, "path", path, "gpu leaf" if a.left[i] < 0 else "gpu split", repr(a.thr[i]), terms(a, i)[:8], a.pred[i],
                  "| ref", "leaf" if b.left[j] < 0 else "split", repr(b.thr[j]), terms(b, j)[:8], b.pred[j])
            return True
        return False
    return walk(a, b, a.left[i], b.left[j], depth + 1, path + "L") or walk(a, b, a.right[i], b.right[j], depth + 1, path + "R")
for t in range(3):
    a, b = gg.tree(t), o.tree(t)
    print("tree", t); walk(a, b, 0, 0, 0, "")

# ---- reconstruct tree 2, path LLRR, and compare the node split
t = 2; path = "LLRR"
b = o.tree(t)
ts = ref.derive_seed(17, t + 1)
act = sofg.bootstrap_sample(3000, 0.632, ref.derive_seed(ts, 0))
s = ref.derive_seed(ts, 1)
node = 0
for ch in path:
    fa = b.feat[b.term_off[node]:b.term_off[node+1]]; wa = b.weight[b.term_off[node]:b.term_off[node+1]]
    v = ref.apply_projection(X, fa, wa, act)
    left = v <= b.thr[node]
    if ch == "L":
        act = act[left]; node = b.left[node]; s = ref.derive_seed(s, 1)
    else:
        act = act[~left]; node = b.right[node]; s = ref.derive_seed(s, 2)
print("node n", len(act), "labels", np.bincount(y[act], minlength=2))
R, e, dens = ref.projection_config(24)
rp, feat, w, used = ref.sample_projection(24, R, dens, s, 0)
z = int(rp[-1]); feat = feat[:z]; w = w[:z]
meth = "histogram" if len(act) > 300 else "exact"
os_, oused, ovals = ref.find_node_split(X, y, 2, act, rp, feat, w, meth, 256, s, used)
gs = ctx.find_node_split(act, rp, feat, w, meth, 256, s, used)
print("method", meth)
print("ref", os_.found, os_.projection_index, repr(np.float32(os_.threshold)), os_.n_left, repr(os_.gain))
print("gpu", gs.found, gs.projection_index, repr(np.float32(gs.threshold)), gs.n_left, repr(gs.gain))
for r in sorted({int(os_.projection_index), int(gs.projection_index)}):
    fr = feat[rp[r]:rp[r+1]]; wr = w[rp[r]:rp[r+1]]
    vals = ref.apply_projection(X, fr, wr, act)
    o1 = ref.find_node_split(X, y, 2, act, np.array([0, len(fr)], np.uint32), fr, wr, meth, 256, s, used)[0]
    g1 = ctx.find_node_split(act, np.array([0, len(fr)], np.uint32), fr, wr, meth, 256, s, used)
    print(" row", r, list(zip(fr.tolist(), wr.tolist())), "ref single-row", o1.found, repr(np.float32(o1.threshold)), o1.n_left, repr(o1.gain), "| gpu", g1.found, repr(np.float32(g1.threshold)), g1.n_left, repr(g1.gain))
    sv = np.sort(vals); print("   smallest |v|:", sorted(vals[np.abs(vals) < 1e-30].tolist())[:20])
