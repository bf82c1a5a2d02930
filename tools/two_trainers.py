"""Experiment: two trainers (contexts, host pools) on one GPU, each a 100-tree batch, concurrently."""
import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_00326_b200 as sofg

n, d = 1_000_000, 4096
W = int(sys.argv[1]) if len(sys.argv) > 1 else 8
A, B = sofg.Context(0), sofg.Context(0)
A.generate_trunk(n, d, 2, seed=1)
B.generate_trunk(n, d, 2, seed=1)
cfg = lambda b, w: sofg.TrainConfig(n_trees=100000, mode="dynamic", breakeven=512, seed=7, tree_begin=b, tree_end=b + 100,
                                    n_workers=w)
for c in (A, B):
    c.train_forest(cfg(0, W)); c.train_forest(cfg(100, W))
torch.cuda.synchronize()
t = time.perf_counter()
for s in range(3):
    A.train_forest(cfg(1000 + 100 * s, 16))
print("sequential, 16 threads: %.1f trees/s" % (300 / (time.perf_counter() - t)))
res = {}
def run(c, base):
    for s in range(3):
        c.train_forest(cfg(base + 100 * s, W))
t = time.perf_counter()
th = [threading.Thread(target=run, args=(A, 2000)), threading.Thread(target=run, args=(B, 3000))]
[x.start() for x in th]; [x.join() for x in th]
print("two concurrent trainers, %d threads each: %.1f trees/s" % (W, 600 / (time.perf_counter() - t)))
