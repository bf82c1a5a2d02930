import sys, time
sys.path.insert(0, '.')
import paper_2603_00326_b200 as sofg
trees = int(sys.argv[1]) if len(sys.argv) > 1 else 4
ctx = sofg.Context(0)
ctx.generate_trunk(1_000_000, 4096, 2, seed=1)
cfg = sofg.TrainConfig(n_trees=trees, mode="dynamic", breakeven=512, seed=7, n_workers=0)
t = time.perf_counter(); f = ctx.train_forest(cfg); print("trees", f.n_trees, "nodes", len(f.left), "s", time.perf_counter() - t)
