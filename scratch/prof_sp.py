import sys; sys.path.insert(0, '.')
import paper_2603_00326_b200 as sofg
ctx = sofg.Context(0)
ctx.generate_trunk(250000, 16384, 4, seed=1)
cfg = sofg.TrainConfig(n_trees=8, mode="dynamic", breakeven=512, seed=7, cell_density=0.001)
f = ctx.train_forest(cfg); print("nodes", len(f.left))
