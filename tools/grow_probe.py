"""Diagnostic: buffer growth events (SOFG_GROW_LOG=1 prints them on stderr) per training call."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_00326_b200 as sofg
ctx = sofg.Context(0)
ctx.generate_trunk(1_000_000, 4096, 2, seed=1)
for s in range(7):
    print(f"[call {s}]", file=sys.stderr, flush=True)
    ctx.train_forest(sofg.TrainConfig(n_trees=100000, mode="dynamic", breakeven=512, seed=7,
                                      tree_begin=100 * s, tree_end=100 * s + 100))
