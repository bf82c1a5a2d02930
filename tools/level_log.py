import sys, time, os
sys.path.insert(0, '.')
import paper_2603_00326_b200 as sofg
ctx = sofg.Context(0)
ctx.generate_trunk(1_000_000, 4096, 2, seed=1)
for it in range(3):

    ctx.set_stats(1 if it < 2 else 0); ctx.reset_stats()
    cfg = sofg.TrainConfig(n_trees=1000, mode="dynamic", breakeven=512, seed=7, tree_begin=100 * it, tree_end=100 * it + 100)
    t = time.perf_counter(); f = ctx.train_forest(cfg); t = time.perf_counter() - t
    st = ctx.stats()
    print(it, round(t * 1e3), {k: round(v, 1) for k, v in st.items() if k.startswith("ms_")}, flush=True)
