"""Per-wave host / GPU timeline of three 100-tree steps at 1M x 4096 (stderr):
  SOFG_LEVEL_LOG=1 [WORKERS=<host threads>] python tools/level_log.py
prints one line per wave (prep, submit, speculative draws, GPU wait, collect, child creation; the
log synchronises each wave, so per-step times are slightly higher than in the bench) and the
host phase totals (ctx.stats())."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import paper_2603_00326_b200 as sofg
with sofg.Context(0) as ctx:
    ctx.generate_trunk(1_000_000, 4096, 2, seed=1)
    cfg = sofg.TrainConfig(n_trees=100, mode="dynamic", breakeven=512, seed=7, n_workers=int(os.environ.get("WORKERS", "0")))
    for i in range(3):
        t = time.perf_counter(); f = ctx.train_forest(cfg); print("STEP", i, (time.perf_counter()-t)*1e3, file=sys.stderr, flush=True)
    st = ctx.stats()
    print({k: v for k, v in st.items() if k != "kernels"}, file=sys.stderr)
