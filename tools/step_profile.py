"""One training step of the bench workload (generate the table in HBM, train one batch of trees),
for an ncu launch list of exactly one step: run under
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file L \
      python tools/step_profile.py [--n N --d D --trees T --breakeven B --classes K --density X]
then `python tools/launch_summary.py L profiles/<round>_step_dram.json --config '<json>'` (the
table generator and its row-major transpose are data setup and are left out of the step)."""
import argparse, os, sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_00326_b200 as sofg

p = argparse.ArgumentParser()
p.add_argument("--n", type=int, default=1_000_000)
p.add_argument("--d", type=int, default=4096)
p.add_argument("--trees", type=int, default=100)
p.add_argument("--breakeven", type=int, default=512)
p.add_argument("--mode", default="dynamic")
p.add_argument("--classes", type=int, default=2)
p.add_argument("--density", type=float, default=0.0)
p.add_argument("--seed", type=int, default=7)
p.add_argument("--stats", action="store_true", help="print CUDA-event time per launch site (3 steps)")
a = p.parse_args()
with sofg.Context(0) as ctx:
    ctx.generate_trunk(a.n, a.d, a.classes, seed=1)
    cfg = sofg.TrainConfig(n_trees=a.trees, mode=a.mode, breakeven=a.breakeven, seed=a.seed,
                           cell_density=a.density, n_workers=0)
    f = ctx.train_forest(cfg)
    print("trees", f.n_trees, "nodes", len(f.left))
    if a.stats:
        import time
        ctx.set_stats(1)
        ctx.reset_stats()
        t = time.perf_counter()
        for _ in range(2):
            ctx.train_forest(cfg)
        t = (time.perf_counter() - t) / 2
        st = ctx.stats()
        print(f"step {t * 1e3:.1f} ms (stats on)", {k: round(v["ms"] / 2, 1) for k, v in st["kernels"].items()})
