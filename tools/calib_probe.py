"""Prints the GPU crossover calibration (sofg_calibrate) on the bench table (1M x 4096 trunk)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_00326_b200 as sofg
from paper_2603_00326_b200.model_io import CalibrationOptions

n, d = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (1_000_000, 4096)
with sofg.Context(0) as ctx:
    ctx.generate_trunk(n, d, 2, 1)
    for budget in (0.1, 1.0):
        t = time.time()
        cal = ctx.calibrate(sofg.TrainConfig(calibration=CalibrationOptions(budget_seconds=budget)))
        print(f"budget {budget}: breakeven {cal.breakeven} fallback {cal.fallback} elapsed {cal.elapsed_seconds:.3f}s "
              f"wall {time.time() - t:.2f}s")
        for s in cal.samples:
            print(f"   n={s[0]:6d} exact {s[1] * 1e6:9.3f} us  hist {s[2] * 1e6:9.3f} us")
