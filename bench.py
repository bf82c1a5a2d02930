#!/usr/bin/env python
"""Throughput benchmark: trees/s to purity at 1M x 4096 (BASELINE.json), per B200 and aggregate.

One step = one pass of the hot path over one batch: training --trees trees (default 100 per GPU,
BASELINE config 3: synthetic 1M x 4096, 2-class, trained to purity, dynamic split switch with a
fixed recorded breakeven) through the level-wise frontier scheduler and the sm_100a kernels.
Multi-GPU (torchrun): trees are sharded tree-wise across ranks (weak scaling, no collective on
the data path); rank r trains its own slice of the forest each step.

value  device-timed trees/s over all ranks (CUDA events on the trainer's stream, max over ranks)
e2e    the same through the C ABI with host buffers: every step uploads the 16.4 GB table from
       page-locked memory (sofg_upload_dataset), trains, and reads the forest back; a second context
       on the same GPU holds a second resident table so step s+1's upload overlaps step s's training
       (--e2e-serial: upload, then train); each context trains a contiguous half of the tree
       ranges. Per-step wall times in e2e.step_ms (the first step pays the unhidden upload).
roofline  the dominant kernel, k_row_sweep (projection sweep): algorithmic bytes per launch (table
       rows streamed + projected rows written + term lists read) over its CUDA-event time, against
       MEASURED_PEAKS.json's HBM copy bandwidth, measured in one extra untimed profile step; traffic =
       DRAM bytes per launch from the committed ncu launch list (profiles/). Also the SURVEY 8(d)
       sector-model rate of the whole split finder.
cpu_baseline  the reference itself (oracle/_ref, compiled from the reference headers) training
       trees of the same forest on this host's cores; those trees are also compared bit-for-bit
       with the GPU's.

`--impl reference` times the reference's CPU learner alone (all host threads).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "trees/sec to purity at 1M x 4096 (2-class synthetic trunk, dynamic split switch)"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--samples", "--n", dest="n", type=int, default=1_000_000)
    p.add_argument("--features", "--d", dest="d", type=int, default=4096)
    p.add_argument("--trees", type=int, default=100, help="trees per GPU per step")
    p.add_argument("--breakeven", type=int, default=512,
                   help="dynamic-switch threshold; 512 = B200 calibration (DESIGN.md 3, calibrate.py)")
    p.add_argument("--mode", default="dynamic", choices=["dynamic", "exact", "histogram"])
    p.add_argument("--seed", type=int, default=7)
    p.add_argument("--e2e-steps", type=int, default=8)
    p.add_argument("--e2e-serial", action="store_true", help="e2e without the second-context input pipeline")
    p.add_argument("--cpu-trees", type=int, default=0, help="CPU baseline sample (0 = one per core)")
    p.add_argument("--holdout", type=int, default=20000, help="hold-out rows for the accuracy check")
    p.add_argument("--classes", type=int, default=2, help="trunk-model classes (BASELINE config 5: 4)")
    p.add_argument("--density", type=float, default=0.0,
                   help="projection cell density (0 = the reference default; config 5 'dense' > 0)")
    p.add_argument("--workers", type=int, default=0,
                   help="host threads of the trainer (0 = this rank's share of the host's cores)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-profile", action="store_true", help="skip the untimed per-kernel profile step")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        def run():
            q = "clocks.sm,clocks.max.sm,clocks_event_reasons.active"
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    sm, mx, reasons = [x.strip() for x in out.split(",")]
                    self.samples.append((float(sm), float(mx), int(reasons, 16)))
                except Exception:
                    pass
                self._stop.wait(0.2)

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        names = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
                 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
                 0x100: "display_clock_setting"}
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        reasons = 0
        for s in self.samples:
            reasons |= s[2]
        return {"sm_mhz": statistics.median(s[0] for s in self.samples),
                "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": [v for k, v in names.items() if reasons & k and k != 0x1],
                "samples": len(self.samples)}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def step_profile_key(args):
    return {"n": args.n, "d": args.d, "trees": args.trees, "mode": args.mode, "breakeven": args.breakeven,
            "classes": args.classes, "density": args.density}


def committed_step_profile(args):
    """ncu launch list of ONE training step of exactly this workload (tools/step_profile.py under
    ncu, summarised by tools/launch_summary.py into profiles/r*_step_dram*.json). None when no
    committed profile matches the configuration."""
    import glob

    key = step_profile_key(args)
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_step_dram*.json")), reverse=True):
        try:
            with open(path) as fh:
                d = json.load(fh)
        except Exception:
            continue
        if d.get("config") == key:
            return d, os.path.basename(path)
    return None, None


def roofline_block(st, args):
    """Dominant kernel, the projection sweep (k_row_sweep / k_row_sweep_pipe): algorithmic bytes
    (table rows streamed + projected rows written + term lists read, engine accounting) per launch
    over its CUDA-event time per launch. `traffic` = ncu DRAM bytes per sweep launch of the same
    workload (committed step profile), null when none matches. The split finder's fraction is DRAM
    bytes actually moved by all wave kernels of a step (same profile) over their CUDA-event time."""
    peak, peak_kind = measured_peak()
    kern = st.get("kernels", {})
    rs = kern.get("row_sweep", {"ms": 0.0, "launches": 0})
    launches = max(1, int(st["sweep_waves"]))
    avg_ms = rs["ms"] / launches if rs["launches"] else 0.0
    alg = st["sweep_alg_bytes"] / launches
    achieved = alg / (avg_ms / 1e3) / 1e9 if avg_ms > 0 else 0.0
    prof, src = committed_step_profile(args)
    traffic = None
    split = {"ms_per_step": round(st["ms_waves_total"], 2)}
    if prof:
        ks = prof["kernels"]
        sw = [v for k, v in ks.items() if k.startswith("k_row_sweep")]
        if sw:
            traffic = sum(v["dram_bytes"] for v in sw) / sum(v["launches"] for v in sw)
        dram = prof["total_dram_bytes"]
        split.update({"dram_bytes_per_step": dram,
                      "dram_GBps": round(dram / (st["ms_waves_total"] / 1e3) / 1e9, 1),
                      "dram_frac": round(dram / (st["ms_waves_total"] / 1e3) / 1e9 / peak, 4),
                      "dram_source": src,
                      "note": "DRAM bytes actually moved by every wave kernel of one step (ncu, same workload) "
                              "over the waves' CUDA-event time this run"})
    sector = st["hist_sector_bytes"] + st["exact_sector_bytes"]
    strict = st["hist_strict_bytes"] + st["exact_strict_bytes"]
    split_ms = st["ms_waves_total"]
    if split_ms:
        split["secondary_sector_model"] = {
            "GBps": round(sector / (split_ms / 1e3) / 1e9, 1),
            "frac": round(sector / (split_ms / 1e3) / 1e9 / peak, 4),
            "strict_GBps": round(strict / (split_ms / 1e3) / 1e9, 1),
            "note": "SURVEY 8(d) sector model: bytes a per-node GATHER implementation would move (32 B per "
                    "gathered value), not bytes this implementation moves"}
    return {"bound": "hbm", "kernel": "projection sweep (k_row_sweep_pipe / k_row_sweep): sample-major sweep of the row-major table",
            "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4),
            "peak_kind": peak_kind, "traffic": traffic, "traffic_source": src,
            "algorithmic_bytes_per_launch": alg, "avg_launch_ms": round(avg_ms, 3), "launches": launches,
            "algorithmic_bytes_definition": "XR rows streamed (n*ldr*4) + V written (sum n_i*Rp*4) + "
                                            "augmented term lists read, per sweep launch",
            "split_finder": split,
            "phase_ms": {k: round(st[k], 2) for k in ("ms_sample", "ms_hist_rng", "ms_hist_count", "ms_exact",
                                                      "ms_partition", "ms_waves_total", "ms_train_total")},
            "kernel_ms": kern, "profile_step": "one extra untimed step, one tree group, CUDA events per launch site"}


def cpu_reference_sample(X, y, n_trees, args, threads, predict_rows=None):
    """Reference learner (oracle/_ref) on this host: `n_trees` trees of the bench forest (timed);
    optionally the reference's own predict over `predict_rows` (untimed)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib

    orc = oracle_lib.get("reference") if oracle_lib.have_reference() else oracle_lib.get("port")
    k = int(getattr(args, "classes", 2))
    ds = orc.dataset(X, y, k)
    cfg = oracle_lib.make_config(n_trees=n_trees, mode=args.mode, breakeven=args.breakeven, seed=args.seed,
                                 n_workers=threads, cell_density=float(getattr(args, "density", 0.0)))
    timing = {}
    pred = None
    if predict_rows is None:
        forest = orc.train_forest_ds(ds, cfg, timing=timing)
    else:  # the reference's predict on the trained handle, outside the timed call
        forest, (pred, _) = orc.train_forest_ds(ds, cfg, predict_rows=predict_rows, d=X.shape[0], k=k,
                                                timing=timing)
    orc.dataset_free(ds)
    return forest, timing["train_s"], orc.kind, pred


def cpu_reference_trees(X, y, ids, n_trees_cfg, args, threads):
    """Reference learner (oracle/_ref) on this host: trees `ids` of the bench forest, each through
    the reference's train_tree on its derived stream (tree t: derive_seed(seed, t + 1); bootstrap
    derive_seed(ts, 0), root derive_seed(ts, 1), forest.hpp:153-154,305 — exactly the per-tree work
    train_forest's workers do, forest.hpp:302-306), on `threads` concurrent host threads. Timed:
    the trees only (the dataset conversion is outside)."""
    from concurrent.futures import ThreadPoolExecutor

    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib

    orc = oracle_lib.get("reference") if oracle_lib.have_reference() else oracle_lib.get("port")
    k = int(getattr(args, "classes", 2))
    n = X.shape[1]
    ds = orc.dataset(X, y, k)
    cfg = oracle_lib.make_config(n_trees=n_trees_cfg, mode=args.mode, breakeven=args.breakeven, seed=args.seed,
                                 n_workers=1, cell_density=float(getattr(args, "density", 0.0)))

    def one(t):
        ts = orc.derive_seed(args.seed, t + 1)
        boot = orc.bootstrap(n, 0.632, orc.derive_seed(ts, 0))
        return orc.train_tree_ds(ds, boot, cfg, orc.derive_seed(ts, 1))

    try:
        t0 = time.perf_counter()
        with ThreadPoolExecutor(max(1, min(threads, len(ids)))) as ex:
            trees = list(ex.map(one, ids))
        dt = time.perf_counter() - t0
    finally:
        orc.dataset_free(ds)
    return trees, dt, orc.kind


def physical_cores():
    try:
        import psutil

        return psutil.cpu_count(logical=False)
    except Exception:
        return None


def host_trunk(n, d, seed=1):
    """Trunk-model table on the host for the reference arm (multi-threaded numpy)."""
    from concurrent.futures import ThreadPoolExecutor

    X = np.empty((d, n), np.float32)
    mu = (1.0 / np.sqrt(np.arange(1, d + 1))).astype(np.float32)
    sign = np.where(np.arange(n) % 2 == 0, 1.0, -1.0).astype(np.float32)

    def fill(f0):
        rng = np.random.default_rng([seed, f0])
        for f in range(f0, min(d, f0 + 64)):
            X[f] = rng.standard_normal(n, dtype=np.float32) + sign * mu[f]

    with ThreadPoolExecutor(os.cpu_count() or 8) as ex:
        list(ex.map(fill, range(0, d, 64)))
    return X, (np.arange(n) % 2).astype(np.int32)


def run_reference(args, rank, world):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    X, y = host_trunk(args.n, args.d)
    n_trees = args.cpu_trees or threads
    steps = max(1, min(args.steps, 2))
    times = []
    for _ in range(steps):
        _, dt, kind, _ = cpu_reference_sample(X, y, n_trees, args, threads)
        times.append(dt)
    v = n_trees / statistics.median(times)
    line = {"metric": METRIC, "value": v, "unit": "trees/s", "n_gpus": 0, "steps": steps,
            "steps_requested": args.steps, "warmup": 0, "ms_per_step": 1000 * statistics.median(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32/f64",
            "data": "synthetic trunk model (numpy, host)", "impl": "reference",
            "config": {"workload": f"synthetic {args.n}x{args.d} {args.classes}-class, trees to purity"
                                   + (" (BASELINE config 3)" if (args.n, args.d) == (1_000_000, 4096) else ""),
                       "n_samples": args.n, "n_features": args.d, "trees_per_step": n_trees,
                       "breakeven": args.breakeven, "mode": args.mode, "seed": args.seed},
            "cpu_baseline": {"value": v, "unit": "trees/s", "cores": threads, "physical_cores": physical_cores(), "kind": kind,
                             "sample": f"{n_trees} full trees of the {args.n} x {args.d} forest on {threads} threads "
                                       f"per step; {steps} step(s), no warm-up (each step ~{times[0]:.0f} s)"},
            "e2e": {"value": v, "unit": "trees/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank, world, local = dist_env()
    dist = None
    if world > 1:
        import torch.distributed as dist

        # SOFG_BENCH_BACKEND / SOFG_BENCH_DEVICE: test hooks to run several ranks on one GPU
        backend = os.environ.get("SOFG_BENCH_BACKEND") or ("nccl" if args.impl == "ours" else "gloo")
        dist.init_process_group(backend)
    if args.impl == "reference":
        run_reference(args, rank, world)
        if dist:
            dist.barrier()
            dist.destroy_process_group()
        return

    import torch

    import paper_2603_00326_b200 as sofg

    if os.environ.get("SOFG_BENCH_DEVICE"):
        local = int(os.environ["SOFG_BENCH_DEVICE"])
    torch.cuda.set_device(local)
    ctx = sofg.Context(local)
    t0 = time.perf_counter()
    ctx.generate_trunk(args.n, args.d, args.classes, seed=1)
    gen_s = time.perf_counter() - t0
    stream = torch.cuda.ExternalStream(ctx.stream_ptr(), device=torch.device("cuda", local))
    T = args.trees
    per_step = T * world
    total_trees = (args.warmup + args.steps + args.e2e_steps + 2) * per_step

    # host threads split between the ranks sharing this host (one rank per GPU)
    workers = args.workers or max(1, (os.cpu_count() or 1) // max(1, int(os.environ.get("LOCAL_WORLD_SIZE", world))))

    def cfg_for(step):
        b = step * per_step + rank * T
        return sofg.TrainConfig(n_trees=total_trees, mode=args.mode, breakeven=args.breakeven, seed=args.seed,
                                n_workers=workers, tree_begin=b, tree_end=b + T, cell_density=args.density)

    def barrier():
        if dist:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if not dist:
            return x
        dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- warm-up ---------------------------------------------------------------------------------
    for s in range(args.warmup):
        ctx.train_forest(cfg_for(s))
    # ---- timed region (no per-kernel events, no accounting kernels) ---------------------------
    ctx.set_stats(0)
    ctx.reset_stats()
    nodes = 0
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clocks:
        ev0.record(stream)
        for s in range(args.warmup, args.warmup + args.steps):
            f = ctx.train_forest(cfg_for(s))
            nodes += len(f.left)
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier()
    last = f  # the last timed step's forest: trees last_begin .. last_begin + T - 1
    last_begin = (args.warmup + args.steps - 1) * per_step + rank * T
    ms = ev0.elapsed_time(ev1)
    ms_max = max_over_ranks(ms)
    gpu_launches = int(ctx.stats()["kernel_launches"])
    value = world * T * args.steps / (ms_max / 1000.0)

    # ---- profile step (untimed): one more step with CUDA events per launch site, one tree group
    #      on one stream (so a kernel's event time is its own), and sector accounting ---------------
    roofline = None
    if not args.no_profile:
        ctx.set_stats(2)
        ctx.reset_stats()
        # the last timed step's range again: context 0's next call (the first e2e step) then continues
        # its range and finds its bootstrap samples drawn ahead, like every timed step
        ctx.train_forest(cfg_for(args.warmup + args.steps - 1))
        st = ctx.stats()
        ctx.set_stats(0)
        roofline = roofline_block(st, args)

    # ---- end to end through the C ABI with host buffers ---------------------------------------
    e2e = None
    if not args.no_e2e and args.e2e_steps > 0:
        import ctypes as C

        nbytes = args.n * args.d * 4
        hptr = ctx.L.sofg_host_alloc(nbytes)
        if not hptr:
            raise RuntimeError("page-locked allocation failed")
        Xh = np.ctypeslib.as_array((C.c_float * (args.n * args.d)).from_address(hptr)).reshape(args.d, args.n)
        yh = np.zeros(args.n, np.int32)
        ctx.download(Xh, yh)
        # Input pipeline: a second context on the same GPU holds a second resident table, so step
        # s + 1's table upload (page-locked source, the context's own stream) runs while step s
        # trains; every step still uploads its whole table and reads its forest back inside the
        # timed region. Falls back to upload-then-train when the second table does not fit.
        ctxs = [ctx]
        if not args.e2e_serial:
            try:
                c2 = sofg.Context(local)
                c2.upload_ptr(hptr, yh, args.n, args.d, args.classes)
                # buffers (untimed); the range before context 1's first e2e range (see below)
                c2.train_forest(cfg_for(args.warmup + args.steps + (args.e2e_steps + 1) // 2 - 1))
                ctxs.append(c2)
            except Exception as exc:  # noqa: BLE001 - any allocation failure: serial pipeline
                print(f"e2e: second context unavailable ({exc}); serial upload + train", file=sys.stderr)
        barrier()
        d2h = 0
        first = args.warmup + args.steps
        torch.cuda.synchronize()
        ts = time.perf_counter()
        step_wall = [ts]
        ctxs[0].upload_ptr(hptr, yh, args.n, args.d, args.classes)
        # With two contexts, each trains a contiguous half of the e2e tree ranges (context 0 the first
        # half, context 1 the second, alternating steps), so a context's next call continues its
        # previous range and finds that range's bootstrap samples already drawn in the idle time
        # of its last call (api.cpp BootAhead). Same trees as ranges first .. first + steps - 1.
        half = (args.e2e_steps + len(ctxs) - 1) // len(ctxs)
        for j in range(args.e2e_steps):
            cur = ctxs[j % len(ctxs)]
            if len(ctxs) > 1 and j + 1 < args.e2e_steps:  # next step's table, in flight during this step
                ctxs[(j + 1) % len(ctxs)].upload_ptr(hptr, yh, args.n, args.d, args.classes)
            rng = first + (j % len(ctxs)) * half + j // len(ctxs)
            f = cur.train_forest(cfg_for(rng))
            step_wall.append(time.perf_counter())
            d2h = sum(a.nbytes for a in (f.tree_off, f.left, f.right, f.pred, f.thr, f.term_off, f.feat, f.weight))
            if len(ctxs) == 1 and j + 1 < args.e2e_steps:
                cur.upload_ptr(hptr, yh, args.n, args.d, args.classes)
        torch.cuda.synchronize()
        e_s = max_over_ranks(time.perf_counter() - ts)
        e2e = {"value": world * T * args.e2e_steps / e_s, "unit": "trees/s", "h2d_bytes_per_step": nbytes + 4 * args.n,
               "d2h_bytes_per_step": d2h, "steps": args.e2e_steps,
               "step_ms": [round(1e3 * (b - a), 1) for a, b in zip(step_wall, step_wall[1:])],
               "timing": "host wall clock, cuda-synchronized, max over ranks",
               "pipeline": ("two contexts: step s+1's table upload overlaps step s's training"
                            if len(ctxs) > 1 else "serial: upload, then train")}
        for c2 in ctxs[1:]:
            c2.close()
    else:
        Xh = None

    # ---- CPU baseline (rank 0, N = 1) -----------------------------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        n_cpu = min(args.cpu_trees or threads, T)
        if Xh is None:
            Xh = np.zeros((args.d, args.n), np.float32)
            yh = np.zeros(args.n, np.int32)
            ctx.download(Xh, yh)
        # hold-out rows: a second draw of the same trunk model (device generator, seed 2)
        hctx = sofg.Context(0)
        Xt = np.zeros((args.d, args.holdout), np.float32)
        yt = np.zeros(args.holdout, np.int32)
        hctx.generate_trunk(args.holdout, args.d, args.classes, seed=2)
        hctx.download(Xt, yt)
        hctx.close()
        rows = np.ascontiguousarray(Xt.T)
        ids = list(range(last_begin, last_begin + n_cpu))
        trees, dt, kind = cpu_reference_trees(Xh, yh, ids, total_trees, args, threads)
        import oracle_lib

        ff = oracle_lib.FlatForest(last.tree_off, last.left, last.right, last.pred, last.thr, last.term_off,
                                   last.feat, last.weight)
        same = sum(ff.tree_equal(tr, t, 0) for t, tr in enumerate(trees))
        cpu_forest = oracle_lib.FlatForest.concat(trees)
        orc = oracle_lib.get("reference") if oracle_lib.have_reference() else oracle_lib.get("port")
        cpu_lab, _ = orc.predict_flat(cpu_forest, rows, args.d, args.classes)
        hf = ff.head(n_cpu)
        head = type(last)(hf.tree_off, hf.left, hf.right, hf.pred, hf.thr, hf.term_off, hf.feat, hf.weight,
                          last.breakeven, last.class_count, last.n_features)
        gpu_lab_head, _ = ctx.predict(head, rows)
        gpu_lab_all, _ = ctx.predict(last, rows)
        cpu = {"value": n_cpu / dt, "unit": "trees/s", "cores": threads, "physical_cores": physical_cores(),
               "kind": kind,
               "sample": f"trees {ids[0]}..{ids[-1]} of the forest (the first {n_cpu} trees of the LAST TIMED step; "
                         f"full {args.n} x {args.d} trees, each the reference's train_tree on its derived stream = "
                         f"train_forest's per-tree work, forest.hpp:302-306), {n_cpu} concurrent threads, {dt:.1f} s",
               "bitexact_trees": f"{same}/{n_cpu}",
               "holdout": {"rows": int(args.holdout), "data": "trunk model (device generator), seed 2",
                           f"cpu_accuracy_{n_cpu}_trees": round(float((cpu_lab == yt).mean()), 5),
                           f"gpu_accuracy_{n_cpu}_trees": round(float((gpu_lab_head == yt).mean()), 5),
                           "identical_labels": bool(np.array_equal(cpu_lab, gpu_lab_head)),
                           f"gpu_accuracy_{T}_trees": round(float((gpu_lab_all == yt).mean()), 5)}}

    line = {"metric": METRIC, "value": value, "unit": "trees/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32 values / f64 accumulate+gain",
            "data": "synthetic trunk model generated in HBM (counter-based RNG), inputs > L2",
            "config": {"workload": f"synthetic {args.n}x{args.d} {args.classes}-class, {T} trees per GPU to purity"
                                   + (" (BASELINE config 3)" if (args.n, args.d) == (1_000_000, 4096) else ""),
                       "n_samples": args.n, "n_features": args.d, "trees_per_gpu_per_step": T,
                       "mode": args.mode, "breakeven": args.breakeven, "bin_count": 256, "seed": args.seed,
                       "classes": args.classes, "cell_density": args.density or "reference default",
                       "parallelism": f"tree-sharded x{world}", "host_threads_per_rank": workers,
                       "l2": f"inputs {args.n * args.d * 4 / 1e9:.2f} GB table (+ row-major copy) vs 126 MB L2",
                       "nodes_per_step": nodes / args.steps, "datagen_s": round(gen_s, 2)},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": gpu_launches,
            "clocks": clocks.summary()}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if Xh is not None and not args.no_e2e and args.e2e_steps > 0:
        ctx.L.sofg_host_free(hptr)
    ctx.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
