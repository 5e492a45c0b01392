#!/usr/bin/env python
"""bench.py -- fp64 Q~v + Q~^T v throughput (beads/s) of the B200 operators.

One step = one Q~v over every bead of the batch plus one Q~^T g over every
complement coordinate (BASELINE.json metric), on BASELINE config 2 by default
(1000 triaxial-ellipsoid-shell bodies x 4096 beads, fp64, synthetic seeded
input).  Operator (~0.6 GB of chunk blobs) and vectors (~0.2 GB) are far
larger than the 126 MB L2, so no L2 flush is needed between steps.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

N > 1 runs under torchrun, one rank per GPU; bodies are independent so every
rank owns its own 1000-body shard (weak scaling, no data-path collective);
times are device-measured (CUDA events) and max-reduced over ranks.
--sharding strong instead splits ONE config-sized model across the ranks by
cumulative bead count (e.g. config 4's 20000 bodies over 8 GPUs).

--impl reference times the reference algorithm on the host CPU: the C oracle
(oracle/, a restatement of the pure-Python reference package that is 30-100x
faster than the Python original) with all host threads, same config/metric.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fp64 Q̃v+Q̃ᵀv beads/s (batched bodies) at 1/2/4/8 B200; % of HBM roofline"
UNIT = "beads/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=[2, 3, 4, 5])
    ap.add_argument("--scale", type=float, default=1.0, help="fraction of the config's bodies (tests)")
    ap.add_argument("--cpu-sample-s", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sharding", default="weak", choices=["weak", "strong"],
                    help="weak: every rank owns a full config-sized shard; strong: one config-sized "
                         "model split across the ranks by cumulative bead count (parallel.shard_bounds)")
    return ap.parse_args()


def workload(cfg: int, rank: int, scale: float, world: int = 1, strong: bool = False):
    from paper_1708_08427_b200.parallel import shard_of
    from paper_1708_08427_b200.workloads import CONFIGS, make_config

    if strong:  # one model for the whole job, this rank's contiguous shard of its bodies
        pos, off = make_config(cfg, seed=1000, scale=scale)
        pos, off, _ = shard_of(pos, off, rank, world)
    else:
        pos, off = make_config(cfg, seed=1000 + rank, scale=scale)
    name = CONFIGS[cfg]["workload"] if cfg in CONFIGS else "cfg4: 20000 ellipsoid bodies, n_j log-uniform [500, 50000]"
    k = CONFIGS.get(cfg, {}).get("k", 1)
    return pos, off, name, k


def config_dict(name, off, k, n_gpus, strong=False):
    n = np.diff(off)
    return {"workload": name, "bodies": int(len(n)), "beads": int(off[-1]),
            "beads_per_body": int(n[0]) if np.all(n == n[0]) else "mixed", "rhs_k": k,
            "l2": "operator + vectors >> 126 MB L2 (no flush needed)",
            "sharding": (f"strong: one model split by cumulative bead count over {n_gpus} ranks "
                         f"(bodies/beads above are rank 0's shard)") if strong else
                        f"weak: one independent shard per rank x{n_gpus}"}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self, dev: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,utilization.gpu")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(dev), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        rows = []
        for line in self.f.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        load = [r for r in rows if r[6] not in ("0", "[N/A]")] or rows
        sm = sorted(float(r[0]) for r in load)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in load for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": float(load[0][1]), "reasons": reasons,
                "samples": len(rows), "samples_under_load": len(load)}


def cpu_oracle_rate(pos, off, seconds: float, threads: int, steps=None, warmup=0):
    """Reference algorithm (C oracle) on the host: Q~v + Q~^T g per step over the given bodies."""
    from oracle.oracle import OracleBatch

    ob = OracleBatch(pos, off, threads=threads)
    N, m = int(off[-1]), len(off) - 1
    rng = np.random.default_rng(7)
    v = rng.normal(size=3 * N)
    g = rng.normal(size=3 * N - 6 * m)
    for _ in range(warmup):
        ob.apply("qtilde_v", v)
        ob.apply("qtilde_tv", g)
    n_steps, t0 = 0, time.perf_counter()
    while True:
        ob.apply("qtilde_v", v)
        ob.apply("qtilde_tv", g)
        n_steps += 1
        el = time.perf_counter() - t0
        if (steps is not None and n_steps >= steps) or (steps is None and el >= seconds):
            break
    return N * n_steps / el, n_steps, el


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    pos, off, name, k = workload(args.config, 0, args.scale)
    threads = len(os.sched_getaffinity(0))
    N = int(off[-1])
    # bound the run to a few minutes: sample bodies if the full batch is too slow
    from oracle.oracle import OracleBatch

    probe = min(len(off) - 1, 64)
    ob = OracleBatch(pos[:off[probe]], off[:probe + 1], threads=threads)
    t0 = time.perf_counter()
    rng = np.random.default_rng(0)
    ob.apply("qtilde_v", rng.normal(size=3 * int(off[probe])))
    per_bead = (time.perf_counter() - t0) * 2 / off[probe]
    budget = 120.0 / max(1, args.steps + args.warmup)
    nb = len(off) - 1
    if per_bead * N > budget:
        nb = max(1, int(nb * budget / (per_bead * N)))
    sub_off = off[:nb + 1]
    rate, steps, el = cpu_oracle_rate(pos[:sub_off[-1]], sub_off, 0.0, threads, steps=args.steps, warmup=args.warmup)
    sample = (f"{nb} of {len(off) - 1} bodies ({int(sub_off[-1])} beads) of the config; "
              f"{steps} steps of Q~v+Q~^T g in {el:.1f} s")
    line = {"impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": el / steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(name, off, k, args.gpus),
            "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
            "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import ctypes as C

    import torch

    import paper_1708_08427_b200 as rq
    from paper_1708_08427_b200 import _lib as L

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    strong = args.sharding == "strong"
    pos, off, name, k = workload(args.config, rank, args.scale, world, strong)
    N, m = int(off[-1]), len(off) - 1
    # beads processed per step by the whole job (strong: the sum of the shards)
    n_job = world * N
    if strong and dist:
        t = torch.tensor([N], device=dev, dtype=torch.int64)
        dist.all_reduce(t)
        n_job = int(t.item())
    model = rq.MultiBodyModel.from_arrays(pos, off)
    # load the library's kernels (lazy module loading) before the setup is timed
    from paper_1708_08427_b200.workloads import make_config

    wp, wo = make_config(2, seed=7, scale=0.002)
    wop = rq.MultiBodyOperator(rq.MultiBodyModel.from_arrays(wp, wo))
    for wk in (1, 32):
        wv = np.zeros((3 * int(wo[-1]), wk))
        wop.apply("qtilde_v", wv)
        wop.apply("qtilde_tv", np.zeros((3 * int(wo[-1]) - 6 * (len(wo) - 1), wk)))
    del wop
    # setup timed twice (the plan is rebuilt; the first build also pays one-time driver costs
    # on a fresh box, e.g. lazy kernel loading); the steady-state second build is reported
    setup_times = []
    for rep in range(2):
        if rep:
            del op
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        op = rq.MultiBodyOperator(model)
        torch.cuda.synchronize()
        setup_times.append(time.perf_counter() - t0)
    setup_s = setup_times[-1]
    info = op.plan.info()
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    v = torch.randn((3 * N, k) if k > 1 else (3 * N,), generator=gen, device=dev, dtype=torch.float64)
    g = torch.randn((3 * N - 6 * m, k) if k > 1 else (3 * N - 6 * m,), generator=gen, device=dev,
                    dtype=torch.float64)

    def step():
        op.apply("qtilde_v", v)
        op.apply("qtilde_tv", g)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clocks = Clocks(local)
    time.sleep(0.3)
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(args.steps):
        step()
    e1.record(s)
    torch.cuda.synchronize()
    ck = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    if dist:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    value = n_job / (ms * 1e-3)
    # per-step spread (min / median over >= 10 individually timed steps, as the
    # reference's own bench reports the min of 10); `value` stays the K-step average
    reps = []
    for _ in range(20):
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(s)
        step()
        a1.record(s)
        a1.synchronize()
        reps.append(a0.elapsed_time(a1))
    step_stats = {"min_ms": float(np.min(reps)), "median_ms": float(np.median(reps)), "repeats": len(reps)}

    # ---- kernel-level roofline: the chunk sweep (dominant kernel), timed alone
    lib = L.lib()
    h = op.plan.handle
    stream = C.c_void_p(s.cuda_stream)
    v2 = v.reshape(3 * N, -1)
    g2 = g.reshape(3 * N - 6 * m, -1)
    outs = {"qtilde_v": torch.empty((3 * N - 6 * m, k), device=dev, dtype=torch.float64),
            "qtilde_tv": torch.empty((3 * N, k), device=dev, dtype=torch.float64)}
    kern = {}
    mrhs = k >= info["mrhs_min_k"] and lib.rq_launches_per_apply(h, L.OP_QTILDE_V, k) < 2 * k
    for opn, code, x in (("qtilde_v", L.OP_QTILDE_V, v2), ("qtilde_tv", L.OP_QTILDE_TV, g2)):
        for phase, label in ((1, "chunks"), (2, "top")):
            reps = 50
            for _ in range(3):
                L.check(lib.rq_apply_ex(h, code, x.data_ptr(), outs[opn].data_ptr(), k, stream, phase))
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            for _ in range(reps):
                L.check(lib.rq_apply_ex(h, code, x.data_ptr(), outs[opn].data_ptr(), k, stream, phase))
            b.record(s)
            torch.cuda.synchronize()
            # ms per launch (the single-RHS path launches once per column)
            kern[(opn, label)] = a.elapsed_time(b) / reps / (1 if mrhs else k)
    per_step = 1 if mrhs else k  # launches of each phase per application
    chunk_ms = 0.5 * (kern[("qtilde_v", "chunks")] + kern[("qtilde_tv", "chunks")])
    info = op.plan.info()  # multi-RHS programs are built by the first k >= mrhs_min_k apply
    if mrhs:
        # tile-unit launch: the unit programs (entry headers + records) once per group of
        # 32 columns, every bead row and residue row of the k columns once, and the
        # tile-root exchange rows (written upward / read downward)
        ncg = (k + 31) // 32
        chunk_bytes = (info["mrhs_bytes"]["tiles"] * ncg + 8 * k * (3 * N + (3 * N - 6 * m))
                       + 8 * 6 * k * info["mrhs_units"]["tiles"])
        kname = "k_mrhs (column-parallel stack machine over tile units, lane = RHS column)"
    else:
        # algorithmic bytes per chunk launch: the chunk blobs (records + meta + perm)
        # plus one read and one write of every bead's 3 fp64 and residue coordinates
        chunk_bytes = info["blob_bytes"] + 8 * (3 * N + (3 * N - 6 * m))
        kname = "k_chunk (level-synchronous chunk sweep, TMA bulk-copied blobs)"
    achieved = chunk_bytes / (chunk_ms * 1e-3) / 1e9
    peak, peak_src = peaks()
    step_ms_kernels = sum(kern.values()) * per_step
    share = (kern[("qtilde_v", "chunks")] + kern[("qtilde_tv", "chunks")]) * per_step / step_ms_kernels
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "chunk_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            tj = json.load(f)
        # dram bytes per launch measured by ncu on the same config, scaled per bead
        if tj.get("config") == args.config and tj.get("beads"):
            traffic = tj["dram_bytes_per_launch"] * N / tj["beads"]

    # ---- config 3 also as ONE batched application of its 100 fresh vectors (SURVEY 8(d):
    # "report sequential and, separately, batched k=100"): the multi-RHS kernels
    batched = None
    if args.config == 3 and k == 1:
        kb = 100
        vb = torch.randn((3 * N, kb), generator=gen, device=dev, dtype=torch.float64)
        gb = torch.randn((3 * N - 6 * m, kb), generator=gen, device=dev, dtype=torch.float64)
        for _ in range(2):
            op.apply("qtilde_v", vb)
            op.apply("qtilde_tv", gb)
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(s)
        for _ in range(5):
            op.apply("qtilde_v", vb)
            op.apply("qtilde_tv", gb)
        a1.record(s)
        torch.cuda.synchronize()
        bms = a0.elapsed_time(a1) / 5
        batched = {"k": kb, "ms_per_step": bms, "value": N * kb / (bms * 1e-3), "unit": "bead-RHS/s",
                   "note": "Q~V + Q~^T G on (rows, 100) blocks: the 100 applications of config 3 batched"}
        del vb, gb

    # ---- Zf / Z^T u (config 4 names them): 48 algorithmic bytes per
    # bead (positions in + forces in / velocities out), device-resident inputs
    zops = {}
    fz = torch.randn(3 * N, generator=gen, device=dev, dtype=torch.float64)
    uz = torch.randn(6 * m, generator=gen, device=dev, dtype=torch.float64)
    for zname, zfn in (("zf", lambda: op.zf(fz)), ("ztu", lambda: op.ztu(uz))):
        for _ in range(3):
            zfn()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(s)
        for _ in range(20):
            zfn()
        a1.record(s)
        torch.cuda.synchronize()
        zms = a0.elapsed_time(a1) / 20
        zops[zname] = {"ms": zms, "beads_per_s": N / (zms * 1e-3), "achieved_gbs": 48 * N / (zms * 1e-3) / 1e9,
                       "frac": 48 * N / (zms * 1e-3) / 1e9 / peaks()[0]}

    # ---- end to end through the C ABI with HOST buffers (pinned), copies inside
    e2e = None
    if not args.no_e2e:
        hv = torch.empty(v2.shape, dtype=torch.float64, pin_memory=True)
        hg = torch.empty(g2.shape, dtype=torch.float64, pin_memory=True)
        hv.copy_(v2)
        hg.copy_(g2)
        ho1 = torch.empty((3 * N - 6 * m, k), dtype=torch.float64, pin_memory=True)
        ho2 = torch.empty((3 * N, k), dtype=torch.float64, pin_memory=True)
        e_steps = max(3, min(50, args.steps))
        for _ in range(2):
            L.check(lib.rq_apply_host(h, L.OP_QTILDE_V, hv.data_ptr(), ho1.data_ptr(), k))
            L.check(lib.rq_apply_host(h, L.OP_QTILDE_TV, hg.data_ptr(), ho2.data_ptr(), k))
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e_steps):
            L.check(lib.rq_apply_host(h, L.OP_QTILDE_V, hv.data_ptr(), ho1.data_ptr(), k))
            L.check(lib.rq_apply_host(h, L.OP_QTILDE_TV, hg.data_ptr(), ho2.data_ptr(), k))
        e2e_ms = (time.perf_counter() - t0) / e_steps * 1e3
        if dist:
            t = torch.tensor([e2e_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        nbytes_in = (hv.numel() + hg.numel()) * 8
        nbytes_out = (ho1.numel() + ho2.numel()) * 8
        e2e = {"value": n_job * k / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": nbytes_in,
               "d2h_bytes_per_step": nbytes_out, "ms_per_step": e2e_ms,
               "path": "rq_apply_host (C ABI, pinned host buffers, H2D+D2H inside the timed region)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = len(os.sched_getaffinity(0))
        nb = min(m, 200)
        rate, steps, el = cpu_oracle_rate(pos[:off[nb]], off[:nb + 1], args.cpu_sample_s, threads)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"first {nb} bodies ({int(off[nb])} beads) of the workload, {steps} steps "
                         f"of Q~v+Q~^T g in {el:.1f} s (C oracle, OpenMP over bodies)"}

    launches = args.steps * (lib.rq_launches_per_apply(h, L.OP_QTILDE_V, k) +
                             lib.rq_launches_per_apply(h, L.OP_QTILDE_TV, k))
    if rank == 0:
        line = {
            "metric": METRIC, "value": value * k, "unit": UNIT if k == 1 else "bead-RHS/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": args.sharding, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(name, off, k, world, strong),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": kname,
                         "bytes_per_launch": chunk_bytes, "launch_ms": chunk_ms, "peak_source": peak_src,
                         "share_of_step": share},
            "kernels_ms": {f"{a}:{b}": v_ for (a, b), v_ in kern.items()},
            "step_ms_single": step_stats,
            "z_ops": zops,
            "batched_k100": batched,
            "cpu_baseline": cpu, "e2e": e2e, "clocks": ck, "gpu_launches": int(launches),
            "setup": {"seconds": setup_s, "beads_per_s": N / setup_s, "first_build_seconds": setup_times[0],
                      "from": "host positions (pageable numpy), tree + factors + apply layout, device-synchronised"},
            "plan": {kk: info[kk] for kk in ("n_chunks", "n_top", "blob_bytes", "max_chunk_bytes", "n_case",
                                             "device_bytes", "tile_leaves", "chunk_smem", "top_staged", "chunk_ctas_per_sm", "chunk_smem_bytes",
                                             "top_global")},
            "bytes_per_bead_per_op": chunk_bytes / N,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
