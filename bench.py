#!/usr/bin/env python
"""bench.py -- fp64 Q~v + Q~^T v throughput (beads/s) of the B200 operators.

One step = one Q~v over every bead of the batch plus one Q~^T g over every
complement coordinate (BASELINE.json metric), on BASELINE config 2 by default
(1000 triaxial-ellipsoid-shell bodies x 4096 beads, fp64, synthetic seeded
input).  Operator (~0.8 GB of step blocks) and vectors (~0.2 GB) are far
larger than the 126 MB L2, so no L2 flush is needed between steps.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

N > 1 runs under torchrun, one rank per GPU.  Bodies are independent, so the
config's model is split across the ranks by cumulative bead count
(parallel.shard_bounds; strong scaling, the default) and every rank applies
its shard with no data-path collective; times are device-measured (CUDA
events) and max-reduced over ranks; the one-time NCCL gather of the shard
outputs is timed separately (gather_ms).  --sharding weak instead gives every
rank its own full config-sized model.  --emulate-shard R/N times shard R of N
alone on one GPU (per-shard device time for a strong-scaling estimate).

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
    ap.add_argument("--sharding", default=None, choices=["weak", "strong"],
                    help="strong (default for --gpus > 1): one config-sized model split across the ranks "
                         "by cumulative bead count (parallel.shard_bounds); weak: every rank owns a full "
                         "config-sized shard")
    ap.add_argument("--emulate-shard", default=None, help="R/N: time shard R of an N-way strong split alone")
    return ap.parse_args()


def workload(cfg: int, rank: int, scale: float, world: int = 1, strong: bool = False):
    from paper_1708_08427_b200.parallel import shard_of
    from paper_1708_08427_b200.workloads import CONFIGS, make_config

    if strong and world > 1:  # one model for the whole job, this rank's contiguous shard of its bodies
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
    # RQ_BENCH_SHARE_GPU=1 (functional check of the multi-rank path on a one-GPU box only: ranks
    # share the visible GPUs round-robin over gloo; its timings mean nothing)
    share = os.environ.get("RQ_BENCH_SHARE_GPU") == "1"
    if share:
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dist = None
    # RQ_BENCH_FORCE_DIST=1: initialise the process group even at world size 1 (under torchrun),
    # so the NCCL calls of the multi-rank path execute on a one-GPU box
    if world > 1 or os.environ.get("RQ_BENCH_FORCE_DIST") == "1":
        import torch.distributed as dist

        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    sharding = args.sharding or ("strong" if dist else "weak")
    strong = sharding == "strong"
    emu = None
    if args.emulate_shard:  # one shard of an N-way strong split, alone on this GPU
        er, en = (int(x) for x in args.emulate_shard.split("/"))
        emu = (er, en)
        pos, off, name, k = workload(args.config, er, args.scale, en, True)
    else:
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

    # ---- kernel-level roofline: the tile sweep (dominant kernel), timed alone
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
        for phase, label in ((1, "sweep"), (2, "top")):
            nrep = 50
            for _ in range(3):
                L.check(lib.rq_apply_ex(h, code, x.data_ptr(), outs[opn].data_ptr(), k, stream, phase))
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            for _ in range(nrep):
                L.check(lib.rq_apply_ex(h, code, x.data_ptr(), outs[opn].data_ptr(), k, stream, phase))
            b.record(s)
            torch.cuda.synchronize()
            # ms per launch (the single-RHS path launches once per column)
            kern[(opn, label)] = a.elapsed_time(b) / nrep / (1 if mrhs else k)
    per_step = 1 if mrhs else k  # launches of each phase per application
    sweep_ms = 0.5 * (kern[("qtilde_v", "sweep")] + kern[("qtilde_tv", "sweep")])
    info = op.plan.info()  # multi-RHS programs are built by the first k >= mrhs_min_k apply
    if mrhs:
        # tile-unit launch: the unit programs (entry headers + records) once per group of
        # 32 columns, every bead row and residue row of the k columns once, and the
        # tile-root exchange rows (written upward / read downward)
        ncg = (k + 31) // 32
        sweep_bytes = (info["mrhs_bytes"]["tiles"] * ncg + 8 * k * (3 * N + (3 * N - 6 * m))
                       + 8 * 6 * k * info["mrhs_units"]["tiles"])
        kname = "k_mrhs (column-parallel stack machine over tile units, lane = RHS column)"
    else:
        # algorithmic bytes per sweep launch (mean of the two directions): the step blocks the
        # direction streams (records + its metadata + gather lists), one read and one write of
        # every bead's 3 fp64 and residue coordinates, the tile-root exchange 6-vectors
        sweep_bytes = (0.5 * (info["sweep_bytes"]["up"] + info["sweep_bytes"]["down"])
                       + 8 * (3 * N + (3 * N - 6 * m)) + 48 * info["n_tiles"])
        kname = "k_wave (wavefront step sweep, TMA bulk-copied step blocks)"
    achieved = sweep_bytes / (sweep_ms * 1e-3) / 1e9
    peak, peak_src = peaks()
    step_ms_kernels = sum(kern.values()) * per_step
    share = (kern[("qtilde_v", "sweep")] + kern[("qtilde_tv", "sweep")]) * per_step / step_ms_kernels
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "wave_traffic.json")
    if os.path.exists(tpath) and not mrhs:
        with open(tpath) as f:
            tj = json.load(f)
        # dram bytes per sweep launch measured by ncu on the same config, scaled per bead
        if tj.get("config") == args.config and tj.get("beads"):
            traffic = tj["dram_bytes_per_launch"] * N / tj["beads"]

    # ---- parity of this run's own outputs against the CPU oracle on a sample of bodies
    parity = None
    if rank == 0:
        from oracle.oracle import OracleBatch

        nb = min(m, 64 if args.config != 3 else 1)
        if k == 1 and (args.config != 3 or N <= (1 << 20)):
            ob = OracleBatch(pos[:off[nb]], off[:nb + 1], threads=len(os.sched_getaffinity(0)))
            outv = op.apply("qtilde_v", v).cpu().numpy()
            outg = op.apply("qtilde_tv", g).cpu().numpy()
            vh, gh = v.cpu().numpy(), g.cpu().numpy()
            worst = 0.0
            for opn, x, y, li, lo in (("qtilde_v", vh, outv, 3, 3), ("qtilde_tv", gh, outg, 3, 3)):
                xi = x[:3 * int(off[nb])] if opn == "qtilde_v" else x[:3 * int(off[nb]) - 6 * nb]
                ref = ob.apply(opn, xi)
                yo = y[:len(ref)]
                o = 0
                for j in range(nb):
                    nj = int(off[j + 1] - off[j])
                    ln = 3 * nj - 6 if opn == "qtilde_v" else 3 * nj
                    r = ref[o:o + ln]
                    worst = max(worst, float(np.linalg.norm(yo[o:o + ln] - r) / max(np.linalg.norm(r), 1e-300)))
                    o += ln
            parity = {"max_rel": worst, "bodies": nb, "ops": ["qtilde_v", "qtilde_tv"],
                      "against": "C oracle (oracle/rq_oracle.c, pinned to the reference by tests/golden)",
                      "tolerance": 1e-12}

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
    # A Zf / Z^T u call is a few microseconds of device time -- less than one Python + ctypes
    # call -- so 20 calls are captured in a CUDA graph and the graph replays are timed (device
    # time of the kernels back to back); the per-call host path is reported beside it.
    zs = torch.cuda.Stream()
    zs.wait_stream(torch.cuda.current_stream())
    for zname, zfn in (("zf", lambda: op.zf(fz)), ("ztu", lambda: op.ztu(uz))):
        with torch.cuda.stream(zs):
            for _ in range(3):
                zfn()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(zs)
            for _ in range(20):
                zfn()
            a1.record(zs)
        torch.cuda.synchronize()
        host_ms = a0.elapsed_time(a1) / 20
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=zs):
            for _ in range(20):
                zfn()
        with torch.cuda.stream(zs):
            graph.replay()
            torch.cuda.synchronize()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(zs)
            for _ in range(5):
                graph.replay()
            a1.record(zs)
        torch.cuda.synchronize()
        zms = a0.elapsed_time(a1) / 100
        del graph
        zops[zname] = {"ms": zms, "beads_per_s": N / (zms * 1e-3), "achieved_gbs": 48 * N / (zms * 1e-3) / 1e9,
                       "frac": 48 * N / (zms * 1e-3) / 1e9 / peaks()[0], "timing": "CUDA graph of 20 calls",
                       "ms_per_python_call": host_ms}

    # ---- end to end with HOST buffers, copies inside the timed region: the C ABI on pinned
    # buffers (what a binding that owns pinned memory calls) and the drop-in Python API on
    # numpy arrays (MultiBodyOperator.apply, the reference's own calling convention)
    e2e = None
    if not args.no_e2e:
        hv = torch.empty(v2.shape, dtype=torch.float64, pin_memory=True)
        hg = torch.empty(g2.shape, dtype=torch.float64, pin_memory=True)
        hv.copy_(v2)
        hg.copy_(g2)
        ho1 = torch.empty((3 * N - 6 * m, k), dtype=torch.float64, pin_memory=True)
        ho2 = torch.empty((3 * N, k), dtype=torch.float64, pin_memory=True)
        e_steps = max(3, min(50, args.steps))
        def host_step():  # both applications queued on the async host path
            L.check(lib.rq_apply_host_async(h, L.OP_QTILDE_V, hv.data_ptr(), ho1.data_ptr(), k))
            L.check(lib.rq_apply_host_async(h, L.OP_QTILDE_TV, hg.data_ptr(), ho2.data_ptr(), k))

        for _ in range(2):
            host_step()
            L.check(lib.rq_host_wait(h))
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        # (1) streaming: the K steps queued back to back (two staging slots: the H2D of the next
        # operand overlaps the D2H of the previous result), one wait after the last step
        t0 = time.perf_counter()
        for _ in range(e_steps):
            host_step()
        L.check(lib.rq_host_wait(h))
        e2e_ms = (time.perf_counter() - t0) / e_steps * 1e3
        # (2) every step waited for before the next one starts
        t0 = time.perf_counter()
        for _ in range(e_steps):
            host_step()
            L.check(lib.rq_host_wait(h))
        sync_ms = (time.perf_counter() - t0) / e_steps * 1e3
        # numpy (pageable) through the Python API
        nv, ng = hv.numpy().reshape(v.shape).copy(), hg.numpy().reshape(g.shape).copy()
        for _ in range(2):
            op.apply("qtilde_v", nv)
            op.apply("qtilde_tv", ng)
        n_steps = max(3, min(10, args.steps))
        t0 = time.perf_counter()
        for _ in range(n_steps):
            op.apply("qtilde_v", nv)
            op.apply("qtilde_tv", ng)
        np_ms = (time.perf_counter() - t0) / n_steps * 1e3
        # the same pair through MultiBodyOperator.apply_many (both queued, one wait)
        for _ in range(2):
            op.apply_many([("qtilde_v", nv), ("qtilde_tv", ng)])
        t0 = time.perf_counter()
        for _ in range(n_steps):
            op.apply_many([("qtilde_v", nv), ("qtilde_tv", ng)])
        npm_ms = (time.perf_counter() - t0) / n_steps * 1e3
        if dist:
            t = torch.tensor([e2e_ms, np_ms, npm_ms, sync_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms, np_ms, npm_ms, sync_ms = (float(x) for x in t.tolist())
        nbytes_in = (hv.numel() + hg.numel()) * 8
        nbytes_out = (ho1.numel() + ho2.numel()) * 8
        e2e = {"value": n_job * k / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": nbytes_in,
               "d2h_bytes_per_step": nbytes_out, "ms_per_step": e2e_ms,
               "path": "rq_apply_host_async x2 per step, K steps queued, one rq_host_wait (C ABI, pinned "
                       "host buffers; every step's H2D of its inputs and D2H of its results inside the timed "
                       "region)",
               "per_step_wait": {"value": n_job * k / (sync_ms * 1e-3), "ms_per_step": sync_ms,
                                 "path": "the same with rq_host_wait after every step"},
               "numpy": {"value": n_job * k / (np_ms * 1e-3), "ms_per_step": np_ms,
                         "path": "MultiBodyOperator.apply x2 on numpy arrays (pageable inputs staged by "
                                 "host threads; results returned in page-locked numpy arrays)"},
               "numpy_many": {"value": n_job * k / (npm_ms * 1e-3), "ms_per_step": npm_ms,
                              "path": "MultiBodyOperator.apply_many([(qtilde_v, v), (qtilde_tv, g)]) on numpy "
                                      "arrays (both queued, one wait)"}}

    # ---- one-time gather of the shard outputs (strong sharding): NCCL all_gather of the
    # max-padded shards, timed on the device, max over ranks
    gather = None
    if dist and strong:
        from paper_1708_08427_b200.parallel import gather_shards

        yv = op.apply("qtilde_v", v).reshape(-1)
        rt = torch.tensor([yv.shape[0]], device=dev, dtype=torch.int64)
        rows = [torch.zeros_like(rt) for _ in range(world)]
        dist.all_gather(rows, rt)
        rows = [int(r.item()) for r in rows]
        torch.cuda.synchronize()
        dist.barrier()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(s)
        full = gather_shards(yv, rows)
        a1.record(s)
        torch.cuda.synchronize()
        gms = torch.tensor([a0.elapsed_time(a1)], device=dev)
        dist.all_reduce(gms, op=dist.ReduceOp.MAX)
        gather = {"ms": float(gms.item()), "bytes": int(full.numel()) * 8, "what": "Q~v of the whole job to every rank"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = len(os.sched_getaffinity(0))
        nb = min(m, 200)
        rate, steps, el = cpu_oracle_rate(pos[:off[nb]], off[:nb + 1], args.cpu_sample_s, threads)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"first {nb} bodies ({int(off[nb])} beads) of the workload, {steps} steps "
                         f"of Q~v+Q~^T g in {el:.1f} s (C oracle, OpenMP over bodies)"}
        # the reference as shipped is pure Python and cannot travel to the GPU box: its rate on
        # config-2 bodies was measured in the build container (tools/ref_python_timing.py) and is
        # quoted here as recorded, not re-measured
        rp = os.path.join(ROOT, "profiles", "r02f_reference_python_timing.json")
        if os.path.exists(rp):
            with open(rp) as fh:
                r = json.load(fh)
            cpu["reference_python_recorded"] = {
                "single_process_beads_per_s": r["reference_python_single_process"]["step_beads_per_s"],
                "pool_beads_per_s": r["reference_python_pool"]["step_beads_per_s"],
                "pool_workers": r["reference_python_pool"]["workers"],
                "c_oracle_over_python_pool": r["oracle_over_python_pool"],
                "where": r["where"] + "; " + r["config"] + " (recorded file, not this run)"}

    launches = args.steps * (lib.rq_launches_per_apply(h, L.OP_QTILDE_V, k) +
                             lib.rq_launches_per_apply(h, L.OP_QTILDE_TV, k))
    if rank == 0:
        cfgd = config_dict(name, off, k, world, strong and world > 1)
        if emu:
            cfgd["sharding"] = f"emulated: shard {emu[0]} of a {emu[1]}-way strong split, alone on one GPU"
        line = {
            "metric": METRIC, "value": value * k, "unit": UNIT if k == 1 else "bead-RHS/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if (strong and world > 1) else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": cfgd,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": kname,
                         "bytes_per_launch": sweep_bytes, "launch_ms": sweep_ms, "peak_source": peak_src,
                         "share_of_step": share},
            "kernels_ms": {f"{a}:{b}": v_ for (a, b), v_ in kern.items()},
            "step_ms_single": step_stats,
            "parity": parity,
            "z_ops": zops,
            "batched_k100": batched,
            "cpu_baseline": cpu, "e2e": e2e, "gather": gather, "clocks": ck, "gpu_launches": int(launches),
            "setup": {"seconds": setup_s, "beads_per_s": N / setup_s, "first_build_seconds": setup_times[0],
                      "from": "host positions (pageable numpy), tree + factors + apply layout, device-synchronised"},
            "plan": {kk: info[kk] for kk in ("n_streams", "n_steps", "n_top", "n_tiles", "blob_bytes", "sweep_bytes",
                                             "n_case", "device_bytes", "tile_leaves", "rounds",
                                             "node_slots", "stage_bytes", "sweep_smem", "sweep_ctas_per_sm",
                                             "top_staged", "top_global")},
            "bytes_per_bead_per_op": sweep_bytes / N,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
