#!/usr/bin/env python
"""Benchmark of the element-based P1 hot path (BASELINE.json metric, config C2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1], "C2"): 2D P1 triangles on the unit square at level 11
(n_n = 4,198,401, n_e = 8,388,608), node numbering randomly permuted from the seed,
x ~ U[-1,1], nu = 1, f = 1; one step = one element-based residual r = b - A x.
Prints ONE JSON line (rank 0).  `value` = GDoF/s with inputs resident in HBM, timed with
CUDA events over exactly K steps; `e2e` = the same through the public API
(`residual(batch, x_host)`) with the host->device copy of x and the device->host copy of r
inside the timed region.  `--impl reference` times the CPU oracle port of the reference
residual (oracle/, NumPy, all host threads) on the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0}
METRIC = "element matvec GDoF/s & HBM GB/s (fraction of peak); PCG iterations/sec"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return PEAKS_FALLBACK, "fallback"


def residual_bytes(n_n, n_e, nb=3):
    """matvec n_e(8 nb^2 + 4 nb) + 16 n_n, residual + 8 n_n (b pre-assembled)."""
    return n_e * (8 * nb * nb + 4 * nb) + 24 * n_n


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """Samples SM clock and throttle reasons (NVML) in a thread while running."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index=0, period=0.01):
        self.samples = []
        self.reasons = 0
        self.max_mhz = None
        self.period = period
        self._stop = threading.Event()
        self._ok = False
        self._gate = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._ok = True
        except Exception:
            self._ok = False
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            if self._gate.is_set():
                try:
                    mhz = self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM)
                    r = self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                    self.samples.append(mhz)
                    self.reasons |= int(r)
                except Exception:
                    pass
            time.sleep(self.period)

    def start(self):
        if self._ok:
            self._t.start()
        return self

    def on(self):
        self._gate.set()

    def off(self):
        self._gate.clear()

    def stop(self):
        self._stop.set()
        if self._ok:
            self._t.join(timeout=1.0)

    def summary(self):
        if not self._ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        names = [v for k, v in self.REASONS.items() if self.reasons & k]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(self.samples)}


# ------------------------------------------------------------- CPU oracle --
def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def oracle_residual_rate(A, b_e, indt, x, budget_s=10.0, min_calls=3, threads=None):
    """Time oracle.residual (the reference algorithm, NumPy, T threads) for ~budget_s."""
    import oracle as o
    T = threads or cpu_threads()
    o.residual(A, b_e, indt, x, threads=T)  # warm
    t0 = time.perf_counter()
    calls = 0
    while calls < min_calls or time.perf_counter() - t0 < budget_s:
        o.residual(A, b_e, indt, x, threads=T)
        calls += 1
    dt = time.perf_counter() - t0
    return x.shape[0] * calls / dt / 1e9, T, calls, dt


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def _reference_package():
    """The unmodified reference package `ebsolve`, pip-installed into baseline/_ref
    (`python -m pip install --no-index --no-build-isolation --no-deps --target
    baseline/_ref <copy of /root/reference/pkg>`), or None when it is not installed."""
    if not os.path.isdir(os.path.join(REF_DIR, "ebsolve")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import ebsolve
        return ebsolve
    except Exception:  # noqa: BLE001
        return None


def reference_c2_inputs(eb_ref, seed, size):
    """The BASELINE C2 workload built with the reference's own public API: the level-11
    unit square (mesh.py:104-137), nodes relabelled by the seeded permutation (new id of
    old node i = perm[i]; oracle config_inputs' recipe: one default_rng(seed), permutation
    then x ~ U[-1, 1]), build_element_batch(nu=1, f=1) (elements.py:124-137)."""
    import numpy as np
    level = 11 if size is None else size
    m0 = eb_ref.build_unit_square_mesh(level)
    rng = np.random.default_rng(seed)
    perm = rng.permutation(m0.n_nodes)
    nodes = np.empty_like(m0.nodes)
    nodes[perm] = m0.nodes
    m = eb_ref.Mesh(nodes, perm[m0.elements], np.sort(perm[m0.boundary_nodes]))
    x = rng.uniform(-1.0, 1.0, m.n_nodes)
    return eb_ref.build_element_batch(m, nu=1.0), x, m


def run_reference(args):
    """--impl reference: the reference's own CPU implementation of the path on this host's
    cores -- the unmodified `ebsolve.residual(batch, x, threads=T, deterministic=False)`
    (operators.py:72-111; its fast mode, like the GPU arm's value; the default bit-exact
    mode timed beside it under exact_mode) from baseline/_ref when installed ("kind":
    "reference"), else the oracle port of the same algorithm (oracle/ebs_oracle.py, "kind":
    "port").  Under torchrun only rank 0 runs it."""
    import numpy as np
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    T = cpu_threads()
    t_setup = time.perf_counter()
    eb_ref = _reference_package()
    if eb_ref is not None:
        batch, x, m = reference_c2_inputs(eb_ref, args.seed, args.size)
        n_n, n_e = m.n_nodes, m.n_elements
        kind = "reference"
        # the same mode as the GPU arm's `value` / `e2e` (fast: per-chunk partial sums,
        # operators.py:108-111); the bit-exact default mode is timed beside it below
        run = lambda: eb_ref.residual(batch, x, threads=T, deterministic=False)  # noqa: E731
        run_exact = lambda: eb_ref.residual(batch, x, threads=T, deterministic=True)  # noqa: E731
        what = (f"ebsolve.residual(batch, x, threads={T}, deterministic=False) -- the unmodified "
                "reference package from baseline/_ref, its fast mode like the GPU arm's value")
    else:
        import oracle as o
        inp = o.config_inputs(2, seed=args.seed, size=args.size)
        _, _, A, b_e = o.element_matrices(inp["nodes"], inp["elements"], nu=inp["nu"])
        indt = np.ascontiguousarray(inp["elements"].T)
        x = inp["x"]
        n_n, n_e = x.shape[0], indt.shape[1]
        kind = "port"
        run = lambda: o.residual(A, b_e, indt, x, threads=T)  # noqa: E731
        run_exact = None
        what = (f"oracle/ebs_oracle.py residual (the reference algorithm restated, deterministic "
                f"chunked mode, {T} threads; baseline/_ref not installed)")
    setup = time.perf_counter() - t_setup
    for _ in range(args.warmup):
        run()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        run()
    dt = time.perf_counter() - t0
    value = n_n * args.steps / dt / 1e9
    exact = None
    if run_exact is not None:  # the reference's default (bit-exact) mode, a bounded sample
        run_exact()
        k = max(1, min(args.steps, 10))
        t1 = time.perf_counter()
        for _ in range(k):
            run_exact()
        exact = {"value": n_n * k / (time.perf_counter() - t1) / 1e9, "unit": "GDoF/s",
                 "steps": k, "note": "deterministic=True (the reference default)"}
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GDoF/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded BASELINE C2 recipe)",
        "config": workload_config(n_n, n_e, args, mode="fast (per-chunk partial sums)"
                                  if kind == "reference" else "reference order (bincount)"),
        "cpu_baseline": {"value": value, "unit": "GDoF/s", "cores": T, "kind": kind,
                         "sample": f"{args.steps} full C2 residuals: {what}"},
        "e2e": {"value": value, "unit": "GDoF/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "setup_s": setup,
    }
    if exact is not None:
        line["exact_mode"] = exact
    print(json.dumps(line), flush=True)


def workload_config(n_n, n_e, args, mode):
    """The bench workload: BASELINE C2 at every N (one GPU, or strong-scaled over N element
    slabs np.linspace(0, n_e, N+1) -- operators.py:100's chunk rule -- under torchrun)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    return {"workload": "C2: 2D P1 unit square, level 11, permuted node numbering, "
                        "x~U[-1,1], nu=1, f=1; element residual r=b-Ax per step",
            "n_nodes": n_n, "n_elements": n_e, "seed": args.seed, "mode": mode,
            "l2": "inputs larger than L2 (slot stream ~1 GB vs 126 MB L2); no flush",
            "parallelism": "single GPU" if world <= 1 else
            f"element slabs x{world} (strong scaling of the fixed C2 mesh, NCCL halo)"}


# ---------------------------------------------------------------- GPU arm --
def run_ours(args):
    import ctypes

    import numpy as np
    import torch

    import paper_1911_03973_b200 as eb
    from paper_1911_03973_b200 import _device as D
    from paper_1911_03973_b200._lib import EBS_RES_EXACT, EBS_RES_FAST, load
    from paper_1911_03973_b200.inputs import config_problem

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 or os.environ.get("EBS_BENCH_DIST") == "1":
        import bench_dist
        return bench_dist.bench_rank(args, rank, world, local)
    torch.cuda.set_device(local)
    peaks, peak_kind = load_peaks()
    sampler = ClockSampler(index=local).start()

    t_setup = time.perf_counter()
    p = config_problem(2, seed=args.seed, size=args.size)
    batch, m = p["batch"], p["mesh"]
    n_n, n_e = m.n_nodes, m.n_elements
    pl = batch.operator(n_n)
    torch.cuda.synchronize()
    setup = time.perf_counter() - t_setup
    lib = load()
    h = pl.handle
    x_np = p["x"]
    x_dev = torch.from_numpy(x_np).cuda()
    x_int = D.empty(n_n)
    r_dev = D.empty(n_n)
    stream = torch.cuda.current_stream()
    s = ctypes.c_void_p(stream.cuda_stream)
    xp, xip, rp = (ctypes.c_void_p(t.data_ptr()) for t in (x_dev, x_int, r_dev))

    flag = D.zeros(1, torch.int32)
    fp = ctypes.c_void_p(flag.data_ptr())

    def step(op, st=None):
        # one residual through the C-ABI entry point (x and r in the caller's numbering,
        # finiteness check included): x permutation (+ r := -0.0), SELL pass
        lib.ebs_residual(h, xp, rp, EBS_RES_FAST if op == 1 else EBS_RES_EXACT, 0, fp, st or s)

    unit_stats = {}

    def timed(op, K):
        """K residual steps timed as a whole (no events inside the timed region), then a
        separate K-step pass with events around each launch for the per-kernel times."""
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        n0 = lib.ebs_launch_count()
        e0.record(stream)
        for k in range(K):
            step(op)
        e1.record(stream)
        torch.cuda.synchronize()
        launches = lib.ebs_launch_count() - n0
        total = e0.elapsed_time(e1) / 1e3
        # per-step pass: the same two kernels called separately with events around each
        # step (the -0.0 pre-fill of r that ebs_residual runs is done outside the events)
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(K)]
        for k in range(K):
            r_dev.fill_(-0.0)
            evs[k][0].record(stream)
            lib.ebs_to_internal(h, xp, xip, None, s)
            evs[k][1].record(stream)
            lib.ebs_plan_apply(h, op, xip, rp, 2, 0, s)
            evs[k][2].record(stream)
        torch.cuda.synchronize()
        per_step = sorted(ev[0].elapsed_time(ev[2]) for ev in evs)
        unit_stats.update(median_ms=statistics.median(per_step), best_ms=per_step[0])
        # per-kernel durations inside the step sequence: the median over the K steps (the
        # mean would count the rare host gaps of an eager launch loop)
        gather = statistics.median(ev[0].elapsed_time(ev[1]) for ev in evs) / 1e3
        sell = statistics.median(ev[1].elapsed_time(ev[2]) for ev in evs) / 1e3
        return total, gather, sell, launches

    # warm-up: W steps, then keep the clocks busy for ~1 s before timing
    for _ in range(max(3, args.warmup)):
        step(1)
    torch.cuda.synchronize()
    sampler.on()
    t_soak = time.perf_counter()
    while time.perf_counter() - t_soak < 1.0:
        for _ in range(20):
            step(1)
        torch.cuda.synchronize()
    total, gather, sell, launches = timed(1, args.steps)
    fast_stats = dict(unit_stats)
    r_fast = r_dev.clone()
    # the same K steps replayed from a captured CUDA graph (launch gaps removed)
    total_graph = None
    try:
        G = 10
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            cs = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
            for _ in range(G):
                step(1, cs)
        g.replay()
        torch.cuda.synchronize()
        eg0, eg1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        eg0.record(stream)
        done = 0
        while done + G <= args.steps:
            g.replay()
            done += G
        for _ in range(args.steps - done):
            step(1)
        eg1.record(stream)
        torch.cuda.synchronize()
        total_graph = eg0.elapsed_time(eg1) / 1e3
        assert torch.equal(r_dev, r_fast)
        del g
    except Exception as e:  # noqa: BLE001 -- report, keep the eager number
        print(f"graph replay unavailable: {e}", file=sys.stderr)
    # the K independent residuals as ONE call with two in flight (ebs_residual_many: odd
    # steps on a second stream with their own workspace, so the x permutation and -0.0 fill
    # of one step overlap the SELL pass of the other); every step writes its own output row
    total_many = None
    total_many_ex = None
    r_exact_many = None
    launches_many = None
    try:
        rows = min(args.steps, 128)   # output rows per call (4.3 GB at most)
        r_rows = D.empty((rows, n_n))
        flags_many = D.zeros(rows, torch.int32)
        rrp, fmp = (ctypes.c_void_p(t.data_ptr()) for t in (r_rows, flags_many))

        def many(k, mode=EBS_RES_FAST):
            rc = lib.ebs_residual_many(h, xp, 0, rrp, n_n, k, mode, 0, fmp, s)
            assert rc == 0, rc

        many(rows)
        torch.cuda.synchronize()
        em0, em1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n0 = lib.ebs_launch_count()
        em0.record(stream)
        done = 0
        while done < args.steps:
            k = min(rows, args.steps - done)
            many(k)
            done += k
        em1.record(stream)
        torch.cuda.synchronize()
        launches_many = lib.ebs_launch_count() - n0
        total_many = em0.elapsed_time(em1) / 1e3
        assert torch.equal(r_rows[0], r_fast) and torch.equal(r_rows[k - 1], r_fast), \
            "ebs_residual_many and ebs_residual disagree"
        assert not bool(flags_many.any())
        # the bit-exact mode the same way
        many(rows, EBS_RES_EXACT)
        torch.cuda.synchronize()
        em0.record(stream)
        done = 0
        while done < args.steps:
            k = min(rows, args.steps - done)
            many(k, EBS_RES_EXACT)
            done += k
        em1.record(stream)
        torch.cuda.synchronize()
        total_many_ex = em0.elapsed_time(em1) / 1e3
        r_exact_many = r_rows[k - 1].clone()
        del r_rows
    except Exception as e:  # noqa: BLE001 -- report, keep the one-at-a-time number
        print(f"ebs_residual_many unavailable: {e}", file=sys.stderr)
        total_many = None
    total_ex, gather_ex, sell_ex, _ = timed(2, args.steps)
    total_ex_seq = total_ex
    if total_many_ex is not None:
        assert torch.equal(r_exact_many, r_dev), "exact ebs_residual_many and ebs_residual disagree"
        total_ex = total_many_ex
    # the solver path's operator: matvec on internal-numbered vectors (no permutation in
    # or out, coalesced output) -- what Jacobi / CG / PCG iterate on
    y_int = D.empty(n_n)
    yp = ctypes.c_void_p(y_int.data_ptr())
    ev_i = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for _ in range(3):
        lib.ebs_plan_apply(h, 0, xip, yp, 0, 0, s)
    ev_i[0].record(stream)
    for _ in range(args.steps):
        lib.ebs_plan_apply(h, 0, xip, yp, 0, 0, s)
    ev_i[1].record(stream)
    torch.cuda.synchronize()
    t_int = ev_i[0].elapsed_time(ev_i[1]) / 1e3 / args.steps
    sampler.off()

    # end to end through the public API: pinned host x in, host r out.  Headline: the
    # pipelined many-vector call (H2D, kernels and D2H of consecutive steps overlap);
    # also the one-call-per-step figure (every copy and a host sync serialised).
    x_host = torch.from_numpy(x_np).pin_memory()
    r_host = torch.empty(n_n, dtype=torch.float64).pin_memory()
    chunk = min(args.steps, 128)   # rows of pinned output per call (4.3 GB at most)
    r_many = torch.empty((chunk, n_n), dtype=torch.float64).pin_memory()
    xs_host = x_host.unsqueeze(0).expand(chunk, n_n)   # the step's x: same pinned host vector
    for _ in range(max(3, args.warmup)):
        r_host.copy_(eb.residual(batch, x_host, deterministic=False), non_blocking=True)
    # warm the host-pipeline buffers and the DMA mappings of every pinned output row
    eb.residual_many(batch, xs_host, out=r_many, deterministic=False)
    torch.cuda.synchronize()
    for _ in range(int(os.environ.get("EBS_E2E_REPEAT", "0"))):   # diagnostics: spread
        t0 = time.perf_counter()
        eb.residual_many(batch, xs_host, out=r_many, deterministic=False)
        print(f"e2e pass: {(time.perf_counter() - t0) / chunk * 1e3:.3f} ms/step", file=sys.stderr)
    sampler.on()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    done = 0
    while done < args.steps:
        k = min(chunk, args.steps - done)
        eb.residual_many(batch, xs_host[:k], out=r_many[:k], deterministic=False)
        done += k
    e1.record(stream)
    torch.cuda.synchronize()
    wall_e2e = time.perf_counter() - t0
    t_e2e = e0.elapsed_time(e1) / 1e3
    assert torch.equal(r_many[k - 1], r_fast.cpu()), "pipelined API and C-ABI paths disagree"
    e1s = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e1s[0].record(stream)
    for _ in range(args.steps):
        r_host.copy_(eb.residual(batch, x_host, deterministic=False), non_blocking=True)
    e1s[1].record(stream)
    torch.cuda.synchronize()
    sampler.off()
    sampler.stop()
    t_e2e_single = e1s[0].elapsed_time(e1s[1]) / 1e3
    assert torch.equal(r_host, r_fast.cpu()), "public API and C-ABI paths disagree"

    bytes_alg = residual_bytes(n_n, n_e)
    total_eager = total
    if total_graph is not None:  # one at a time: CUDA-graph replay of the same K residuals
        total = total_graph
    total_seq = total
    if total_many is not None:   # headline: the K residuals with two in flight
        total = total_many
        launches = launches_many
    value = n_n * args.steps / total / 1e9
    achieved = bytes_alg / sell / 1e9
    peak = float(peaks["hbm_gbs"])
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic = json.load(f).get("k_sell_op<3,1,1>@C2")
    except Exception:
        pass

    cpu = None
    if not args.no_cpu:
        import oracle  # noqa: F401  (CPU baseline only)
        A = batch.A_e.permute(2, 0, 1).contiguous().cpu().numpy().transpose(1, 2, 0)
        b_e = batch.b_e.cpu().numpy()
        indt = batch.index.indt.cpu().numpy().astype(np.int64)
        rate, T, calls, dt = oracle_residual_rate(A, b_e, indt, x_np, budget_s=args.cpu_budget)
        cpu = {"value": rate, "unit": "GDoF/s", "cores": T, "kind": "port",
               "sample": f"{calls} full C2 residuals in {dt:.1f} s (oracle/ebs_oracle.py residual, "
                         f"reference algorithm, {T} threads)"}

    extra = {}
    paper = None
    if args.extra:
        extra = solver_extras(args)
        try:
            paper = paper_experiment()
        except Exception as e:  # noqa: BLE001
            paper = {"error": f"{type(e).__name__}: {e}"}

    line = {
        "metric": METRIC, "value": value, "unit": "GDoF/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE C2 recipe: permuted level-11 mesh, x~U[-1,1])",
        "config": workload_config(
            n_n, n_e, args,
            mode="fast (pre-assembled b)" + (
                "; the K independent residuals issued as one ebs_residual_many call, two in "
                "flight on two streams, each writing its own output row (one at a time: "
                "`sequential`)" if total_many is not None else "")),
        "hbm_gbs_algorithmic": bytes_alg / (total / args.steps) / 1e9,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": "k_sell_op<3,1,1> (fused gather-product-ordered-sum, packed ids, red.add caller-order output)",
                     "bytes_per_launch": bytes_alg, "kernel_ms": sell * 1e3,
                     "gather_kernel_ms": gather * 1e3, "peak_source": peak_kind,
                     "step_frac": bytes_alg / (total / args.steps) / 1e9 / peak,
                     "step_frac_sequential": bytes_alg / (total_seq / args.steps) / 1e9 / peak,
                     "step_note": "step_frac: the same algorithmic bytes over the whole "
                                  "ms_per_step (x permutation + -0.0 fill + SELL pass); "
                                  "kernel_ms / frac: the SELL pass timed alone in the "
                                  "one-at-a-time sequence"},
        "sequential": {"value": n_n * args.steps / total_seq / 1e9, "unit": "GDoF/s",
                       "ms_per_step": total_seq / args.steps * 1e3,
                       "note": "one residual at a time (ebs_residual, CUDA-graph replay of 10 "
                               "steps): the `value` of round 1 and of the earlier round-2 runs"},
        "timing": {"mode": ("residual_many (two in flight), eager call" if total_many is not None
                            else "cuda_graph" if total_graph is not None else "eager"),
                   "eager_value": n_n * args.steps / total_eager / 1e9,
                   "eager_ms_per_step": total_eager / args.steps * 1e3,
                   "per_step_events_ms": {k: round(v, 5) for k, v in fast_stats.items()},
                   "note": "value: the K residuals (fast mode: x permutation, r := -0.0, SELL "
                           "pass adding into r) through ebs_residual_many, two in flight; "
                           "sequential: ebs_residual replayed from a captured CUDA graph of "
                           "10 steps; eager: one ctypes call per step; "
                           "per_step_events_ms: the unfused split (ebs_to_internal, "
                           "ebs_plan_apply out_user=2) with events around each launch; "
                           "roofline.kernel_ms / gather_kernel_ms: the medians of those "
                           "per-launch intervals"},
        "internal_matvec": {"kernel_ms": t_int * 1e3,
                            "achieved_gbs": (bytes_alg - 8 * n_n) / t_int / 1e9,
                            "frac": (bytes_alg - 8 * n_n) / t_int / 1e9 / peak,
                            "bytes_per_launch": bytes_alg - 8 * n_n,
                            "note": "y = A x on plan-internal vectors (solver path), "
                                    "matvec bytes n_e(8nb^2+4nb)+16n_n"},
        "exact_mode": {"value": n_n * args.steps / total_ex / 1e9, "unit": "GDoF/s",
                       "sequential_value": n_n * args.steps / total_ex_seq / 1e9,
                       "kernel_ms": sell_ex * 1e3,
                       "note": "bit-identical to ebsolve.residual (b_e streamed per slot); value: two in flight (ebs_residual_many), sequential_value: one at a time"},
        "e2e": {"value": n_n * args.steps / t_e2e / 1e9, "unit": "GDoF/s",
                "h2d_bytes_per_step": 8 * n_n, "d2h_bytes_per_step": 8 * n_n,
                "wall_s": wall_e2e,
                "api": "paper_1911_03973_b200.residual_many(batch, xs_pinned_host, out=pinned_host, "
                       f"deterministic=False) over chunks of {chunk} steps (copies overlap kernels)",
                "single_call": {"value": n_n * args.steps / t_e2e_single / 1e9, "unit": "GDoF/s",
                                "api": "residual(batch, x_pinned_host, deterministic=False) "
                                       "+ copy to pinned host, one call per step"}},
        "gpu_launches": launches,
        "clocks": sampler.summary(),
        "cpu_baseline": cpu,
        "setup_s": setup,
    }
    if cpu:  # like-for-like speed-ups over the CPU reference algorithm (reference order)
        line["vs_cpu_baseline"] = {
            "fast": value / cpu["value"],
            "fast_sequential": line["sequential"]["value"] / cpu["value"],
            "exact": line["exact_mode"]["value"] / cpu["value"],
            "e2e": line["e2e"]["value"] / cpu["value"],
            "note": "exact: the bit-identical (reference-order) GPU residual vs the same "
                    "algorithm on the host; fast: pre-assembled b (within 1e-12)"}
    if extra:
        line["solvers"] = extra
    if paper:
        line["paper_experiment"] = paper
    print(json.dumps(line), flush=True)


def emulated_slabs(batch, d, m, cfg, iters, t1, h1, P=8):
    """The C4 / C5 slab solve on P element slabs EMULATED on this one GPU through the
    peer-memory transport (dist.emulate(..., peer=True): the ranks' windows, fused sweeps,
    combines and fused all-reduce, every rank's kernels back to back, CUDA-graph batches):
    the emulated time is the sum of the ranks' work, so E = T1 / T_emulated is the
    compute-side strong-scaling efficiency at P GPUs before any NVLink latency.  The slab
    norm history is checked against the 1-GPU solve (h1)."""
    import numpy as np
    import torch

    from paper_1911_03973_b200 import dist
    prob, _ = dist.emulate(batch, m.n_nodes, d, P, peer=True)
    try:
        x0 = torch.zeros(m.n_nodes, dtype=torch.float64, device="cuda")
        xin = [op.to_internal(x0) for op in prob.ops]
        run = (lambda: dist.jacobi(prob, xin, iters, 0.8, graph=True)) if cfg == 4 else \
            (lambda: dist.pcg(prob, xin, iters, graph=True))
        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _, norms = run()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3
        h1 = np.asarray(h1)
        live = np.abs(h1) >= 1e-10 * abs(h1[0]) if len(h1) == len(norms) else None
        dev = (float(np.max(np.abs(norms[live] - h1[live]) / np.abs(h1[live])))
               if live is not None else None)
        return {"slabs": P, "it_per_s": iters / t, "e_compute": t1 / t,
                "history_vs_1gpu_max_rel": dev, "diverged": bool(prob.diverged),
                "transport": "peer memory (LocalPeerTransport: windows, fused sweeps, combines, "
                             "fused all-reduce)",
                "note": f"{P} element slabs emulated on this ONE GPU, ranks back to back: "
                        "the time is the sum of the ranks' work, e_compute = T_1GPU / T_emulated "
                        "(compute-side strong-scaling efficiency, no NVLink latency)"}
    finally:
        prob.comm.close()
        del prob
        torch.cuda.empty_cache()


def solver_extras(args):
    """Solver throughput on the other BASELINE configs (C3 JPCG, C4 Jacobi, C5 JPCG)."""
    import numpy as np
    import torch

    import paper_1911_03973_b200 as eb
    from paper_1911_03973_b200.inputs import config_problem
    out = {}
    peaks, _ = load_peaks()
    runs = [(3, 20000, 1e-8, False), (4, 200, None, False), (5, 500, None, False),
            (3, 20000, 1e-8, True)]
    for cfg, iters, tol, permuted in runs:
        if cfg not in args.solver_configs:
            continue
        try:
            t0 = time.perf_counter()
            if permuted:
                # the unstructured-numbering 3D path: C3 with its node labels randomly
                # permuted (seeded), so the plan falls back from the one-byte tuple codes
                # of a structured numbering to first-appearance ids + 8 B delta words
                p = config_problem(cfg, seed=args.seed, assemble=False)
                perm = np.random.default_rng(args.seed + 1).permutation(p["mesh"].n_nodes)
                m = eb.permute_nodes(p["mesh"], perm)
                nd = eb.face_z0_nodes(m)
                d = eb.DirichletData(nd, torch.zeros(nd.numel(), dtype=torch.float64,
                                                     device="cuda"))
                batch = eb.build_element_batch(m, nu=p["nu"])
                p = {"batch": batch, "dirichlet": d, "mesh": m}
            else:
                p = config_problem(cfg, seed=args.seed)
            batch, d, m = p["batch"], p["dirichlet"], p["mesh"]
            pl = batch.operator(m.n_nodes)
            pl.ensure_dirichlet(d)
            torch.cuda.synchronize()
            setup = time.perf_counter() - t0
            x0 = torch.zeros(m.n_nodes, dtype=torch.float64, device="cuda")
            solve = (lambda: eb.jacobi(batch, d, x0, iters, omega=0.8)) if cfg == 4 else \
                (lambda: eb.pcg(batch, d, x0, iters, tol=tol))
            solve() if cfg != 3 else eb.pcg(batch, d, x0, 5)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            x, h = solve()
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) / 1e3
            its = h.iterations
            nb = m.n_b
            n_n, n_e = m.n_nodes, m.n_elements
            per_it = n_e * (8 * nb * nb + 4 * nb) + (32 if cfg == 4 else 104) * n_n
            # the same with the plan's own id coding instead of the model's 4 B connectivity
            # per slot (one-byte tuple codes / packed deltas / absolute ids)
            flags = pl.info()["loaded"]
            id_b = 1 if flags & 32 else ((4 if nb == 3 else 8) if flags & 4 else 4 * (nb - 1))
            per_it_stored = n_e * (8 * nb * nb + id_b * nb) + (32 if cfg == 4 else 104) * n_n
            out[f"C{cfg}" + ("_permuted" if permuted else "")] = {
                "method": "jacobi" if cfg == 4 else "pcg", "iterations": its,
                "it_per_s": its / t, "ms_per_it": t / its * 1e3,
                "hbm_gbs_algorithmic": per_it * its / t / 1e9,
                "frac_of_peak": per_it * its / t / 1e9 / float(peaks["hbm_gbs"]),
                "id_bytes_per_slot": id_b,
                "frac_of_peak_stored": per_it_stored * its / t / 1e9 / float(peaks["hbm_gbs"]),
                "final_rel_residual": float(h.residual_norms[-1] / h.residual_norms[0]),
                "n_nodes": n_n, "n_elements": n_e, "setup_s": setup}
            if cfg in (4, 5) and not permuted and getattr(args, "emulate", True):
                try:
                    out[f"C{cfg}"]["emulated_8_slabs"] = emulated_slabs(
                        batch, d, m, cfg, iters, t, h.residual_norms)
                except Exception as e:  # noqa: BLE001
                    out[f"C{cfg}"]["emulated_8_slabs"] = {"error": f"{type(e).__name__}: {e}"}
            del p, batch, pl, x
            torch.cuda.empty_cache()
        except Exception as e:  # report, never kill the headline line
            out[f"C{cfg}" + ("_permuted" if permuted else "")] = {
                "error": f"{type(e).__name__}: {e}"}
    try:  # C1 (the reference's CPU-scale case): JPCG to 1e-8, three launches per
        # iteration vs the whole loop as one cooperative kernel (pcg(..., fused=True))
        p = config_problem(1, seed=args.seed)
        batch, d, m = p["batch"], p["dirichlet"], p["mesh"]
        x0 = torch.zeros(m.n_nodes, dtype=torch.float64, device="cuda")
        c1 = {"method": "pcg", "n_nodes": m.n_nodes, "n_elements": m.n_elements}
        for fused in (False, True):
            eb.pcg(batch, d, x0, 10000, tol=1e-8, fused=fused)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _, h = eb.pcg(batch, d, x0, 10000, tol=1e-8, fused=fused)
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) / 1e3
            c1["fused_kernel" if fused else "launch_loop"] = {
                "iterations": h.iterations, "it_per_s": h.iterations / t,
                "us_per_it": t / h.iterations * 1e6, "solve_ms": t * 1e3}
        c1["note"] = ("latency-bound (1.1 MB per iteration): no roofline claim; fused_kernel = "
                      "the whole solve in one thread-block cluster (k_pcg_cluster: slot rows and "
                      "p in shared memory, DSMEM broadcasts, cluster barriers)")
        out["C1"] = c1
    except Exception as e:  # noqa: BLE001
        out["C1"] = {"error": f"{type(e).__name__}: {e}"}
    return out


def paper_experiment():
    """The paper's one published timing: level-10
    unit square (1,050,625 nodes, 2,097,152 triangles): K_e and M_e assembly ~5 s each,
    124 element-based iterations ~50 s (MATLAB, hardware unstated).  Same workload here:
    fused assembly of K_e, M_e, A_e, b_e and 124 Richardson / Chebyshev iterations."""
    import torch

    import paper_1911_03973_b200 as eb
    m = eb.build_unit_square_mesh(10)
    d = eb.constant_dirichlet(m, 1.0)
    eb.build_element_batch(m, nu=0.0)  # warm (plan caches, kernels)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    batch = eb.build_element_batch(m, nu=0.0)
    torch.cuda.synchronize()
    t_asm = time.perf_counter() - t0
    bounds = eb.model_eigen_bounds(2**10 + 1)
    x0 = torch.ones(m.n_nodes, dtype=torch.float64, device="cuda")
    out = {"nodes": m.n_nodes, "elements": m.n_elements,
           "assembly_s": t_asm, "paper_assembly_s": "~5 (K_e) + ~5 (M_e)"}
    for name, run in (("richardson", lambda: eb.richardson(batch, d, x0, bounds, 124)),
                      ("cheb2_N32", lambda: eb.chebyshev2(batch, d, x0, bounds, 32, 124)),
                      ("cheb3", lambda: eb.chebyshev3(batch, d, x0, bounds, 124))):
        run()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, h = run()
        torch.cuda.synchronize()
        out[f"{name}_124_iterations_s"] = time.perf_counter() - t0
    out["paper_124_iterations_s"] = "~50"
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--size", type=int, default=None, help="override the C2 level")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--extra", action=argparse.BooleanOptionalAction, default=True,
                    help="also time the C3/C4/C5 solvers (default on; --no-extra to skip)")
    ap.add_argument("--solver-configs", type=int, nargs="*", default=[3, 4, 5])
    ap.add_argument("--emulate", action=argparse.BooleanOptionalAction, default=True,
                    help="C4 / C5 on 8 element slabs emulated on this GPU (peer transport)")
    ap.add_argument("--c4-size", type=int, default=None, help="override the C4 level (tests)")
    ap.add_argument("--c5-size", type=int, default=None, help="override the C5 N (tests)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
