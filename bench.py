"""Benchmark of the B200 PoisFFT solve path (driver contract: one JSON line on rank 0).

Workload (N=1): BASELINE.json config c3 -- 512^3 fp64, staggered Neumann on all
axes (DCT-II/III), FD2 eigenvalues, unit cube; the config the north-star's
">= 60 % of HBM roofline" target is quoted on.  A "step" is one full solve of
one 512^3 field resident in HBM (1 GiB in, 1 GiB out; larger than the 126 MB L2,
so no explicit flush is needed between steps).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c3]

--impl reference times the reference's own CPU solve on the host cores: the
unmodified reference package installed in baseline/_ref (its SolverPlan built
once, then SolverPlan.solve per step, threads = all cores; one extra
single-thread solve is reported as t1), falling back to the oracle port when
baseline/_ref is absent.  Under torchrun (N > 1) the ranks solve ONE global grid together:
slab decomposition along axis 0, two NCCL all-to-alls per solve (strong
scaling), reported against both the HBM and the NVLink rooflines.
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
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "Poisson solves/s & Gpoints/s (512³–2048³); % HBM/NVLink roofline at 1/2/4/8 GPU"
WORKLOADS = {
    "c3": "c3: 512^3 fp64 staggered-Neumann FD2 (DCT-II/III all axes), unit cube",
    "c1": "c1: 64^3 fp64 periodic pseudo-spectral, L=2pi",
    "c2": "c2: 4096^2 fp64 staggered-Dirichlet FD2 (DST-II/III)",
    "c4": "c4: 1024x1024x512 fp64 periodic x,y + staggered-Neumann z, FD2",
    "c5": "c5: 2048^3 fp32 periodic pseudo-spectral, L=2pi",
}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# BASELINE.json configs: per-axis (n, length, bc, grid kind), approximation, precision
TWO_PI = 2.0 * np.pi
BENCH_CONFIGS = {
    "c1": ([(64, TWO_PI, "periodic", "regular")] * 3, "spectral", "double"),
    "c2": ([(4096, 1.0, "dirichlet", "staggered")] * 2, "fd2", "double"),
    "c3": ([(512, 1.0, "neumann", "staggered")] * 3, "fd2", "double"),
    "c4": ([(1024, TWO_PI, "periodic", "regular"), (1024, TWO_PI, "periodic", "regular"),
            (512, 2.0, "neumann", "staggered")], "fd2", "double"),
    "c5": ([(2048, TWO_PI, "periodic", "regular")] * 3, "spectral", "single"),
}
# c5's reference solve needs ~270 GB of host RAM (dense _inv_lam + complex work arrays):
# its CPU baseline runs on the labelled 1024^3 fp32 proxy
CPU_PROXY = {"c5": 2}


def config_axes(name, scale=1):
    axes, approx, precision = BENCH_CONFIGS[name]
    return [(n // scale, length, bc, kind) for n, length, bc, kind in axes], approx, precision


def build_config(mod, name, scale=1):
    """SolverConfig of the named workload from a package with the reference's API
    (ours or the reference itself)."""
    axes, approx, precision = config_axes(name, scale)
    grids = tuple(mod.GridSpec(n, length, mod.BoundaryCondition(bc), mod.GridKind(kind)) for n, length, bc, kind in axes)
    return mod.SolverConfig(grids, mod.Approximation(approx), precision)


def make_config(name):
    import paper_1409_8116_b200 as fp

    return build_config(fp, name), None


def host_rhs(name, config, seed=0):
    """Seeded host RHS with the distribution BASELINE.json names."""
    rng = np.random.default_rng(seed)
    shape = config.shape
    if name == "c2":
        x = config.grids[0].points()
        y = config.grids[1].points()
        return rng.standard_normal(shape) + np.sin(np.pi * x)[:, None] * np.sin(np.pi * y)[None, :]
    if name == "c4":
        dx, dy, dz = (g.dx for g in config.grids)
        u = rng.standard_normal(shape)
        v = rng.standard_normal(shape)
        w = rng.standard_normal(shape[:2] + (shape[2] + 1,))
        w[..., 0] = 0.0
        w[..., -1] = 0.0
        return (np.roll(u, -1, 0) - u) / dx + (np.roll(v, -1, 1) - v) / dy + (w[..., 1:] - w[..., :-1]) / dz
    if config.precision == "single":
        r = rng.standard_normal(shape, dtype=np.float32)
        r -= np.float32(r.astype(np.float64).mean())
        return r
    r = rng.standard_normal(shape)
    return r - r.mean()


def load_reference():
    """The unmodified reference package installed in baseline/_ref (pip --target,
    DESIGN.md section 5); None when it is not there."""
    ref_dir = ROOT / "baseline" / "_ref"
    if not (ref_dir / "fastpoisson" / "__init__.py").exists():
        return None
    sys.path.insert(0, str(ref_dir))
    try:
        import fastpoisson
    except Exception:  # pragma: no cover
        return None
    finally:
        sys.path.remove(str(ref_dir))
    return fastpoisson


class _PortPlan:
    """Fallback when baseline/_ref is absent: the oracle port with its plan-time
    arrays built once (the reference's SolverPlan.__init__, solver.py:136-181)."""

    def __init__(self, name, scale, threads):
        from oracle import fastpoisson_oracle as orc

        self._orc = orc
        self.case = orc.config_case(name, scale)
        self.threads = threads
        self.plan = orc.OraclePlan(self.case, workers=threads)

    def solve(self, rhs):
        return self.plan.solve(rhs)


def reference_plan(name, threads, scale=1):
    """(plan, rhs, kind, label): the reference's own SolverPlan when installed, else the port."""
    ref = load_reference()
    if ref is not None:
        config = build_config(ref, name, scale)
        t0 = time.perf_counter()
        plan = ref.SolverPlan(config, threads=threads)
        plan_s = time.perf_counter() - t0
        return plan, host_rhs(name, config), "reference", plan_s, "fastpoisson.SolverPlan.solve (baseline/_ref, unmodified)"
    import paper_1409_8116_b200 as fp

    config = build_config(fp, name, scale)
    t0 = time.perf_counter()
    plan = _PortPlan(name, scale, threads)
    plan_s = time.perf_counter() - t0
    return plan, host_rhs(name, config), "port", plan_s, "oracle port of the reference algorithm (plan-time arrays built once)"


def time_reference(name, threads, reps, warmup, seconds_cap=None, scale=1):
    plan, rhs, kind, plan_s, label = reference_plan(name, threads, scale)
    for _ in range(warmup):
        plan.solve(rhs)
    times = []
    t_start = time.perf_counter()
    while len(times) < reps:
        t0 = time.perf_counter()
        plan.solve(rhs)
        times.append(time.perf_counter() - t0)
        if seconds_cap is not None and time.perf_counter() - t_start > seconds_cap:
            break
    return {"times": times, "kind": kind, "plan_s": plan_s, "label": label, "shape": tuple(rhs.shape)}


# ------------------------------------------------------------------------------------------
def run_reference(args, ws, rank):
    """CPU reference arm: the reference package's own SolverPlan.solve (plan built once,
    outside the timed steps) on all host cores of rank 0; other ranks exit without work."""
    if rank != 0:
        return
    cores = len(os.sched_getaffinity(0))
    scale = CPU_PROXY.get(args.config, 1)
    r = time_reference(args.config, cores, args.steps, args.warmup, scale=scale)
    dt = sum(r["times"])
    value = len(r["times"]) / dt
    n_pts = int(np.prod(r["shape"]))
    proxy = f" (labelled proxy {r['shape']}: the full grid needs ~270 GB host RAM)" if scale != 1 else ""
    t1 = None
    if not args.no_t1:
        r1 = time_reference(args.config, 1, 1, 0, scale=scale)
        t1 = {"value": 1.0 / statistics.median(r1["times"]), "unit": "solves/s", "cores": 1,
              "sample": f"{len(r1['times'])} solve(s), threads=1, after the T=all run warmed the process"}
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": ws,
        "steps": len(r["times"]), "warmup": args.warmup, "ms_per_step": dt / len(r["times"]) * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32" if BENCH_CONFIGS[args.config][2] == "single" else "f64",
        "data": "synthetic (seeded N(0,1), BASELINE.json distributions)",
        "config": {"workload": WORKLOADS[args.config] + proxy, "grid": list(r["shape"])},
        "gpoints_per_s": value * n_pts / 1e9,
        "cpu_baseline": {"value": value, "unit": "solves/s", "cores": cores, "kind": r["kind"],
                         "sample": f"{len(r['times'])} full solves after {args.warmup} warm-up, plan built once "
                                   f"({r['plan_s']:.2f} s, untimed); {r['label']}, threads={cores}{proxy}",
                         "plan_s": r["plan_s"], "median_s": statistics.median(r["times"]), "t1": t1},
        "e2e": {"value": value, "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_sample(name, seconds_cap=30.0, with_t1=True):
    """Bounded CPU sample for the GPU line: the reference's SolverPlan.solve on all
    host cores (median of <= 3 after 1 warm-up), plus one single-thread solve."""
    cores = len(os.sched_getaffinity(0))
    scale = CPU_PROXY.get(name, 1)
    r = time_reference(name, cores, 3, 1, seconds_cap=seconds_cap, scale=scale)
    med = statistics.median(r["times"])
    proxy = f"; labelled proxy grid {r['shape']} (full grid needs ~270 GB host RAM)" if scale != 1 else ""
    out = {"value": 1.0 / med, "unit": "solves/s", "cores": cores, "kind": r["kind"],
           "sample": f"median of {len(r['times'])} full {name} solves after 1 warm-up, plan built once "
                     f"({r['plan_s']:.2f} s, untimed); {r['label']}, threads={cores}{proxy}",
           "grid": list(r["shape"])}
    if scale != 1:
        out["gpoints_per_s"] = float(np.prod(r["shape"])) / med / 1e9
    if with_t1:
        r1 = time_reference(name, 1, 1, 0, scale=scale)
        out["t1"] = {"value": 1.0 / r1["times"][0], "unit": "solves/s", "cores": 1,
                     "sample": "one solve, threads=1"}
    return out


def measure_pcie(dev, nbytes=1 << 30, reps=5):
    """Pinned host <-> device copy rates (GB/s): each direction alone and both at once
    on two streams (PCIe is full duplex) -- the roofline of the e2e number, so the best
    of `reps` timed copies (a roofline is the best the link did, not its average)."""
    import torch

    h_in = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    h_out = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d_a = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    d_b = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    cur = torch.cuda.current_stream(dev)

    def timed(fn):
        fn()
        torch.cuda.synchronize(dev)
        best = None
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(cur)
            fn()
            e1.record(cur)
            torch.cuda.synchronize(dev)
            t = e0.elapsed_time(e1) * 1e-3
            best = t if best is None else min(best, t)
        return best

    def both():
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d_a.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_b, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    t_in = timed(lambda: d_a.copy_(h_in, non_blocking=True))
    t_out = timed(lambda: h_out.copy_(d_b, non_blocking=True))
    t_both = timed(both)
    del h_in, h_out, d_a, d_b
    return {"h2d_gbs": nbytes / t_in / 1e9, "d2h_gbs": nbytes / t_out / 1e9,
            "duplex_gbs_each_way": nbytes / t_both / 1e9,
            "how": f"pinned {nbytes >> 20} MiB copies, CUDA events, best of {reps}; duplex = both directions "
                   "at once on two streams"}


def measure_e2e(plan, rhs, shape, tdt, n_pts, s, args, ws, dist, dev):
    """Same metric through the public API with pinned host buffers: every step
    copies its rhs host->device and its solution device->host.  Headline: the
    streaming call SolverPlan.solve_batch (copies of neighbouring steps overlap
    the solve, PCIe full duplex); also reported: one synchronous solve() per step."""
    import torch

    rhs_host = torch.empty(shape, dtype=tdt, pin_memory=True)
    rhs_host.copy_(rhs)
    outs = [torch.empty(shape, dtype=tdt, pin_memory=True) for _ in range(2)]
    rhs_np = rhs_host.numpy()
    out_np = [o.numpy() for o in outs]
    # 40 streamed solves (>= K): the pipeline's fill (first H2D) and drain (last D2H) are one
    # transfer each, ~2.5 % of a 40-solve batch instead of ~5 % of a 20-solve one
    e2e_steps = max(40, min(args.steps, 80))
    plan.solve(rhs_np, out=out_np[0])  # warm the path
    plan.solve_batch([rhs_np] * 2, [out_np[0], out_np[1]])
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    plan.solve_batch([rhs_np] * e2e_steps, [out_np[i & 1] for i in range(e2e_steps)])
    batch_dt = time.perf_counter() - t0
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        plan.solve(rhs_np, out=out_np[0])
    single_dt = time.perf_counter() - t0
    if dist is not None:
        tt = torch.tensor([batch_dt, single_dt], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        batch_dt, single_dt = float(tt[0]), float(tt[1])
    pcie = measure_pcie(dev)
    # PCIe roofline of a streamed solve: H2D and D2H overlap (full duplex), so a step
    # costs at least max(bytes_in, bytes_out) / duplex rate
    bound = max(n_pts * s, n_pts * s + 16) / (pcie["duplex_gbs_each_way"] * 1e9)
    value = ws * e2e_steps / batch_dt
    pcie["roofline_solves_per_s"] = ws / bound
    pcie["frac"] = value / pcie["roofline_solves_per_s"]
    return {"value": value, "unit": "solves/s", "h2d_bytes_per_step": n_pts * s,
            "d2h_bytes_per_step": n_pts * s + 16, "pcie": pcie, "pcie_frac": pcie["frac"],
            "path": "SolverPlan.solve_batch(pinned numpy rhs per step -> pinned numpy out per step)",
            "single_call": {"value": ws * e2e_steps / single_dt, "unit": "solves/s",
                            "path": "SolverPlan.solve(pinned numpy rhs, out=pinned numpy) once per step"}}


def run_dist(args, ws, rank, local):
    """N > 1: ONE global grid split over the ranks (slab decomposition, NCCL all-to-all)."""
    import torch
    import torch.distributed as dist

    import paper_1409_8116_b200 as fp  # noqa: F401
    from paper_1409_8116_b200 import _device as dv
    from paper_1409_8116_b200.distributed import DistributedSolverPlan

    # NCCL init lines (rank count, transport: NVLink / NVLS) on stderr, away from the JSON line
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    config, case = make_config(args.config)
    plan = DistributedSolverPlan(config, device=dev)
    shape = config.shape
    n_pts = int(np.prod(shape))
    s = config.dtype.itemsize
    tdt = dv.torch_dtype(config.dtype)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    rhs = torch.randn(plan.local_shape, dtype=tdt, device=dev, generator=gen)
    out = torch.empty_like(rhs)
    stream = torch.cuda.current_stream(dev)
    for _ in range(max(args.warmup, 1)):
        plan.solve_async(rhs, out)
    torch.cuda.synchronize(dev)
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    dist.barrier()
    torch.cuda.synchronize(dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record(stream)
    for _ in range(args.steps):
        plan.solve_async(rhs, out)
    ev[1].record(stream)
    torch.cuda.synchronize(dev)
    dist.barrier()
    clocks = sampler.stop()
    tt = torch.tensor([ev[0].elapsed_time(ev[1])], device=dev, dtype=torch.float64)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    elapsed_ms = float(tt.item())
    ms_step = elapsed_ms / args.steps
    # per-phase breakdown (a second, untimed pass: events between the phases and exchanges)
    ph_ev = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(args.steps)]
    for k in range(args.steps):
        plan.solve_async(rhs, out, events=ph_ev[k])
    torch.cuda.synchronize(dev)
    ph = torch.tensor([[e[j].elapsed_time(e[j + 1]) for j in range(5)] for e in ph_ev], device=dev,
                      dtype=torch.float64).mean(dim=0)
    dist.all_reduce(ph, op=dist.ReduceOp.MAX)
    phase_ms = [float(x) for x in ph.tolist()]
    value = args.steps / (elapsed_ms * 1e-3)          # solves/s of the one global grid
    hbm_peak, peak_src = peaks()
    import ctypes
    from paper_1409_8116_b200 import _native as nat

    pinfo = nat.FpPlanInfo()
    nat.check(nat.load().fp_plan_info_get(plan.backend._handle, ctypes.byref(pinfo)))
    launches = int(pinfo.num_passes) * args.steps   # this rank's kernels (NCCL kernels not counted)
    b_alg = (2 * len(shape) - 1) * 2 * n_pts * s
    xbytes = int(plan.info.exchange_bytes)
    nvl_bytes = 2 * xbytes * (ws - 1) / ws             # sent per GPU per solve (two all-to-alls)
    nvl_peak = 900.0
    roofline = {
        "bound": "hbm+nvlink",
        "achieved": b_alg / ws / (ms_step * 1e-3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
        "frac": b_alg / ws / (ms_step * 1e-3) / 1e9 / hbm_peak, "traffic": None,
        "kernel": "whole distributed solve per GPU (B_alg / P)", "peak_source": peak_src,
        "nvlink": {"bytes_per_gpu_per_solve": nvl_bytes, "achieved": nvl_bytes / (ms_step * 1e-3) / 1e9,
                   "peak": nvl_peak, "unit": "GB/s", "frac": nvl_bytes / (ms_step * 1e-3) / 1e9 / nvl_peak,
                   "peak_source": "nominal NVLink 5 per direction per GPU"},
    }
    # phases (max over ranks of the per-rank means): local forward passes, exchange, MID,
    # exchange back, local inverse passes -- the compute phases against HBM, the exchanges
    # against NVLink (each moves (P-1)/P of the exchange buffer per direction)
    n_local = (len(shape) - 1)
    x_one = xbytes * (ws - 1) / ws
    loc_bytes = 2 * n_pts * s / ws
    roofline["phases"] = {
        "names": ["forward (local axes)", "all-to-all", "MID (axis 0)", "all-to-all back", "backward (local axes)"],
        "ms": phase_ms,
        "hbm_frac": [n_local * loc_bytes / (phase_ms[0] * 1e-3) / 1e9 / hbm_peak, None,
                     loc_bytes / (phase_ms[2] * 1e-3) / 1e9 / hbm_peak, None,
                     n_local * loc_bytes / (phase_ms[4] * 1e-3) / 1e9 / hbm_peak],
        "nvlink_frac": [None, x_one / (phase_ms[1] * 1e-3) / 1e9 / nvl_peak, None,
                        x_one / (phase_ms[3] * 1e-3) / 1e9 / nvl_peak, None],
        "how": "CUDA events on the compute stream between the phases of K extra solves; the exchanges "
               "are torch.distributed.all_to_all_single (NCCL), ordered on that stream",
    }
    # e2e: each rank's slab from pinned host memory, solve, slab back (public distributed API)
    e2e = None
    if not args.no_e2e:
        host_in = torch.empty(plan.local_shape, dtype=tdt, pin_memory=True)
        host_in.copy_(rhs)
        host_out = torch.empty(plan.local_shape, dtype=tdt, pin_memory=True)
        e2e_steps = max(1, min(args.steps, 10))
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            d_in = host_in.to(dev, non_blocking=True)
            o, rep = plan.solve(d_in)
            host_out.copy_(o)
        e2e_dt = time.perf_counter() - t0
        tt = torch.tensor([e2e_dt], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_dt = float(tt.item())
        e2e = {"value": e2e_steps / e2e_dt, "unit": "solves/s",
               "h2d_bytes_per_step": n_pts * s, "d2h_bytes_per_step": n_pts * s,
               "path": "DistributedSolverPlan.solve(slab from pinned host) + slab D2H, every rank"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": config.dtype.name.replace("float", "f"),
            "data": "synthetic (seeded N(0,1) slabs generated on device)",
            "config": {"workload": WORKLOADS[args.config], "grid": list(shape),
                       "parallelism": f"slab decomposition along axis 0 over {ws} GPUs, NCCL all-to-all",
                       "l2": "inputs larger than L2; no flush"},
            "gpoints_per_s": value * n_pts / 1e9,
            "roofline": roofline,
            "cpu_baseline": None,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def run_ours(args, ws, rank, local):
    import ctypes

    import torch

    import paper_1409_8116_b200 as fp
    from paper_1409_8116_b200 import _native as nat
    from paper_1409_8116_b200 import _device as dv

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    config, case = make_config(args.config)
    plan = fp.SolverPlan(config, device=dev)
    lib = plan._lib
    shape = config.shape
    n_pts = int(np.prod(shape))
    s = config.dtype.itemsize
    tdt = dv.torch_dtype(config.dtype)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    rhs = torch.randn(shape, dtype=tdt, device=dev, generator=gen)
    rhs -= rhs.mean()
    out = torch.empty_like(rhs)
    ws_bytes = plan.workspace_bytes(out_dense=True)
    work = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
    info = torch.zeros(16, dtype=torch.uint8, device=dev)
    npass = plan.num_passes
    stream = torch.cuda.current_stream(dev)
    sh = stream.cuda_stream

    def make_events(k):
        arr = (ctypes.c_void_p * k)()
        for i in range(k):
            h = ctypes.c_void_p()
            nat.check(lib.fp_event_create_on(local, ctypes.byref(h)))
            arr[i] = h
        return arr

    rs = nat.strides_array(rhs.stride())
    os_ = nat.strides_array(out.stride())
    rdt = dv.fp_dtype_of_torch(tdt)

    def step(pass_ev=None):
        nat.check(lib.fp_solve_ex(plan._handle, rhs.data_ptr(), rdt, rs, out.data_ptr(), os_, work.data_ptr(),
                                  ws_bytes, sh, info.data_ptr(), None, pass_ev))

    for _ in range(max(args.warmup, 1)):
        step()
    torch.cuda.synchronize(dev)
    pass_events = [make_events(npass + 1) for _ in range(args.steps)]
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize(dev)
    # small grids are launch-bound: one CUDA-graph replay per solve (SolverPlan.capture)
    use_graph = n_pts <= (1 << 22)
    if use_graph:
        cap = plan.capture(rhs, out)
        for _ in range(max(args.warmup, 1)):
            cap.replay()
        torch.cuda.synchronize(dev)
        timed = cap.replay
    else:
        timed = step
    l2_resident = n_pts * s < (128 << 20)
    if l2_resident:
        # the field fits L2: flush it (write 256 MiB) before every step and time
        # each solve alone between its own events
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        for k in range(args.steps):
            flush.zero_()
            evs[k][0].record(stream)
            timed()
            evs[k][1].record(stream)
        torch.cuda.synchronize(dev)
        elapsed_ms = sum(a.elapsed_time(b) for a, b in evs)
    else:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for k in range(args.steps):
            timed()
        t_end.record(stream)
        torch.cuda.synchronize(dev)
        elapsed_ms = t_start.elapsed_time(t_end)
    if dist is not None:
        dist.barrier()
    clocks = sampler.stop()
    # per-kernel durations: a second pass of K solves with events between the kernels
    # (kept out of the timed region: on 64^3 the event records cost more than a kernel)
    for k in range(args.steps):
        step(pass_events[k])
    torch.cuda.synchronize(dev)
    if dist is not None:
        tt = torch.tensor([elapsed_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        elapsed_ms = float(tt.item())
    # per-kernel durations (CUDA events on the launching stream)
    per_pass = np.zeros((args.steps, npass))
    ms = ctypes.c_float()
    for k in range(args.steps):
        for i in range(npass):
            nat.check(lib.fp_event_elapsed_ms(pass_events[k][i], pass_events[k][i + 1], ctypes.byref(ms)))
            per_pass[k, i] = ms.value
    for arr in pass_events:
        for i in range(npass + 1):
            lib.fp_event_destroy(arr[i])
    # (the median over the K steps: a single slow step -- clock ramp, another tenant -- moves a mean)
    avg_pass = np.median(per_pass, axis=0)
    hbm_peak, peak_src = peaks()
    pass_bytes = 2 * n_pts * s  # each pass reads and writes the field once
    top = int(np.argmax(avg_pass))
    ms_step = elapsed_ms / args.steps
    value = ws * args.steps / (elapsed_ms * 1e-3)
    b_alg = (2 * len(shape) - 1) * 2 * n_pts * s
    traffic = None
    prof = ROOT / "profiles" / "ncu_traffic.json"
    if prof.exists():
        try:
            tj = json.loads(prof.read_text())
            traffic = tj.get(args.config, {}).get(str(top))
        except Exception:
            traffic = None
    roofline = {
        "bound": "hbm",
        "achieved": pass_bytes / (avg_pass[top] * 1e-3) / 1e9,
        "peak": hbm_peak,
        "unit": "GB/s",
        "frac": pass_bytes / (avg_pass[top] * 1e-3) / 1e9 / hbm_peak,
        "traffic": traffic,
        "kernel": f"pass {top} of {npass}" + (
            f" (MID: forward transform, eigenvalue divide, inverse transform along axis {int(plan._info.middle_axis)})"
            if top == npass // 2 and npass % 2 == 1 else ""),
        "algorithmic_bytes_per_launch": pass_bytes,
        "peak_source": peak_src,
        "per_pass_ms": [round(float(x), 4) for x in avg_pass],
        "per_pass_stat": "median over the timed step count, CUDA events between the kernels (untimed second pass)",
        "solve": {"algorithmic_bytes": b_alg, "achieved": b_alg / (ms_step * 1e-3) / 1e9,
                  "frac": b_alg / (ms_step * 1e-3) / 1e9 / hbm_peak},
    }
    # e2e through the public API with pinned host buffers (H2D + solve + D2H each step)
    e2e = None
    if not args.no_e2e:
        e2e = measure_e2e(plan, rhs, shape, tdt, n_pts, s, args, ws, dist, dev)
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_sample(args.config)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": config.dtype.name.replace("float", "f"),
            "data": "synthetic (seeded N(0,1) field with its mean removed, generated on device)",
            "config": {"workload": WORKLOADS[args.config], "grid": list(shape),
                       "parallelism": "replicas" if ws > 1 else "single-gpu",
                       "l2": ("inputs (%.2f GiB/field) larger than L2; no flush" % (n_pts * s / 2**30))
                       if not l2_resident else
                       "field (%.1f MiB) smaller than L2: 256 MiB flush before every step, each solve timed alone"
                       % (n_pts * s / 2**20),
                       "launch": "cuda-graph replay of one solve per step" if use_graph else "one fp_solve call per step"},
            "gpoints_per_s": value * n_pts / 1e9,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": npass * args.steps,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-t1", action="store_true", help="reference arm: skip the single-thread timing")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    ws, rank, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # launched without torchrun: start the N ranks ourselves (one process per GPU)
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    if args.gpus != ws:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    if ws > 1:
        run_dist(args, ws, rank, local)
        return
    run_ours(args, ws, rank, local)


if __name__ == "__main__":
    main()
