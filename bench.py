#!/usr/bin/env python
"""Benchmark of the spectral-coarse-solver Parareal hot path (arXiv 2508.08873).

One step = the whole hot path on one batch of synthetic input:
    pr_build_coarse  (rSVD of F_n' on every interval: 2*l batched fine solves
                      per interval + CholeskyQR + Jacobi SVD + lift)
  + pr_parareal      (offsets b_n, initialisation, K iterations of batched fine
                      solves + reduced coarse sweep + update norms)
Metric (BASELINE.json): fine-solve DOF-steps/s of the step, plus the rSVD build
and Parareal wall times.  Default workload: C4 (BASELINE.json configs[3], the
largest 1D configuration; DESIGN.md "Benchmark workload" says why).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl reference]

Multi-GPU (torchrun, one rank per GPU): intervals are sharded over the ranks.
The build needs no communication; Parareal exchanges only the interval-
boundary blocks (P2P) and the k-dimensional sweep data (all-gather) --
paper_2508_08873_b200/parallel.py.  Strong scaling: the config is fixed.
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
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "fine-solve DOF-steps/s (batched implicit Euler) + rSVD build & Parareal wall time"
L2_BYTES = 126 * 2 ** 20


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _ncu_traffic(cfg_name):
    """dram bytes per stepper launch from the committed ncu --set full capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "stepper_traffic.json")) as f:
            d = json.load(f)
        return d.get(cfg_name)
    except Exception:
        return None


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------- workload
class Workload:
    """Device-resident inputs of one rank and the step function."""

    def __init__(self, cfg, rank: int, world: int, dev):
        import torch
        from paper_2508_08873_b200 import Operator, SourceTerm
        from workloads import generators as G
        self.cfg, self.rank, self.world, self.dev = cfg, rank, world, dev
        # interval shard: the build and the Parareal fine solves of intervals q0..q0+nq-1
        self.q0, self.nq = _shard(cfg.N, rank, world)
        self.s0, self.ns = 0, cfg.nsrc
        u0 = G.initial_value(cfg)
        if cfg.dim == 1 and cfg.problem.startswith("exp2"):
            # the time-dependent pencil of Exp 2
            from workloads import exp2
            L, rs, M = exp2.step_matrices(cfg.problem, cfg.n, cfg.T, cfg.N * cfg.m)
            self.host = dict(pencil=(L, rs, M))
            space, time_, amp = G.source_1d(cfg)
            self.host.update(space=space, time=time_, amp=amp[self.s0:self.s0 + self.ns])
            self.host["u0"] = np.ascontiguousarray(np.stack([u0] * self.ns).T)
            self.op = Operator.pencil(*L, cfg.dt, lrowsum=rs, mass=M)
            self.src = SourceTerm.sep1d(space, time_, self.host["amp"])
            self.U = torch.empty((cfg.n, (self.nq + 1) * self.ns), dtype=torch.float64, device=dev)
        elif cfg.dim == 1:
            self.host = dict(op=G.operator_1d(cfg), sums=G.operator_1d_sums(cfg))
            space, time_, amp = G.source_1d(cfg)
            self.host.update(space=space, time=time_, amp=amp[self.s0:self.s0 + self.ns])
            self.host["u0"] = np.ascontiguousarray(np.stack([u0] * self.ns).T)   # (n, ns)
            rs, cs = self.host["sums"]
            self.op = Operator.tridiag(*self.host["op"], cfg.dt, rowsum=rs, colsum=cs)
            self.src = SourceTerm.sep1d(space, time_, self.host["amp"])
            self.U = torch.empty((cfg.n, (self.nq + 1) * self.ns), dtype=torch.float64, device=dev)
        else:
            gx, gy = G.source_2d(cfg)
            P = cfg.n + 1
            self.host = dict(gx=G.pad1d_last(gx), gy=G.pad1d_last(gy),
                             u0=G.pad2d(u0).reshape(1, P * P))
            self.op = Operator.sep2d(cfg.n, cfg.dt)
            self.src = SourceTerm.bump2d(self.host["gx"], self.host["gy"])
            self.U = torch.empty(((self.nq + 1) * self.ns, P * P), dtype=torch.float64, device=dev)
        self.u0 = torch.tensor(self.host["u0"], dtype=torch.float64, device=dev)
        # interval-sharded runs: one pr_comm (NCCL) over the torch.distributed group
        self.comm = None
        if world > 1:
            from paper_2508_08873_b200.parallel import nccl_comm
            self.comm = nccl_comm()

    def dof_steps(self) -> float:
        """Fine-solve DOF-steps this rank performs per step: the rSVD build
        (2 l solves per interval), the offsets b_n (one solve per interval and
        source term when there are more sources than terms -- libpr combines
        them by linearity, reading R-SRC -- else one per source) and
        K iterations of one solve per interval and source."""
        c = self.cfg
        build = self.nq * 2 * c.l * c.n_dof * c.m
        nb = self.ns
        if c.dim == 1:
            R = self.host["time"].shape[0]
            nb = min(self.ns, R)
        par = (c.K * self.ns + nb) * self.nq * c.n_dof * c.m
        return float(build + par)

    def step(self, events=None, op=None, src=None, u0=None):
        """rSVD build of the own intervals + Parareal, through the C ABI only
        (N GPUs: pr_build_coarse / pr_parareal with the NCCL pr_comm; libpr
        moves the interval-boundary data itself)."""
        from paper_2508_08873_b200 import Coarse, parareal
        c = self.cfg
        op = op or self.op
        src = src or self.src
        u0 = self.u0 if u0 is None else u0
        G = Coarse.build(op, c.N, c.m, c.k, c.p, c.seed_omega, comm=self.comm)
        if events is not None:
            events.append(_event())
        upd, bn = parareal(G, op, u0 if self.rank == 0 else None, src, c.K, self.U, nsrc=self.ns)
        self.last_upd = upd
        G.close()
        return self.U


def _fp64_peaks(dev):
    """Measured FP64 ceilings of this pool's B200 (profiles/fp64_peaks.json,
    written by tools/fp64_peaks.py: DFMA and DMMA microkernels and cuBLAS
    DGEMM 8192^3); MEASURED_PEAKS.json carries no FP64 figure.  Falls back to
    a live DGEMM measurement and the unit-count DFMA figure, saying so."""
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peaks.json")) as f:
            d = json.load(f)
        return {"dfma": float(d["dfma_tflops"]), "dgemm": float(d["dgemm_tflops"]),
                "dmma": float(d.get("dmma_m8n8k4_tflops", 0.0)),
                "source": "measured (profiles/fp64_peaks.json, tools/fp64_peaks.py)"}
    except Exception:
        import torch
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        return {"dfma": sms * 64 * 2 * 1965e6 / 1e12, "dgemm": _fp64_peak(dev), "dmma": 0.0,
                "source": "fallback: DFMA from unit counts x 1965 MHz, DGEMM measured live"}


def _fp64_peak(dev):
    """cuBLAS DGEMM 8192^3 measured live (best of 5, CUDA events)."""
    import torch
    n = 8192
    a = torch.randn((n, n), dtype=torch.float64, device=dev)
    b = torch.randn((n, n), dtype=torch.float64, device=dev)
    torch.matmul(a, b)
    best = 0.0
    for _ in range(5):
        e0, e1 = _event(), None
        torch.matmul(a, b)
        e1 = _event()
        torch.cuda.synchronize()
        best = max(best, 2.0 * n ** 3 / (e0.elapsed_time(e1) / 1e3) / 1e12)
    del a, b
    return best


def _shard(total: int, rank: int, world: int):
    base, rem = divmod(total, world)
    start = rank * base + min(rank, rem)
    return start, base + (1 if rank < rem else 0)


def _event():
    import torch
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


# ----------------------------------------------------------- CPU oracle leg
def oracle_sample(cfg):
    """A bounded sample of the same workload on the host cores, through the
    oracle as it stands: the rSVD of one interval (steps 1-6) and (K+1) fine
    solves of that interval for every source (the offset b plus the K
    Parareal fine solves).  Returns (dof_steps, seconds)."""
    from oracle.fine import fine, make_op
    from oracle.rsvd import rsvd_interval
    from workloads import generators as G
    op = make_op(cfg)
    if cfg.dim == 1:
        src = G.source_1d(cfg)
        u0 = np.stack([G.initial_value(cfg)] * cfg.nsrc)
        sidx = np.arange(cfg.nsrc)
    else:
        src = G.source_2d(cfg)
        u0 = G.initial_value(cfg)[None]
        sidx = None
    t0 = time.perf_counter()
    rsvd_interval(op, 1, cfg.k, cfg.p, cfg.seed_omega)
    for _ in range(cfg.K + 1):
        fine(op, 1, u0, "affine", src, sidx)
    dt = time.perf_counter() - t0
    dof = 2 * cfg.l * cfg.n_dof * cfg.m + (cfg.K + 1) * cfg.nsrc * cfg.n_dof * cfg.m
    return float(dof), dt


def _host_info():
    """CPU model (lscpu) and the number of host threads the oracle may use."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.lower().startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "threads_used": _cores()}


def oracle_one_thread(cfg):
    """Per-core rate of the oracle: the rSVD forward solves of one interval
    (l vectors x m steps, the oracle's fine solver as it stands) with one
    thread, in a subprocess with OMP / BLAS pinned to 1 thread."""
    env = dict(os.environ, OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1", MKL_NUM_THREADS="1")
    try:
        out = subprocess.run([sys.executable, os.path.abspath(__file__), "--oracle-1t", "--config", cfg.name],
                             capture_output=True, text=True, timeout=300, env=env).stdout
        return json.loads(out.strip().splitlines()[-1])
    except Exception as e:
        return {"error": str(e)[:200]}


def _oracle_1t_main(cfg):
    from oracle import _clib
    from oracle.fine import fine, make_op
    _clib.build()
    op = make_op(cfg)
    nv = min(cfg.l, 16) if cfg.dim == 2 else cfg.l
    shape = (nv, cfg.n) if cfg.dim == 1 else (nv, cfg.n, cfg.n)
    X = np.random.default_rng(0).standard_normal(shape)
    t0 = time.perf_counter()
    fine(op, 1, X, "linear")
    sec = time.perf_counter() - t0
    dof = float(nv * cfg.n_dof * cfg.m)
    print(json.dumps({"value": dof / sec, "unit": "DOF-steps/s", "threads": 1,
                      "sample": f"{nv} fine solves (F' of interval 1, {cfg.m} steps): {dof:.3g} DOF-steps in {sec:.2f} s"}))


def _cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# --------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sub", action="store_true", help="skip the C3 (2D) sub-record")
    ap.add_argument("--oracle-1t", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()

    from workloads.configs import get
    cfg = get(args.config)
    if args.oracle_1t:
        _oracle_1t_main(cfg)
        return
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    config = {"workload": cfg.name, "dim": cfg.dim, "n": cfg.n, "N": cfg.N, "m": cfg.m, "k": cfg.k,
              "p": cfg.p, "K": cfg.K, "nsrc": cfg.nsrc, "T": cfg.T,
              "l2": "inputs larger than L2: %.2f GB state per stepper phase vs 126 MB L2"
                    % (cfg.n_dof * cfg.N * max(cfg.l, cfg.nsrc) * 8 / 1e9),
              "parallelism": f"intervals sharded over {args.gpus} GPU(s) (P2P halos + all-gather of sweep data)"}

    if args.impl == "reference":
        if rank != 0:
            return
        from oracle import _clib
        _clib.build()
        for _ in range(args.warmup):
            oracle_sample(cfg)
        vals = []
        for _ in range(args.steps):
            dof, sec = oracle_sample(cfg)
            vals.append((dof, sec))
        dof = sum(v[0] for v in vals)
        sec = sum(v[1] for v in vals)
        value = dof / sec
        sample = (f"rSVD of interval 1 + {cfg.K + 1} fine solves of interval 1 x {cfg.nsrc} sources "
                  f"({vals[0][0]:.3g} DOF-steps per step)")
        line = {"metric": METRIC, "value": value, "unit": "DOF-steps/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sec / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded generators, workloads/)", "config": config,
                "impl": "reference",
                "cpu_baseline": {"value": value, "unit": "DOF-steps/s", "cores": _cores(),
                                 "kind": "oracle", "sample": sample, "host": _host_info()},
                "e2e": {"value": value, "unit": "DOF-steps/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    import __graft_entry__
    __graft_entry__.build()
    from paper_2508_08873_b200 import counters, profile
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    # memory plan: the coarse factors U, V of a
    # rank's intervals plus the Parareal state arrays must fit in HBM; C5 (205 GB
    # of factors) does not fit one B200 -- say so instead of failing inside libpr
    q0_, nq_ = _shard(cfg.N, rank, world)
    rows = cfg.n if cfg.dim == 1 else (cfg.n + 1) ** 2
    need = (2.0 * nq_ * rows * cfg.k + 4.0 * (nq_ + 1) * rows * max(cfg.nsrc, 1)) * 8
    free = torch.cuda.mem_get_info(dev)[0]
    if need > 0.95 * free:
        if rank == 0:
            per = 2.0 * cfg.N * rows * cfg.k * 8
            print(json.dumps({"metric": METRIC, "unit": "DOF-steps/s", "n_gpus": world, "config": config,
                              "unavailable": "%s needs %.1f GB of coarse factors + state on each of %d GPU(s) "
                                             "(%.1f GB free); run with --gpus >= %d"
                                             % (cfg.name, need / 1e9, world, free / 1e9,
                                                int(np.ceil(per / (0.8 * free))))}), flush=True)
        return
    wl = Workload(cfg, rank, world, dev)
    peaks = _fp64_peaks(dev)
    sampler = ClockSampler(local_rank)
    sampler.start()
    rec = _timed(wl, args.steps, args.warmup, barrier, world, dev, peaks)
    clocks = sampler.stop()
    value, ms_per_step, dof_total = rec["value"], rec["ms_per_step"], rec["dof_steps_per_step"]
    roofline = rec.pop("roofline")

    # ------------------------------------------------------------- e2e run
    e2e = None
    if not args.no_e2e:
        e2e = _e2e(wl, args.steps, barrier, world)

    # ------------------------------------------- 2D sub-record (C3, 1 GPU)
    sub = None
    if world == 1 and cfg.name != "C3" and not args.no_sub:
        from workloads.configs import get as _get
        c3 = _get("C3")
        del wl
        torch.cuda.empty_cache()
        wl3 = Workload(c3, rank, world, dev)
        sub = {"workload": "C3", "note": "the 2D (FP64 tensor-core) path: BASELINE.json configs[2], "
                                         "same step definition, timed after the headline workload"}
        sub.update(_timed(wl3, args.steps, args.warmup, barrier, world, dev, peaks))
        del wl3

    # --------------------------------------------------------- CPU baseline
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import _clib
        _clib.build()
        dof, sec = oracle_sample(cfg)
        cpu = {"value": dof / sec, "unit": "DOF-steps/s", "cores": _cores(), "kind": "oracle",
               "sample": f"rSVD of interval 1 + {cfg.K + 1} fine solves of interval 1 x "
                         f"{cfg.nsrc} sources ({dof:.3g} DOF-steps, {sec:.1f} s)",
               "host": _host_info(), "one_thread": oracle_one_thread(cfg)}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "DOF-steps/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic (seeded generators, workloads/)",
                "config": config,
                "build_ms": rec["build_ms"], "parareal_ms": rec["parareal_ms"],
                "dof_steps_per_step": dof_total, "phases": rec["phases"],
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": rec["gpu_launches"], "clocks": clocks,
                "fp64_peaks": peaks}
        if sub is not None:
            line["sub"] = sub
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def _timed(wl, steps, warmup, barrier, world, dev, peaks):
    """W untimed steps, then K steps bracketed by barrier + synchronize, max
    over ranks; device time per step, per-phase fine-solve rates (SURVEY §8(d)
    "Definitions") and the roofline of the dominant fine-stepper kernel."""
    import torch
    from paper_2508_08873_b200 import counters, profile
    from paper_2508_08873_b200.api import phase_counters
    cfg = wl.cfg
    for _ in range(warmup):
        wl.step()
    barrier()
    counters(reset=True)
    profile(True)
    barrier()
    ev = [_event()]
    mid = []
    for _ in range(steps):
        wl.step(events=mid)
        ev.append(_event())
    barrier()
    profile(False)
    total_ms = ev[0].elapsed_time(ev[-1])
    build_ms = [ev[i].elapsed_time(mid[i]) for i in range(steps)]
    par_ms = [mid[i].elapsed_time(ev[i + 1]) for i in range(steps)]
    ph = phase_counters(reset=False)
    ctr = counters(reset=True)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    ms_per_step = total_ms / steps
    dof_total = wl.dof_steps() if world == 1 else _sum_dof(wl, world)
    phases = {}
    for name in ("build", "offsets", "iteration"):
        p = ph[name]
        if p["launches"]:
            phases[name] = {"launches_per_step": p["launches"] / steps, "ms_per_step": p["ms"] / steps,
                            "dof_steps_per_s": p["dof_steps"] / (p["ms"] / 1e3) if p["ms"] > 0 else None}
    st_ms = ctr["stepper_ms"] / max(ctr["stepper_launches"], 1)
    st_dof = ctr["stepper_dof_steps"] / max(ctr["stepper_launches"], 1)
    st_fl = ctr["stepper_flops"] / max(ctr["stepper_launches"], 1)
    if cfg.dim == 1 and cfg.problem.startswith("exp2"):
        # K1T (time-dependent pencil): two streaming passes per step over the
        # state (down: read + write, up: read + write): 32 B per DOF-step of HBM
        peak, peak_kind = _peaks()
        achieved = 32.0 * st_dof / (st_ms / 1e3) / 1e9 if st_ms > 0 else None
        roofline = {"kernel": "k_pencil_cta / k_pencil_step (K1T, time-dependent pencil; 32 B per DOF-step of per-step factors)", "bound": "hbm",
                    "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": (achieved / peak) if achieved else None,
                    "traffic": None, "algorithmic_bytes_per_launch": 32.0 * st_dof,
                    "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)"}
    elif cfg.dim == 1 and st_fl > 0:
        # K1P: the state stays on chip for all m steps, so HBM carries only the
        # input and output (16 B per DOF per launch); the bound is the FP64
        # pipe: 5 algorithmic flops per DOF-step (+2R with an R-term source)
        achieved = st_fl / (st_ms / 1e3) / 1e12 if st_ms > 0 else None
        roofline = {"kernel": "k_part_step (K1P, cluster-partitioned implicit Euler, state in registers)",
                    "bound": "alu", "achieved": achieved, "peak": peaks["dfma"], "unit": "TFLOP/s",
                    "frac": (achieved / peaks["dfma"]) if achieved else None,
                    "traffic": _ncu_traffic(cfg.name),
                    "algorithmic_flops_per_launch": st_fl,
                    "algorithmic_bytes_per_launch": 16.0 * st_dof / cfg.m,
                    "peak_source": "FP64 FMA pipe, " + peaks["source"]}
    elif cfg.dim == 1:
        peak, peak_kind = _peaks()
        achieved = 16.0 * st_dof / (st_ms / 1e3) / 1e9 if st_ms > 0 else None
        roofline = {"kernel": "k_stepper (K1, batched tridiagonal implicit Euler)", "bound": "hbm",
                    "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": (achieved / peak) if achieved else None,
                    "traffic": _ncu_traffic(cfg.name),
                    "algorithmic_bytes_per_launch": 16.0 * st_dof,
                    "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)"}
    else:
        achieved = st_fl / (st_ms / 1e3) / 1e12 if st_ms > 0 else None
        roofline = {"kernel": "k_gemm_st (K2, FP64 DMMA sine-transform passes + fused Euler steps)",
                    "bound": "tensor", "achieved": achieved, "peak": peaks["dgemm"], "unit": "TFLOP/s",
                    "frac": (achieved / peaks["dgemm"]) if achieved else None,
                    "traffic": _ncu_traffic(cfg.name),
                    "algorithmic_flops_per_launch": st_fl,
                    "peak_source": "cuBLAS DGEMM 8192^3, " + peaks["source"],
                    "dmma_pipe_peak": peaks.get("dmma")}
    roofline.update({"launches_timed": ctr["stepper_launches"],
                     "ms_per_launch": st_ms,
                     "share_of_step": ctr["stepper_ms"] / total_ms if total_ms > 0 else None})
    return {"value": dof_total / (ms_per_step / 1e3), "ms_per_step": ms_per_step,
            "build_ms": statistics.median(build_ms), "parareal_ms": statistics.median(par_ms),
            "dof_steps_per_step": dof_total, "phases": phases, "roofline": roofline,
            "gpu_launches": ctr["kernel_launches"]}


def _sum_dof(wl, world):
    import torch
    import torch.distributed as dist
    t = torch.tensor([wl.dof_steps()], dtype=torch.float64, device=wl.dev)
    dist.all_reduce(t)
    return float(t.item())


def _e2e(wl, steps, barrier, world):
    """Same metric through the public API from HOST buffers: per step the
    operator data, u0 and the source factors go host->device from pinned
    memory, and the Parareal solution u^K (all interval boundaries) comes back
    device->host."""
    import torch
    from paper_2508_08873_b200 import Coarse, Operator, SourceTerm, parareal
    c = wl.cfg
    keys = ("space", "time", "amp", "u0") if c.dim == 1 else ("gx", "gy", "u0")
    pin = {k: torch.from_numpy(np.ascontiguousarray(wl.host[k])).pin_memory() for k in keys}
    out_host = torch.empty(tuple(wl.U.shape), dtype=torch.float64).pin_memory()
    pencil = "pencil" in wl.host
    if pencil:
        L_, rs_, M_ = wl.host["pencil"]
        h2d_op = sum(a.size for a in L_) * 8 + rs_.size * 8 + (3 * c.n * 8 if M_ is not None else 0)
    else:
        h2d_op = 5 * c.n * 8 if c.dim == 1 else 0
    h2d = sum(t.numel() * 8 for t in pin.values()) + h2d_op
    d2h = out_host.numel() * 8
    # The solution of step i goes device->host on a copy stream while step i+1
    # computes into the other of two device buffers (every copy starts and ends
    # inside the timed region; the last one is waited for before the end event).
    copy_stream = torch.cuda.Stream(device=wl.dev)
    main_stream = torch.cuda.current_stream(wl.dev)
    U_home = wl.U
    Ubuf = [U_home, torch.empty_like(U_home)]
    freed = [None, None]
    barrier()
    e0 = _event()
    for it in range(steps):
        wl.U = Ubuf[it & 1]
        if freed[it & 1] is not None:
            main_stream.wait_event(freed[it & 1])      # its previous copy has left the buffer
        dv = {k: v.to(wl.dev, non_blocking=True) for k, v in pin.items()}
        if pencil:
            op = Operator.pencil(*L_, c.dt, lrowsum=rs_, mass=M_)                   # host arrays
            src = SourceTerm(1, dv["time"].shape[0], dv["amp"].shape[0], dv["time"].shape[1],
                             {"space": dv["space"], "time": dv["time"], "amp": dv["amp"]})
        elif c.dim == 1:
            rs, cs = wl.host["sums"]
            op = Operator.tridiag(*wl.host["op"], c.dt, rowsum=rs, colsum=cs)      # host arrays
            src = SourceTerm(1, dv["time"].shape[0], dv["amp"].shape[0], dv["time"].shape[1],
                             {"space": dv["space"], "time": dv["time"], "amp": dv["amp"]})
        else:
            op = Operator.sep2d(c.n, c.dt)
            src = SourceTerm(2, dv["gx"].shape[0], 1, dv["gx"].shape[1],
                             {"gx": dv["gx"], "gy": dv["gy"]})
        U = wl.step(op=op, src=src, u0=dv["u0"])
        ready = torch.cuda.Event()
        ready.record(main_stream)
        op.close()                 # frees device memory (a device-wide wait): before the copy is queued
        if os.environ.get("BENCH_E2E_SERIAL"):     # dev aid: the copy on the compute stream
            out_host.copy_(U, non_blocking=True)
            continue
        with torch.cuda.stream(copy_stream):
            copy_stream.wait_event(ready)
            out_host.copy_(U, non_blocking=True)
            freed[it & 1] = torch.cuda.Event()
            freed[it & 1].record(copy_stream)
    main_stream.wait_stream(copy_stream)
    e1 = _event()
    wl.U = U_home
    barrier()
    ms = e0.elapsed_time(e1) / steps
    t = torch.tensor([ms], dtype=torch.float64, device=wl.dev)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    dof = wl.dof_steps() if world == 1 else _sum_dof(wl, world)
    return {"value": dof / (ms / 1e3), "unit": "DOF-steps/s", "ms_per_step": ms,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "pipelining": "the D2H copy of step i runs on a copy stream while step i+1 computes"}


if __name__ == "__main__":
    main()
