#!/usr/bin/env python
"""Benchmark of the B200 explicit phonon-BTE step (arXiv 2305.19400).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                  [--config 2|3|5|6|1] [--start random|physical] [--decomp slab|band]

Prints ONE JSON line (rank 0).  Metric: DOF-updates/s (cell x direction x
channel per second) of the whole step (boundary pass + fused sweep +
reduction/Newton [+ halo]) -- BASELINE.json `metric`.

Workload (N=1): BASELINE.json configs[1] -- 2-D non-gray silicon, 120x120
cells, 400 directions, 40 channels, Gaussian hot spot + cold wall, specular
sides, dt = 1e-12 s, synthetic seeded inputs (bte_inputs.config2).  Each
intensity buffer is 1.84 GB >> 126 MB L2, so no L2 flush is needed between
steps.  For N > 1 the mesh grows along y (120 rows per GPU, weak scaling) and
is slab-decomposed with NCCL halo exchange; --decomp band instead keeps the
BASELINE problem fixed and splits its channels over the N GPUs (the paper's
band partition: one ncclAllGather of a scalar per cell per
step, strong scaling).

--impl reference times the CPU oracle (oracle/, plain fp64 C, all host cores)
on a bounded sample of the same workload -- the paper has no runnable code,
so the oracle is the reference arm.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import bte_inputs as bi  # noqa: E402

BYTES_PER_DOF = 16  # read I^n + write I^{n+1}, fp64


def _problem(config: int, nranks: int):
    if config not in (1, 2, 3, 4, 5, 6, 7, 8, 9, 10):
        raise SystemExit(f"unsupported --config {config}")
    if config in (7, 8, 9) and nranks > 1:
        raise SystemExit("unstructured workloads (--config 7/8) run on one GPU")
    if config == 7:  # unstructured analogue of config 2: 28,800 triangles
        return bi.config_u2()
    if config == 8:  # unstructured analogue of config 3: 196,608 tetrahedra
        return bi.config_u3()
    if config == 9:  # config 7 on jittered quadrilaterals: 14,400 cells
        return bi.config_uq()
    if config == 10:  # the paper's second example (Fig. 9): elongated, corner heat source
        return bi.config_fig9()
    if config == 2:
        p = bi.config2()
        if nranks > 1:  # weak scaling: 120 rows per GPU along the slab axis
            n = p.mesh.nx
            p.mesh = bi.Mesh(2, n, n * nranks, 1, p.mesh.dx, p.mesh.dy, 1.0)
            p.name = f"config2_2d_si_{n}x{n * nranks}x400x40"
        return p
    if config == 3:
        return bi.config3()
    if config == 4:  # BASELINE configs[3]: 100^3 (10^6 cells), strong scaling over the slabs;
        return bi.config4()  # one GPU holds it only with octant-slot rotation (144 GB)
    if config == 5:
        return bi.config5(nranks)
    if config == 6:  # the paper's own demo shape, single GPU
        return bi.config_demo()
    if config == 1:  # BASELINE configs[0]: latency-bound, not roofline-gated
        return bi.config1()
    raise SystemExit(f"unsupported --config {config}")


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _traffic_per_dof(workload: str):
    """DRAM bytes per DOF of the sweep kernel, from the committed ncu --set full
    summary (dram__bytes_read.sum + dram__bytes_write.sum of one launch / its DOF)."""
    path = os.path.join(ROOT, "profiles", "ncu_sweep_summary.json")
    if not os.path.exists(path):
        return None
    try:
        d = json.load(open(path))
        e = d.get(workload)
        if e and e.get("dram_bytes_per_dof"):
            return float(e["dram_bytes_per_dof"])
    except Exception:
        return None
    return None


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device: int):
        self.samples = []
        self.max_mhz = None
        self._stop = threading.Event()
        self._ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._ok = True
        except Exception:
            self._ok = False

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
                try:
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                except Exception:
                    r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
                util = nv.nvmlDeviceGetUtilizationRates(self._h).gpu
                self.samples.append((time.time(), sm, r, util))
            except Exception:
                pass
            time.sleep(0.005)

    def start(self):
        if self._ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def stop(self):
        if self._ok:
            self._stop.set()
            self._t.join()

    def summary(self, t0: float, t1: float):
        if not self._ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        inside = [s for s in self.samples if t0 <= s[0] <= t1]
        if not inside:
            inside = sorted(self.samples, key=lambda s: abs(s[0] - 0.5 * (t0 + t1)))[:3]
        reasons = set()
        for _, _, r, _ in inside:
            for bit, name in self.REASONS.items():
                if r & bit and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": float(statistics.median(s[1] for s in inside)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(inside)}


def _oracle_sample(p, target_s: float, max_steps: int = 1000):
    """Time the oracle (as it stands) on a bounded y-slab sample of the workload:
    returns (DOF-updates/s, description, threads)."""
    import oracle
    m = p.mesh
    nthreads = os.cpu_count() or 1
    rows = (m.ny if m.dim == 2 else m.nz) if not hasattr(m, "cells") else 0
    # one-step probe on a thin slab to size the sample
    def make(nrows):
        if m.dim == 2:
            box = ((0, m.nx), (m.ny - nrows, m.ny), (0, 1))
        else:
            box = ((0, m.nx), (0, m.ny), (m.nz - nrows, m.nz))
        sp = bi.subproblem(p, box)
        o = oracle.Oracle(sp, nthreads=nthreads)
        T = bi.random_temperature(m, p.seed, p.T_init, 20.0, box=box)
        I = o.equilibrium(T) * bi.intensity_noise_factor(p.seed, 0, p.dirs.nd, p.bands.nb, 0.05, mesh=m, box=box)
        return sp, o, I, T
    if hasattr(m, "cells"):  # unstructured: a smaller mesh of the same generator
        return _oracle_sample_umesh(p, target_s, max_steps, nthreads)
    nr = max(1, min(rows, 4))
    sp, o, I, T = make(nr)
    t = time.perf_counter()
    o.run(I, T, 1)
    dt1 = time.perf_counter() - t
    per_row = dt1 / nr
    nr = int(max(1, min(rows, (target_s / 3) / max(per_row, 1e-9))))
    sp, o, I, T = make(nr)
    steps = 0
    t = time.perf_counter()
    while True:
        I, T, _, _ = o.run(I, T, 1)[:4]
        steps += 1
        if time.perf_counter() - t >= target_s or steps >= max_steps:
            break
    el = time.perf_counter() - t
    dof = sp.mesh.ncells * p.dirs.nd * p.bands.nb
    desc = (f"oracle C fp64 (gcc -O2 -ffp-contract=off, OpenMP), {steps} step(s) of a "
            f"{sp.mesh.nx}x{sp.mesh.ny}x{sp.mesh.nz}-cell slab of {p.name} (random start), {el:.1f} s")
    return dof * steps / el, desc, nthreads


def _umesh_problem(p, n):
    if p.mesh.dim == 3:
        return bi.config_u3(n=n)
    return bi.config_uq(n=n) if p.mesh.cells.shape[1] == 4 else bi.config_u2(n=n)


def _oracle_sample_umesh(p, target_s, max_steps, nthreads):
    import oracle
    n_full = 120 if p.mesh.dim == 2 else 32
    sp = _umesh_problem(p, 4)
    o = oracle.Oracle(sp, nthreads=nthreads)
    I, T = o.random_state()
    t = time.perf_counter()
    o.run(I, T, 1)
    per_cell = (time.perf_counter() - t) / sp.mesh.ncells
    cells = (target_s / 3) / max(per_cell, 1e-12)
    per_unit = 2 if p.mesh.dim == 2 else 6
    n = int(max(2, min(n_full, (cells / per_unit) ** (1.0 / p.mesh.dim))))
    sp = _umesh_problem(p, n)
    o = oracle.Oracle(sp, nthreads=nthreads)
    I, T = o.random_state()
    steps = 0
    t = time.perf_counter()
    while True:
        I, T, _, _ = o.run(I, T, 1)[:4]
        steps += 1
        if time.perf_counter() - t >= target_s or steps >= max_steps:
            break
    el = time.perf_counter() - t
    dof = sp.mesh.ncells * p.dirs.nd * p.bands.nb
    desc = (f"oracle C fp64 (gcc -O2 -ffp-contract=off, OpenMP), {steps} step(s) of {sp.name} "
            f"(the same generator at n = {n} instead of {n_full}, random start), {el:.1f} s")
    return dof * steps / el, desc, nthreads


def run_reference(args):
    """--impl reference: the CPU oracle on the host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    import oracle
    p = _problem(args.config, 1)
    m = p.mesh
    nthreads = os.cpu_count() or 1
    # each step = a bounded y-slab sample sized to ~target seconds per step so the
    # whole --warmup W --steps K run stays within a few minutes
    budget = 150.0
    per_step = budget / max(1, args.steps + args.warmup)
    rows_total = (m.ny if m.dim == 2 else m.nz) if not hasattr(m, "cells") else 0

    def make(nrows):
        if m.dim == 2:
            box = ((0, m.nx), (m.ny - nrows, m.ny), (0, 1))
        else:
            box = ((0, m.nx), (0, m.ny), (m.nz - nrows, m.nz))
        sp = bi.subproblem(p, box)
        o = oracle.Oracle(sp, nthreads=nthreads)
        T = bi.random_temperature(m, p.seed, p.T_init, 20.0, box=box)
        I = o.equilibrium(T) * bi.intensity_noise_factor(p.seed, 0, p.dirs.nd, p.bands.nb, 0.05, mesh=m, box=box)
        return sp, o, I, T

    if hasattr(m, "cells"):  # unstructured: each step on a smaller mesh of the same generator
        sp = _umesh_problem(p, 4)
        o = oracle.Oracle(sp, nthreads=nthreads)
        I, T = o.random_state()
        t = time.perf_counter()
        o.run(I, T, 1)
        per_cell = (time.perf_counter() - t) / sp.mesh.ncells
        per_unit = 2 if m.dim == 2 else 6
        n = int(max(2, ((per_step / max(per_cell, 1e-12)) / per_unit) ** (1.0 / m.dim)))
        sp = _umesh_problem(p, n)
        o = oracle.Oracle(sp, nthreads=nthreads)
        I, T = o.random_state()
    else:
        sp, o, I, T = make(1)
        t = time.perf_counter()
        o.run(I, T, 1)
        per_row = time.perf_counter() - t
        nr = int(max(1, min(rows_total, per_step / max(per_row, 1e-9))))
        sp, o, I, T = make(nr)
    I0c, betac = o.refresh(T)
    for _ in range(args.warmup):
        I, T, I0c, betac = o.run(I, T, 1, I0c, betac)
    t = time.perf_counter()
    for _ in range(args.steps):
        I, T, I0c, betac = o.run(I, T, 1, I0c, betac)
    el = time.perf_counter() - t
    dof = sp.mesh.ncells * p.dirs.nd * p.bands.nb
    value = dof * args.steps / el
    if hasattr(m, "cells"):
        sample = f"each step = one oracle step of {sp.name} (same generator, smaller mesh; random start)"
    else:
        sample = (f"each step = one oracle step of a {sp.mesh.nx}x{sp.mesh.ny}x{sp.mesh.nz}-cell slab of "
                  f"{p.name} (random start)")
    line = {
        "impl": "reference", "metric": "BTE DOF-updates/s (cell x dir x band / s), whole step",
        "value": value, "unit": "DOF-updates/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, bte_inputs)",
        "config": {"workload": p.name, "sample": sample},
        "cpu_baseline": {"value": value, "unit": "DOF-updates/s", "cores": nthreads, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": value, "unit": "DOF-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def run_b200(args):
    import torch
    import torch.distributed as dist

    from paper_2305_19400_b200 import Solver, build, nccl_unique_id
    build.build()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    band = args.decomp == "band"
    p = _problem(args.config, 1 if band else world)
    if args.semi > 0:
        p.dt = args.semi * p.dt
        p.semi = 1
    nccl_id = None
    if world > 1:
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    stream = torch.cuda.Stream(local)
    sv = Solver.from_problem(p, device=local, stream=stream, rank=rank, nranks=world, nccl_id=nccl_id,
                             decomp=args.decomp)
    if args.tau == "sc":
        sv.set_tau_mode(1)
    dof_local = sv.ncells * sv.nd * sv.nb
    dof_global = sv.ncells_global * sv.nd * sv.nb_total

    def init_state():
        if args.start == "random":
            sv.init_random(p.seed, bi.random_phases(p.seed), p.T_init, 20.0, 0.05)
        else:
            sv.set_state(None, np.full(sv.ncells, p.T_init))

    def barrier():
        torch.cuda.synchronize(local)
        if world > 1:
            dist.barrier()

    init_state()
    sv.step(args.warmup)
    clocks = ClockSampler(local)
    clocks.start()
    sv.timing_enable(True, args.steps)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    barrier()
    t0 = time.time()
    ev0.record(stream)
    sv.step(args.steps)
    ev1.record(stream)
    barrier()
    t1 = time.time()
    clocks.stop()
    ms = ev0.elapsed_time(ev1)
    tim = sv.timing_read()
    sv.timing_enable(False)
    if world > 1:
        t = torch.tensor([ms], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = dof_global * args.steps / (ms * 1e-3)

    # roofline of the dominant kernel (the fused sweep): algorithmic 16 B/DOF;
    # one step launches the sweep once per column chunk
    peak, peak_src = _peaks()
    launches_per_step = max(1, tim["sweep_launches"] // max(1, tim["steps"]))
    sweep_ms = tim["sweep_ms"] / max(1, tim["sweep_launches"])
    dof_per_launch = dof_local / launches_per_step
    achieved = BYTES_PER_DOF * dof_per_launch / (sweep_ms * 1e-3) / 1e9
    tpd = _traffic_per_dof(p.name)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": None if tpd is None else tpd * dof_per_launch,
                "kernel": ("k_usweep (a1+a2 face-list upwind flux + relaxation on simplices + octant partial sums)"
                           if sv.umesh else ("k_sweep_tma" if sv.nj * sv.nb >= 384 else "k_sweep")
                           + " (a1+a2 fused upwind flux + relaxation + octant partial sums"
                           + (", a3+a4 Newton fused in the tail)" if tim["newton_launches"] == 0 else ")")),
                "bytes_per_launch_algorithmic": BYTES_PER_DOF * dof_per_launch, "kernel_ms_avg": sweep_ms,
                "launches_per_step": launches_per_step, "peak_source": peak_src,
                "device_ms_per_step": {"sweep": tim["sweep_ms"] / args.steps, "newton": tim["newton_ms"] / args.steps,
                                       "boundary": tim["boundary_ms"] / args.steps,
                                       "halo": tim["halo_ms"] / args.steps},
                "note": ("octant-slot rotation: one sweep launch per octant, each into the spare region"
                         if sv.rotate else "sweep and Newton serialised on one stream" if launches_per_step == 1
                         else "Newton of chunk k on a second stream, overlapped with other chunks' sweeps")}

    # e2e through the public API with host buffers (pinned), copies inside the
    # timed region: the job's input state (I, T) goes host->device, K steps run,
    # and the job's result -- the temperature field, "ultimately the quantity of
    # interest" -- comes back device->host.
    e2e = None
    state_gb = sv.ncells * sv.nd * sv.nb * 8 / 1e9
    if state_gb > 16:  # config 4: a 128 GB pinned host copy of the state would exhaust the host
        e2e = {"value": None, "unit": "DOF-updates/s", "skipped": f"state {state_gb:.0f} GB per GPU > 16 GB host staging cap"}
    elif not args.no_e2e:
        I_h = torch.empty((sv.ncells, sv.nd, sv.nb), dtype=torch.float64, pin_memory=True).numpy()
        T_h = torch.empty((sv.ncells,), dtype=torch.float64, pin_memory=True).numpy()
        sv.intensity(I_h)
        sv.temperature(T_h)
        barrier()
        t = time.perf_counter()
        sv.set_state(I_h, T_h)
        sv.step(args.steps)
        sv.temperature(T_h)
        barrier()
        el = time.perf_counter() - t
        if world > 1:
            tt = torch.tensor([el], device=f"cuda:{local}", dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            el = float(tt.item())
        e2e = {"value": dof_global * args.steps / el, "unit": "DOF-updates/s",
               "h2d_bytes_per_step": (I_h.nbytes + T_h.nbytes) / args.steps,
               "d2h_bytes_per_step": T_h.nbytes / args.steps,
               "what": "bte_set_state(pinned host I, T) + bte_step(K) + bte_get_temperature (pinned host T)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, desc, cores = _oracle_sample(p, target_s=args.cpu_seconds)
        cpu = {"value": v, "unit": "DOF-updates/s", "cores": cores, "kind": "oracle", "sample": desc}

    if rank == 0:
        line = {
            "metric": "BTE DOF-updates/s (cell x dir x band / s), whole step",
            "value": value, "unit": "DOF-updates/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if (band or args.config in (4, 7, 8, 9)) else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded bte_inputs; silicon tables are paper-silent data)",
            "config": {"workload": p.name, "cells": sv.ncells_global, "directions": sv.nd, "channels": sv.nb_total,
                       "dof_per_step": dof_global, "start": args.start, "dt": p.dt, "tau": args.tau,
                       "integrator": "semi-implicit" if args.semi > 0 else "explicit",
                       "simulated_s_per_s": p.dt * args.steps / (ms * 1e-3),
                       "parallelism": ((f"band{world}" if band else (f"cells{world}" if sv.umesh else f"slab{world}"))
                                       if world > 1 else "single"),
                       "storage": "octant-slot rotation" if sv.rotate else "two buffers",
                       "l2": f"inputs > L2 ({state_gb:.2f} GB/buffer vs 126 MB), no flush"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(tim["launches"]),
            "clocks": clocks.summary(t0, t1),
        }
        print(json.dumps(line))
    sv.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--start", default="random", choices=["random", "physical"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--decomp", default="slab", choices=["slab", "band"])
    ap.add_argument("--semi", type=float, default=0.0,
                    help="semi-implicit step (reading R-l) at this multiple of the workload's dt (0: explicit)")
    ap.add_argument("--tau", default="lagged", choices=["lagged", "sc"],
                    help="temperature update: lagged tau (reading #15) or self-consistent tau (R-k)")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
