#!/usr/bin/env python
"""Benchmark: explicit-Euler steps/s of the semi-explicit MQS scheme on B200.

Headline workload (BASELINE.json configs[2], the largest single-GPU config and
the north star's HBM case): 128^3 cells, two Brauer iron blocks of 24^3,
annular coil J = 5e6 sin(2 pi 50 t), fp64, PCG (Jacobi, rel_tol 1e-8), POD
start vectors from a 30-snapshot ring, output (recover_an + B probe) every
step: 4 K_n solves per step.  A "step" is one explicit-Euler step plus the
recovery of a_n.  W warm-up steps (untimed; they also fill the snapshot
rings) precede K timed steps of the same trajectory.  L2 is flushed (256 MB
write) before every timed step, outside the timed events.

Outputs one JSON line (rank 0).  `value` is device-timed with the inputs
resident in HBM; `e2e` is the same metric through the host-facing API
(explicit_euler_step + recover_an + probe_b with host arrays, copies inside
the timed region); `roofline` is the fused PCG kernel (pcg_tma1_kernel)
measured with CUDA events inside the timed region.  Secondary keys: configs[1]
(64^3) with CSPE and with POD-20, configs[4] (256^3) on one GPU.
`cpu_baseline` times the CPU port of the reference (oracle/, numpy/scipy) on
a bounded sample of the same steps (see cpu_sampled_steps).

--impl reference runs the CPU port of the reference on the same workload and
prints the same metric.  With torchrun (N > 1) every rank runs an
independent replica of the workload (configs 0-2 do not shard: SURVEY.md
8(e)), no collective on the data path; the timing is the max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "explicit-Euler steps/s (config 2: 128^3 two Brauer blocks, POD-30, recover every step)"
UNIT = "steps/s"


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# clocks sampling during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    def __init__(self, device_index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self._ok = True
        except Exception as exc:  # noqa: BLE001
            self.err = str(exc)

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.02)

    def __enter__(self):
        if self._ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._ok:
            self.t.join()

    def summary(self):
        if not self._ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "note": getattr(self, "err", "")}
        med = float(np.median(self.samples)) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------
def schedule(spec, n_steps, dt=None):
    dt = spec.dt if dt is None else dt
    w = 2.0 * np.pi * spec.freq
    tt = [0.0]
    for _ in range(n_steps):
        tt.append(tt[-1] + dt)
    import math
    wave = np.array([math.sin(w * t) for t in tt])
    return np.full(n_steps, dt), wave, tt


def pcg_launch_bytes(n_n, iters, modes=None):
    """Algorithmic bytes of one fused-PCG launch with `iters` iterations.

    9 vector streams per iteration (72 B/dof), the initial residual pass
    (read b and x0 with the stencil, write r and x: 4 streams) and the final
    x += alpha p (3 streams) when it iterated."""
    iters = np.asarray(iters, dtype=np.float64)
    return 8.0 * n_n * (9.0 * iters + 4.0 + 3.0 * (iters > 0))


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        import datetime
        # ranks wait in collectives while rank 0 runs its single-GPU legs
        timeout = datetime.timedelta(minutes=60)
        if os.environ.get("MQ_BENCH_PLUMBING_TEST"):
            # functional check of the multi-rank path on a one-GPU box (every
            # rank on cuda:0, gloo): never a measurement
            local = 0
            torch.cuda.set_device(0)
            dist.init_process_group("gloo", timeout=timeout)
            return world, rank, local, dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local), timeout=timeout)
        return world, rank, local, dist
    return 1, 0, 0, None


def max_over_ranks(x: float, dist, local):
    if dist is None:
        return x
    import torch
    dev = "cpu" if dist.get_backend() == "gloo" else f"cuda:{local}"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(dist):
    if dist is not None:
        dist.barrier()


# ---------------------------------------------------------------------------
# CPU port of the reference (oracle) on the same workload
# ---------------------------------------------------------------------------
FIELDS = ROOT / "tests" / "golden"


def oracle_iterations(index: int, strategy: str):
    """The oracle's own per-step iteration counts [src, prev, src_rec, cur]
    (tests/golden/fields_*.npz, made by running the oracle on the config)."""
    name = {(1, "cspe"): "cfg1_cspe", (1, "pod"): "cfg1_pod", (2, "pod"): "cfg2"}[(index, strategy)]
    f = np.load(FIELDS / f"fields_{name}.npz")
    n = int(f["steps"])
    src = f["iters_src"][1:].reshape(n, 2)
    return np.stack([src[:, 0], f["iters_prev"], src[:, 1], f["iters_cur"][1:]], axis=1), name


def cpu_sampled_steps(index: int, strategy: str, warmup: int, steps: int, *, iters=(35, 105), kept_modes=4):
    """steps/s of the CPU port (oracle/mq_oracle.py, a numpy/scipy restatement
    of mqsolve) on steps warmup+1 .. warmup+steps, from a bounded sample.

    Running those steps takes minutes each at 128^3 (0.36 s per PCG
    iteration), so the sample measures, on this host and on the config's own
    assembled matrices, the parts a step is made of and adds them up for
    every timed step:
      * t_it: one PCG iteration of the oracle's pcg loop (SpMV, dots, axpys),
        from two truncated solves of iters[0] and iters[1] iterations (the
        per-iteration cost falls over the first tens of iterations of a solve
        as numpy's allocations warm up: 0.27 s at 5, 0.22 s at 105 at 128^3);
      * t_init: a solve that ends at its initial residual (x0 given);
      * t_start(m): one start vector of the strategy with m columns in the
        family's history (POD: Gram of the ring, eigh, basis, k SpMVs, the
        Galerkin solve; CSPE: the projection) measured at two history sizes and
        interpolated linearly in m, plus one observe (POD push / CSPE insert);
      * t_rest: the step's remaining work (K_cn^T products, the Euler update
        with the Brauer K_c, the recovery's subtraction, the B probe).
    Per step: sum over its 4 solves of (t_init + its iteration count * t_it +
    t_start(m) + t_observe) + t_rest, with the oracle's own iteration counts of
    exactly those steps (oracle_iterations) and the history sizes the
    reference's ring / FIFO rules give at that step.  The model is checked
    against timed oracle steps in DESIGN.md."""
    from oracle import mq_oracle as O
    from paper_1611_06721_b200 import configs as C
    spec = C.config_spec(index)
    t0 = time.perf_counter()
    mat = C.material_map(spec)
    loops = C.coil_loops(spec.N, spec.J)
    m = O.assemble(mat, spec.h, O.Conductor(spec.kappa, *spec.brauer),
                   [O.Loop(lp.i0, lp.i1, lp.j0, lp.j1, lp.k0, lp.amps) for lp in loops])
    t_asm = time.perf_counter() - t0
    inv = O.jacobi_inverse(m.kn.diagonal())
    n = m.n_n
    b = m.pattern.copy()
    x0 = np.zeros(n)
    rng0 = np.random.default_rng(1)

    def truncated(k):
        ts = time.perf_counter()
        O.pcg(m.kn_apply, b, x0=x0, rel_tol=1e-300, max_iter=k, inv_diag=inv)
        return time.perf_counter() - ts
    truncated(3)  # first touch of the matrix and of the allocator's pages
    ta, tb = truncated(iters[0]), truncated(iters[1])
    t_it = (tb - ta) / (iters[1] - iters[0])
    # a solve that ends at its initial residual (x0 given, ||r|| <= target)
    ts = time.perf_counter()
    for _ in range(3):
        O.pcg(m.kn_apply, b, x0=x0, rel_tol=1.0, max_iter=1, inv_diag=inv)
    t_init = (time.perf_counter() - ts) / 3
    # history columns: successive solutions of one family are smooth and
    # nearly dependent (POD keeps about kept_modes of them): mixtures of that
    # many Krylov vectors of the Jacobi-scaled K_n plus a 1e-7 perturbation
    cap = spec.n_pod if strategy == "pod" else spec.max_cols
    v = b / np.linalg.norm(b)
    base = []
    for _ in range(kept_modes):
        v = inv * m.kn_apply(v)
        v = v / np.linalg.norm(v)
        base.append(v)
    hist = []
    for jj in range(cap):
        h = sum(np.cos(0.3 * (ii + 1) * jj) * base[ii] for ii in range(kept_modes))
        h = h + 1e-7 * np.linalg.norm(h) / np.sqrt(n) * rng0.standard_normal(n)
        hist.append(h)
    lo_m = max(1, cap // 3)

    def start_cost(mm):
        if strategy == "pod":
            snap = O.Snapshots(n, spec.n_pod, 1e-4)
            for u in hist[:mm]:
                snap.push(u)
            ts = time.perf_counter()
            _, k, _, _ = O.pod_start(snap, b, m.kn_apply)
            return time.perf_counter() - ts, k
        cache = O.SpeCache(n, m.kn_apply, spec.max_cols, spec.rel_tol)
        for u in hist[:mm]:
            cache.insert(u)
        ts = time.perf_counter()
        cache.project(b)
        return time.perf_counter() - ts, cache.k
    (t_lo, _), (t_hi, k_hi) = start_cost(lo_m), start_cost(cap)
    # one observe with a full history
    if strategy == "pod":
        snap = O.Snapshots(n, spec.n_pod, 1e-4)
        for u in hist:
            snap.push(u)
        ts = time.perf_counter()
        snap.push(b)
        t_obs = time.perf_counter() - ts
    else:
        cache = O.SpeCache(n, m.kn_apply, spec.max_cols, spec.rel_tol)
        for u in hist:
            cache.insert(u)
        ts = time.perf_counter()
        cache.insert(b / np.linalg.norm(b) + hist[0])
        t_obs = time.perf_counter() - ts
    # the step's remaining work (schur.py:379-419, model.py:415-425)
    rng = np.random.default_rng(0)
    a_c = rng.standard_normal(m.n_c) * 1e-9
    y1, y2 = rng.standard_normal(n), rng.standard_normal(n)
    cells = O.default_probe_cells(m, (spec.N,) * 3)
    minv = 1.0 / m.mc_diag
    ts = time.perf_counter()
    m.kcn.T @ a_c
    m.kcn.T @ a_c
    rate = m.kcn @ (y1 - y2) - m.kc_apply(a_c, a_c)
    a_next = a_c + spec.dt * (minv * rate)
    np.isfinite(a_next).all()
    a_n = y1 - y2
    O.probe_b(m, O.full_interior(m, a_next, a_n), cells)
    t_rest = time.perf_counter() - ts

    def t_start(mm):
        if mm <= 0:
            return 0.0
        return t_lo + (t_hi - t_lo) * (min(mm, cap) - lo_m) / max(cap - lo_m, 1)

    its, fixture = oracle_iterations(index, strategy)
    tail = its[-10:].mean(axis=0)
    total = 0.0
    for s in range(warmup + 1, warmup + steps + 1):
        row = its[s - 1] if s <= len(its) else tail
        # history sizes before each solve (one record per solve, FIFO/ring cap)
        hsz = [min(cap, 2 * s - 1), min(cap, s - 1), min(cap, 2 * s), min(cap, s)]
        total += sum(t_init + float(row[q]) * t_it + t_start(hsz[q]) + t_obs for q in range(4)) + t_rest
    covered = min(warmup + steps, len(its)) - warmup
    sample = (f"config {index} ({spec.N}^3, {strategy}) steps {warmup + 1}..{warmup + steps}: oracle/mq_oracle.py "
              f"(numpy/scipy port of mqsolve) on this host, per-part timing x the oracle's own iteration counts "
              f"of those steps (tests/golden/fields_{fixture}.npz covers {max(covered, 0)} of them, the rest at "
              f"the mean of its last 10 steps): PCG iteration {t_it * 1e3:.1f} ms, initial residual "
              f"{t_init * 1e3:.1f} ms, start vector {t_lo * 1e3:.0f} ms ({lo_m} columns) .. {t_hi * 1e3:.0f} ms "
              f"({cap} columns, k = {k_hi}), observe {t_obs * 1e3:.0f} ms, rest {t_rest * 1e3:.0f} ms; "
              f"assembly {t_asm:.0f} s not counted; scipy csr_matvec single-threaded, numpy BLAS on all cores")
    parts = {"pcg_iteration_ms": t_it * 1e3, "initial_residual_ms": t_init * 1e3,
             "start_vector_ms": [t_lo * 1e3, t_hi * 1e3], "start_vector_columns": [lo_m, cap],
             "observe_ms": t_obs * 1e3, "rest_ms": t_rest * 1e3,
             "timed_step_iterations": its[warmup:warmup + steps].tolist()}
    return steps / total, total, sample, parts, n


def host_info():
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cores": os.cpu_count(), "cpu_model": model,
            "openblas_threads": os.environ.get("OPENBLAS_NUM_THREADS", "default (all cores)")}


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from paper_1611_06721_b200 import configs as C
    spec = C.config_spec(2)
    v, el, sample, parts, n_n = cpu_sampled_steps(2, "pod", args.warmup, args.steps)
    hi = host_info()
    line = {
        "metric": METRIC, "value": v, "unit": UNIT, "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * el / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "cfg2_128cube_two_blocks_pod30", "grid": [128, 128, 128], "n_n": n_n,
                   "strategy": "pod", "n_pod": 30, "rel_tol": 1e-8, "dt": spec.dt},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": hi["cores"], "kind": "port", "sample": sample,
                         "host": hi, "parts": parts},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# device arm
# ---------------------------------------------------------------------------
def time_device_steps(op, spec, warmup, steps, flush=True, dt=None):
    """W warm-up steps then K timed steps (CUDA events per step on the
    context stream, L2 flushed before each), PCG launches timed inside."""
    import ctypes

    from paper_1611_06721_b200 import _lib
    from paper_1611_06721_b200._lib import check, dptr
    lib, ctx = op.lib, op.grid.ctx
    dts, wave, _ = schedule(spec, warmup + steps, dt)
    op._set_state(np.zeros(op.grid.n_c), 0.0)
    # initial recovery at t = 0 as in the reference loop
    from paper_1611_06721_b200.schur import recover_an
    recover_an(op, np.zeros(op.grid.n_c), 0.0)
    op._set_state(np.zeros(op.grid.n_c), 0.0)
    check(lib.mq_run_prepare(ctx, warmup + steps, dptr(dts), dptr(wave), 1))
    # PCG event records must exist when the step graph is captured (warm-up)
    check(lib.mq_pcg_stats(ctx, None, None, None, 1))
    check(lib.mq_run_steps(ctx, warmup, 1, None))
    check(lib.mq_ctx_sync(ctx))
    l0 = ctypes.c_int64()
    check(lib.mq_kernel_launches(ctx, ctypes.byref(l0)))
    step_ms, pcg_ms = [], []
    ms = ctypes.c_double()
    pm = ctypes.c_double()
    ne = ctypes.c_int32()
    for _ in range(steps):
        if flush:
            check(lib.mq_l2_flush(ctx))
        check(lib.mq_timer_start(ctx))
        check(lib.mq_run_steps(ctx, 1, 1, None))
        check(lib.mq_timer_stop(ctx, ctypes.byref(ms)))
        check(lib.mq_pcg_collect(ctx, ctypes.byref(pm), ctypes.byref(ne)))
        step_ms.append(ms.value)
        pcg_ms.append(pm.value)
    l1 = ctypes.c_int64()
    check(lib.mq_kernel_launches(ctx, ctypes.byref(l1)))
    check(lib.mq_pcg_stats(ctx, None, None, None, 0))
    iters = np.zeros((warmup + steps, 4), dtype=np.int32)
    failed = ctypes.c_int64()
    check(lib.mq_run_finish(ctx, _lib.i32ptr(iters), ctypes.byref(failed)))
    return np.array(step_ms), np.array(pcg_ms), iters[warmup:], int(l1.value - l0.value)


def time_e2e(problem, spec, warmup, steps):
    """Same steps through the host-facing API (explicit_euler_step +
    recover_an + probe_b with host arrays; copies inside the timed region)."""
    from paper_1611_06721_b200 import PcgConfig, SchurOperator, explicit_euler_step, recover_an
    op = SchurOperator(problem, pcg=PcgConfig(rel_tol=spec.rel_tol, max_iter=spec.max_iter),
                       strategy=spec.strategy, max_cols=spec.max_cols, n_pod=spec.n_pod)
    op.set_probe()
    a = np.zeros(op.grid.n_c)
    t = 0.0
    recover_an(op, a, t)
    for s in range(warmup):
        a, _ = explicit_euler_step((a, t), spec.dt, op, s + 1)
        t += spec.dt
        recover_an(op, a, t)
    op.grid.sync()
    t0 = time.perf_counter()
    for s in range(steps):
        a, _ = explicit_euler_step((a, t), spec.dt, op, warmup + s + 1)
        t += spec.dt
        a_n, _ = recover_an(op, a, t)
        op.probe_b()
    el = time.perf_counter() - t0
    n_c, n_n = op.grid.n_c, op.grid.n_n
    h2d = 2 * n_c * 8              # a_c uploaded by each of the two calls
    d2h = n_c * 8 + n_n * 8 + 8    # a_c after the step, a_n after the recovery, B_probe
    op.grid.close()
    return steps / el, el, h2d, d2h


def traffic_for(key, iters):
    """DRAM bytes (read + write) per launch of the PCG kernel, from the
    committed ncu --set full capture (profiles/traffic.json: bytes per
    iteration of that kernel on that grid) x this run's iteration counts."""
    tj = ROOT / "profiles" / "traffic.json"
    if not tj.exists():
        return None
    t = json.loads(tj.read_text()).get(key)
    if not t:
        return None
    its = np.asarray(iters, dtype=np.float64)
    return float(t["dram_bytes_per_iteration"] * its.mean())


def cfg_steps(index, warmup=3, steps=5, strategy=None, with_roofline=None):
    """configs[1] (64^3, CSPE k=5 or POD-20) or configs[4] (256^3, CSPE k=5,
    one GPU) through the same device step loop: steps/s with L2 flushed before
    each step.  Secondary keys; the headline is configs[2].
    with_roofline=<HBM peak>: the PCG kernel's bytes/s inside the timed steps,
    labelled by what bounds it (configs[1]: every PCG vector fits in L2 and
    shared memory, so it is not an HBM figure)."""
    from dataclasses import replace

    from paper_1611_06721_b200 import PcgConfig, SchurOperator, configs as C
    spec = C.config_spec(index)
    if strategy is not None:
        spec = replace(spec, strategy=strategy, name=f"{spec.name.split('_cspe')[0]}_{strategy}{spec.n_pod}")
    op = SchurOperator(C.make_problem(index), pcg=PcgConfig(rel_tol=spec.rel_tol, max_iter=spec.max_iter),
                       strategy=spec.strategy, n_pod=spec.n_pod, max_cols=spec.max_cols)
    op.set_probe()
    kname, kgrid = op.grid.pcg_kernel()
    n_n = op.grid.n_n
    step_ms, pcg_ms, iters, launches = time_device_steps(op, spec, warmup, steps)
    op.grid.close()
    n = spec.N
    out = {"workload": spec.name, "grid": [n, n, n], "strategy": spec.strategy,
           "n_pod" if spec.strategy == "pod" else "max_cols": spec.n_pod if spec.strategy == "pod" else spec.max_cols,
           "dt": spec.dt, "steps_after_warmup": [warmup + 1, warmup + steps],
           "value": steps / (float(step_ms.sum()) * 1e-3), "unit": UNIT,
           "ms_per_step": float(step_ms.mean()), "pcg_share_of_step": float(pcg_ms.sum() / step_ms.sum()),
           "timed_step_iterations": iters.tolist(), "gpu_launches": launches}
    if with_roofline:
        byts = pcg_launch_bytes(n_n, iters.reshape(-1)).sum()
        ach = byts / (float(pcg_ms.sum()) * 1e-3) / 1e9
        out["roofline"] = {
            "bound": "latency (L2/shared-memory resident)", "achieved": ach, "unit": "GB/s",
            "frac_of_hbm_peak": ach / with_roofline, "kernel": kname, "kernel_grid": kgrid,
            "us_per_iteration": 1000.0 * float(pcg_ms.sum()) / max(int(iters.sum()), 1),
            "traffic": traffic_for(f"cfg{index}", iters.reshape(-1)),
            "note": "72 B/dof/iteration convention; the 64^3 vectors (5.7 MB) stay in shared memory and L2, "
                    "DRAM traffic is ~0.3 % of it: the kernel is bound by its grid barriers and "
                    "shared-memory passes, not by HBM"}
    return out


def cfg_pcg_roofline(index, hbm_peak, reps=2):
    """Fused PCG kernel on the grid of configs[index] (2: 128^3, 4: 256^3):
    cold source solve, one launch timed with CUDA events."""
    import ctypes

    from paper_1611_06721_b200 import _lib, configs as C
    from paper_1611_06721_b200._lib import check
    from paper_1611_06721_b200.device import DeviceGrid
    prob = C.make_problem(index)
    g = DeviceGrid(prob)
    lib = g.lib
    b = g.alloc()
    x = g.alloc()
    g.upload(prob.pattern, b)
    rep = _lib.SolveReportC()
    # warm-up solve
    check(lib.mq_pcg_solve_dev(g.ctx, ctypes.c_void_p(b), None, ctypes.c_void_p(x), 1e-8, 0.0, 5000, 1,
                               ctypes.byref(rep)))
    best = None
    for _ in range(reps):
        check(lib.mq_l2_flush(g.ctx))
        check(lib.mq_pcg_stats(g.ctx, None, None, None, 1))
        check(lib.mq_pcg_solve_dev(g.ctx, ctypes.c_void_p(b), None, ctypes.c_void_p(x), 1e-8, 0.0, 5000, 1,
                                   ctypes.byref(rep)))
        ms = ctypes.c_double()
        it = ctypes.c_int64()
        check(lib.mq_pcg_stats(g.ctx, ctypes.byref(ms), ctypes.byref(it), None, 0))
        if best is None or ms.value < best[0]:
            best = (ms.value, int(rep.iterations))
    ms, iters = best
    n_n = g.n_n
    kname, kgrid = g.pcg_kernel()
    byts = float(pcg_launch_bytes(n_n, iters))
    achieved = byts / (ms * 1e-3) / 1e9
    g.close()
    # DRAM traffic per launch from the committed ncu --set full capture of the
    # same kernel on the same grid (per-iteration bytes x this launch's count)
    traffic = traffic_for(f"cfg{index}", [iters])
    return {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
            "frac": achieved / hbm_peak, "traffic": traffic,
            "traffic_source": "profiles/traffic.json (ncu dram__bytes_read+write per iteration)",
            "kernel": kname, "kernel_grid": kgrid, "grid": [prob.material.shape[0]] * 3, "n_n": n_n,
            "iterations": iters, "launch_ms": ms,
            "us_per_iteration": 1000.0 * ms / max(iters, 1),
            "bytes_per_launch": byts, "bytes_per_iteration": 72.0 * n_n}


SHARDED_DEADLINE_S = 600


def cfg4_sharded(dist, world, local, hbm_peak, warmup=1, steps=2):
    """configs[4] (256^3, Brauer, CSPE k = 5) with the sharded step over the
    ranks of this job (slabstep.py: one i-slab per rank and GPU, fused slab
    PCG over CUDA-IPC-mapped neighbour buffers, NCCL all-gathers of the rank
    partials and the owned conducting values).  Strong scaling: the same grid
    at every N.  Every call of a step synchronises the host (reductions), so
    steps are timed by the host clock after a device synchronisation, max
    over ranks."""
    import torch

    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200.slabstep import SlabStepper
    spec = C.config_spec(4)
    prob = C.make_problem(4)
    t0 = time.perf_counter()
    # MQ_BENCH_PLUMBING_TEST (every rank on cuda:0, gloo): ranks on one GPU
    # must never run kernels that wait on one another, so the PCG is the
    # host-driven phase loop there; on one GPU per rank the fused kernel
    pcg = "host" if (os.environ.get("MQ_BENCH_PLUMBING_TEST") and world > 1) else "fused"
    st = SlabStepper(prob, world, dist=dist, device=local, strategy="cspe", max_cols=spec.max_cols,
                     rel_tol=spec.rel_tol, max_iter=spec.max_iter, pcg=pcg)
    setup = time.perf_counter() - t0
    try:
        st.recover(gather=False)
        for _ in range(warmup):
            st.step(spec.dt)
            st.recover(gather=False)
        torch.cuda.synchronize(local)
        barrier(dist)
        its, secs = [], []
        pcg0 = st.pcg_seconds
        for _ in range(steps):
            ts = time.perf_counter()
            r1, r2 = st.step(spec.dt)
            _, (r3, r4) = st.recover(gather=False)
            torch.cuda.synchronize(local)
            secs.append(time.perf_counter() - ts)
            its.append([r1.iterations, r2.iterations, r3.iterations, r4.iterations])
        pcg_s = st.pcg_seconds - pcg0
        n_n = st.n_n
    finally:
        st.close()
    total = max_over_ranks(float(sum(secs)), dist, local)
    pcg_max = max_over_ranks(pcg_s, dist, local)
    byts = float(pcg_launch_bytes(n_n, np.asarray(its).reshape(-1)).sum())
    agg = byts / pcg_max / 1e9
    return {"workload": "cfg4_256cube_two_blocks_cspe5_sharded", "grid": [256, 256, 256], "n_n": n_n,
            "ranks": world, "scaling": "strong", "decomposition": "i-slabs, one per rank/GPU",
            "dt": spec.dt, "steps_after_warmup": [warmup + 1, warmup + steps],
            "value": steps / total, "unit": UNIT, "ms_per_step": 1e3 * total / steps,
            "pcg_share_of_step": pcg_max / total, "timed_step_iterations": its,
            "pcg_GBps_aggregate": agg, "pcg_GBps_per_gpu": agg / world,
            "frac_of_N_hbm": agg / (hbm_peak * world), "setup_s": setup,
            "timing": "host clock around each step after cuda synchronize (the step synchronises at every "
                      "reduction), max over ranks"}


def ensemble_members(dist, world, rank, local, members_per_rank=2, warmup=3, steps=5):
    """configs[3] (256 independent 64^3 members, CSPE k = 5): the members are
    sharded over the ranks (ensemble.shard, weak scaling, no collective); each
    rank times the first ``members_per_rank`` members of its shard through the
    device step loop (CUDA events per step, L2 flushed before each), one member
    at a time on the whole GPU (the resident single-member PCG is
    faster per member-iteration than a batched or sliced one at 64^3)."""
    from paper_1611_06721_b200 import PcgConfig, SchurOperator, configs as C
    from paper_1611_06721_b200 import ensemble as E
    spec = C.config_spec(3)
    mine = list(E.shard(256, world, rank))[:members_per_rank]
    total_ms, per, its = 0.0, [], []
    for m in mine:
        prob, jf, kf, dt = E.member_problem(m)
        op = SchurOperator(prob, pcg=PcgConfig(rel_tol=spec.rel_tol, max_iter=spec.max_iter),
                           strategy="cspe", max_cols=spec.max_cols, device=local)
        op.set_probe()
        step_ms, _, iters, _ = time_device_steps(op, spec, warmup, steps, dt=dt)
        op.grid.close()
        total_ms += float(step_ms.sum())
        per.append({"member": m, "j_factor": jf, "kappa_factor": kf, "dt": dt,
                    "steps_per_s": steps / (float(step_ms.sum()) * 1e-3)})
        its.append(iters.tolist())
    t_max = max_over_ranks(total_ms, dist, local)
    value = world * len(mine) * steps / (t_max * 1e-3)
    return {"workload": "cfg3_ensemble_64cube_cspe5", "scaling": "weak",
            "sharding": "256 members in contiguous blocks over the ranks, no data-path collective",
            "members_per_rank_timed": len(mine), "members_per_rank_total": len(E.shard(256, world, rank)),
            "steps_after_warmup": [warmup + 1, warmup + steps],
            "value": value, "unit": "member-steps/s",
            "projected_s_for_256x200_steps": 256 * 200 / value, "members_rank0": per,
            "timed_step_iterations_rank0": its}


def run_device_arm(args):
    world, rank, local, dist = dist_init()
    from paper_1611_06721_b200 import PcgConfig, SchurOperator, _lib
    from paper_1611_06721_b200 import configs as C
    _lib.load()
    spec = C.config_spec(2)
    problem = C.make_problem(2)
    hbm_peak, peak_kind = peaks()
    op = SchurOperator(problem, pcg=PcgConfig(rel_tol=spec.rel_tol, max_iter=spec.max_iter),
                       strategy=spec.strategy, n_pod=spec.n_pod, device=local)
    # B_probe per output row, as the reference bench records (bench.py:371)
    op.set_probe()
    n_n, n_c = op.grid.n_n, op.grid.n_c
    kname, kgrid = op.grid.pcg_kernel()
    barrier(dist)
    with ClockSampler(local) as clk:
        step_ms, pcg_ms, iters, launches = time_device_steps(op, spec, args.warmup, args.steps,
                                                             flush=not args.no_flush)
    barrier(dist)
    total_ms = float(step_ms.sum())
    total_ms_max = max_over_ranks(total_ms, dist, local)
    value = world * args.steps / (total_ms_max * 1e-3)
    # roofline of the dominant kernel inside the timed region: algorithmic
    # bytes of every PCG launch of the timed steps / their CUDA-event time
    launch_bytes = pcg_launch_bytes(n_n, iters.reshape(-1)).sum()
    pcg_total = float(pcg_ms.sum())
    achieved = launch_bytes / (pcg_total * 1e-3) / 1e9 if pcg_total > 0 else 0.0
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak, "traffic": traffic_for("cfg2", iters.reshape(-1)),
                "traffic_source": "profiles/traffic.json (ncu dram__bytes_read+write per iteration) x this "
                                  "run's mean iterations per launch",
                "kernel": kname, "kernel_grid": kgrid,
                "peak_kind": peak_kind, "pcg_share_of_step": pcg_total / total_ms,
                "pcg_launches": int(iters.size), "pcg_iterations": int(iters.sum()),
                "bytes_per_iteration": 72.0 * n_n,
                "us_per_iteration": 1000.0 * pcg_total / max(int(iters.sum()), 1),
                "algorithmic_bytes": "72 B per dof per iteration (9 fp64 streams) + 32 B/dof initial residual "
                                     "+ 24 B/dof final x update per launch (pcg_launch_bytes)"}
    op.grid.close()
    ens = None
    if not args.skip_secondary:
        ens = ensemble_members(dist, world, rank, local)
    line = None
    if rank == 0:
        # the device leg's steps, host-timed three times from a fresh
        # operator; the median run is reported
        e2e_runs = [time_e2e(problem, spec, args.warmup, args.steps) for _ in range(3)]
        e2e_vals = [r[0] for r in e2e_runs]
        e2e_v = float(np.median(e2e_vals))
        _, e2e_s, h2d, d2h = e2e_runs[int(np.argsort(e2e_vals)[1])]
        cfg1 = cfg1_pod = roof4 = steps4 = None
        if not args.skip_secondary:
            cfg1 = cfg_steps(1, warmup=args.warmup, steps=args.steps, with_roofline=hbm_peak)
            cfg1_pod = cfg_steps(1, warmup=args.warmup, steps=args.steps, strategy="pod")
        if not args.skip_cfg4:
            roof4 = cfg_pcg_roofline(4, hbm_peak, reps=1)
            steps4 = cfg_steps(4, warmup=1, steps=2)
        cpu = None
        if world == 1 and not args.skip_cpu:
            v, el, sample, parts, _ = cpu_sampled_steps(2, "pod", args.warmup, args.steps)
            hi = host_info()
            cpu = {"value": v, "unit": UNIT, "cores": hi["cores"], "kind": "port", "sample": sample,
                   "host": hi, "parts": parts}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (SURVEY 8(d) geometry: two iron blocks + annular coil)",
            "config": {"workload": "cfg2_128cube_two_blocks_pod30", "grid": [128, 128, 128],
                       "n_n": n_n, "n_c": n_c, "strategy": "pod", "n_pod": spec.n_pod, "eps_pod": 1e-4,
                       "rel_tol": spec.rel_tol, "dt": spec.dt,
                       "steps_timed": [args.warmup + 1, args.warmup + args.steps],
                       "l2": "flushed (256 MB write) before every timed step" if not args.no_flush else "not flushed",
                       "parallelism": f"replicas{world} (configs 0-2 do not shard; no collectives)"},
            "timed_step_iterations": iters.tolist(),
            "clocks": clk.summary(),
            "roofline": roofline,
            "cfg1_cspe_steps": cfg1,
            "cfg1_pod_steps": cfg1_pod,
            "roofline_cfg4_1gpu": roof4,
            "cfg4_steps_1gpu": steps4,
            "cfg4_sharded": None,
            "cfg3_ensemble": ens,
            "e2e": {"value": e2e_v, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "api": "explicit_euler_step + recover_an + probe_b (host arrays)",
                    "runs": e2e_vals, "estimator": "median of 3 runs of the timed steps"},
            "gpu_launches": launches,
            "cpu_baseline": cpu,
        }
    # configs[4] sharded over the job's ranks, last and under a watchdog: with
    # N > 1 its slab PCG waits on the peer GPUs (CUDA IPC, device mailboxes
    # with a 5 s watchdog of their own), and a rank that fails while the
    # others sit in a collective would otherwise hold the job -- on expiry
    # rank 0 prints the line with the leg marked and every rank exits
    if not args.skip_cfg4:
        leg = {"workload": "cfg4_256cube_two_blocks_cspe5_sharded", "ranks": world}

        def expire():
            if line is not None:
                line["cfg4_sharded"] = dict(leg, error=f"watchdog: not done after {SHARDED_DEADLINE_S} s")
                print(json.dumps(line), flush=True)
            os._exit(0)

        dog = threading.Timer(SHARDED_DEADLINE_S, expire)
        dog.daemon = True
        dog.start()
        barrier(dist)
        try:
            sharded = cfg4_sharded(dist, world, local, hbm_peak)
        except Exception as exc:  # noqa: BLE001  (reported, never silently dropped)
            sharded = dict(leg, error=f"{type(exc).__name__}: {exc}")
        dog.cancel()
        if line is not None:
            line["cfg4_sharded"] = sharded
    if line is not None:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--skip-secondary", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-cfg4", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_device_arm(args)


if __name__ == "__main__":
    sys.exit(main())
