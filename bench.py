#!/usr/bin/env python
"""Benchmark: shifted solves/sec on BASELINE.json configs[3] (config 4:
IRKA-style interpolation, n=10000, m=p=20, 2000 complex shifts = 1000
conjugate pairs per GPU), FP64 / complex128 -- the largest configuration
that fits one GPU (config 5 is quoted sharded over 8 GPUs).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A "step" is one pass of the hot path over one batch: the transfer function
G(sigma) = C (sigma I - A)^{-1} B for all of this rank's shifts on a
device-resident controller-Hessenberg triple (reduced once, on the GPU, and
broadcast to every rank with NCCL), plus the all-gather of G at N > 1.  The
config's second operation, ``solve_shifted_reduced`` with unit-norm complex
Gaussian b_dirs on the same shifts, is timed the same way and reported under
``reduced``.  Weak scaling: rank r owns config 4's shift set drawn with seed
4 + r (rank 0 = exactly config 4).  The working set (Ahat 800 MB + 6.4 GB of
window state per rank) is far larger than the 126 MB L2, so no explicit L2
flush is needed between steps.

``--gpus N`` with N > 1 and no torchrun environment re-launches itself under
``torch.distributed.run`` (one process per GPU, 127.0.0.1 rendezvous).

Rank 0 prints ONE JSON line.  `--impl reference` times the reference
algorithm's CPU implementation (the C restatement in oracle/, all host
threads) on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "shifted solves/sec (n, m, #shifts) at 1/2/4/8 B200; % of FP64/HBM roofline"
DEFAULT_CFG = 4
WORKLOADS = {
    1: "config1: transfer function n=500, m=p=5, 100 i*omega shifts",
    2: "config2: Bode plot n=4000, m=p=10, 1000 i*omega shifts per GPU (log grid)",
    3: "config3: pseudospectrum-grid shifts n=2000, m=p=1, 100x100 grid",
    4: "config4: IRKA-style interpolation n=10000, m=p=20, 2000 complex shifts "
       "(1000 conjugate pairs) per GPU, transfer function G + solve_shifted_reduced",
    5: "config5: large-scale transfer function n=20000, m=p=50, 500 complex shifts per GPU",
}
# dominant (far-row update) kernel per m, as enqueue_part selects it
FAR_KERNEL = {10: "k_fark<1,8,4> (K-streamed far-row update: one pass per 4-block composite, "
                  "8 shifts x 64 rows per unit)",
              20: "k_fark<2,4,4> (K-streamed far-row update: one pass per 4-block composite, "
                  "4 shifts x 64 rows per unit)",
              1: "k_farkm<4> (window composites: one K-streamed pass per 8 windows, 80 shifts "
                 "per unit as columns) + the near rows' one-level k_far (all update launches)",
              50: "k_fark<5,3,2> (window composites: one K-streamed pass per 8 windows, 3 shifts "
                  "x 64 rows per unit) + the near rows' k_update (all update launches)"}


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--cfg", type=int, default=DEFAULT_CFG, choices=(1, 2, 3, 4, 5),
                    help="BASELINE.json config (default 4; the others are diagnostics)")
    ap.add_argument("--nb", type=int, default=64)
    ap.add_argument("--batch", type=int, default=0, help="shifts per device pass (0: auto)")
    ap.add_argument("--shifts", type=int, default=0, help="override shifts per GPU")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-reduced", action="store_true")
    ap.add_argument("--profile", action="store_true",
                    help="ncu mode: minimal untimed run, no baselines")
    ap.add_argument("--selftest-gloo", action="store_true",
                    help="CPU launcher test: gloo ranks, small system, stub per-rank solver")
    return ap.parse_args(argv)


# ---------------------------------------------------------------------------
# launcher: one process per GPU
# ---------------------------------------------------------------------------
def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def maybe_spawn(args) -> int | None:
    """``--gpus N > 1`` outside torchrun: re-exec under torch.distributed.run
    with N local ranks; returns the launcher's exit code (None: run here)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def world_info(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    return world, rank, local


# ---------------------------------------------------------------------------
# clocks (NVML during the timed region)
# ---------------------------------------------------------------------------
class Clocks:
    """SM clock and throttle-reason samples DURING the timed region: NVML
    polled from a thread every 5 ms, nvidia-smi as the fallback."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.stop_ev = None
        self.thread = None
        self.p = None
        self.f = None
        self.nv = None
        self.windows = []
        try:
            import pynvml
            pynvml.nvmlInit()
            try:
                import torch
                pr = torch.cuda.get_device_properties(index)
                bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
                self.h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.mx = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.nv = pynvml
        except Exception:
            self.nv = None

    def _poll(self):
        nv, h = self.nv, self.h
        get_r = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        mx = self.mx
        while True:
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                r = get_r(h)
                self.rows.append((float(sm), float(mx), int(r), time.perf_counter()))
            except Exception:
                pass
            if self.stop_ev.wait(0.005):
                break

    def start(self):
        """Start polling before the warm-up; begin()/end() mark timed regions."""
        if self.nv is not None:
            import threading
            self.rows = []
            self.stop_ev = threading.Event()
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return
        try:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def begin(self):
        self.windows.append([time.perf_counter(), None])

    def end(self):
        self.windows[-1][1] = time.perf_counter()

    def stop(self) -> dict:
        if self.thread is not None:
            self.stop_ev.set()
            self.thread.join(timeout=5)
            nv = self.nv
            win = [w for w in self.windows if w[1] is not None]
            if win:
                self.rows = [r for r in self.rows if any(a <= r[3] <= b for a, b in win)]
            if not self.rows:
                return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "source": "nvml"}
            bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
            reasons = sorted({k for _, _, r, _ in self.rows for k, b in bits.items() if r & b})
            sm = [r[0] for r in self.rows]
            mx = max(r[1] for r in self.rows)
            load = [v for v in sm if v >= 0.5 * mx] or sm
            return {"sm_mhz": statistics.median(load), "sm_max_mhz": mx, "reasons": reasons,
                    "samples": len(self.rows), "source": "nvml (5 ms poll, timed regions only)"}
        return self._stop_smi()

    def _stop_smi(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.p.kill()
        self.f.flush()
        rows = []
        with open(self.f.name) as fh:
            for line in fh:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4)
                          if r[5 + i].lower() in ("active", "1")})
        load = [v for v in sm if mx and v >= 0.5 * max(mx)] or sm
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


# ---------------------------------------------------------------------------
# workload
# ---------------------------------------------------------------------------
def workload(cfg: int, rank: int, shifts_override: int = 0):
    """(n, m, p, this rank's shifts) for a BASELINE.json config."""
    from paper_1708_06290_b200.systems import CONFIGS, config_shifts
    n, m, p, _ = CONFIGS[cfg]
    if cfg in (4, 5):
        sh = config_shifts(cfg, n, seed=cfg + rank)
        if cfg == 5:
            sh = sh[:500]  # 500 shifts per GPU
    else:
        sh = config_shifts(cfg, n)
    if shifts_override:
        reps = -(-shifts_override // len(sh))
        sh = np.tile(sh, reps)[:shifts_override]
    return n, m, p, np.ascontiguousarray(sh)


def synthetic_triple(n, m, p, seed):
    """m-Hessenberg Ahat / triangular Bhat / dense Chat of the config shape
    (the solve cost does not depend on the values)."""
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((n, n))
    A = np.triu(A, -m) - 1.1 * np.sqrt(n) * np.eye(n)
    B = np.zeros((n, m))
    B[:m, :m] = np.triu(rng.standard_normal((m, m))) + 2 * np.eye(m)
    C = rng.standard_normal((p, n))
    return np.asfortranarray(A), np.asfortranarray(B), np.asfortranarray(C)


def f_alg(n, m, p):
    """SURVEY 8(d) canonical flops per shift: every structural nonzero of
    [Chat; Ahat] meets the m complex columns once (4 flops per real x complex)."""
    return 2.0 * n * n * m + 4.0 * n * m * (m + p)


# ---------------------------------------------------------------------------
# CPU baseline / reference arm: the reference algorithm's C restatement
# ---------------------------------------------------------------------------
def _oracle_time(A, B, C, sample, nb, cores):
    from oracle import oracle as O
    t0 = time.perf_counter()
    O.tf_eval(A, B, C, sample, nb=nb, threads=cores)
    return time.perf_counter() - t0


def cpu_sample_size(A, B, C, shifts, nb, cores, budget_s):
    """Shifts (a multiple of `cores`) that take about `budget_s` of wall time."""
    probe = shifts[: max(1, min(len(shifts), cores))]
    per = _oracle_time(A, B, C, probe, nb, cores) / len(probe)
    k = int(budget_s / max(per, 1e-9))
    return max(len(probe), min(len(shifts), (k // cores) * cores if k >= cores else k))


def cpu_baseline(A, B, C, shifts, nb, cfg, budget_s: float = 15.0) -> dict:
    cores = os.cpu_count() or 1
    k = cpu_sample_size(A, B, C, shifts, nb, cores, budget_s)
    idx = np.linspace(0, len(shifts) - 1, k).astype(int)
    dt = _oracle_time(A, B, C, shifts[idx], nb, cores)
    return {"value": k / dt, "unit": "shifts/s", "cores": cores, "kind": "port",
            "sample": f"{k} of the {len(shifts)} config-{cfg} shifts (evenly spaced), same reduced "
                      f"triple, nb={nb}, oracle/shiftsolve_oracle.c (C restatement of the "
                      f"reference sweep) with OpenMP over {cores} threads, {dt:.1f} s"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    n, m, p, shifts = workload(args.cfg, 0, args.shifts)
    A, B, C = synthetic_triple(n, m, p, seed=args.cfg)
    cores = os.cpu_count() or 1
    # each step: a bounded sample (~8 s of host work) of the same workload
    k = cpu_sample_size(A, B, C, shifts, args.nb, cores, 8.0)
    idx = np.linspace(0, len(shifts) - 1, k).astype(int)
    sample = shifts[idx]
    for _ in range(args.warmup):
        _oracle_time(A, B, C, sample[:cores], args.nb, cores)
    times = [_oracle_time(A, B, C, sample, args.nb, cores) for _ in range(args.steps)]
    dt = statistics.mean(times)  # same statistic as our arm (mean over the K steps)
    value = len(sample) / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "shifts/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64 (complex128 shift arithmetic)",
        "data": "synthetic m-Hessenberg triple of the config shape (cost is value-independent)",
        "config": {"workload": WORKLOADS[args.cfg], "n": n, "m": m, "p": p, "nb": args.nb,
                   "shifts_per_step": len(sample)},
        "cpu_baseline": {"value": value, "unit": "shifts/s", "cores": cores, "kind": "port",
                         "sample": f"{len(sample)} of the {len(shifts)} config-{args.cfg} shifts "
                                   f"per step (evenly spaced), oracle/shiftsolve_oracle.c (C "
                                   f"restatement of the reference sweep), OpenMP over {cores} "
                                   f"threads, mean of {args.steps} steps"},
        "e2e": {"value": value, "unit": "shifts/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# CPU launcher self-test: gloo ranks through the same sharding code
# ---------------------------------------------------------------------------
def run_selftest_gloo(args):
    """Exercises the launcher, the world-size check, broadcast_chf, the
    contiguous shard and the all-gather of G on gloo (CPU); the per-rank
    device solver is stubbed by a dense numpy solve."""
    import torch
    import torch.distributed as dist

    from paper_1708_06290_b200 import ControllerHessForm
    from paper_1708_06290_b200.distributed import broadcast_chf, eval_transfer_function_sharded

    world, rank, _ = world_info(args)
    dist.init_process_group("gloo")
    n, m, p = 24, 3, 2
    chf0 = None
    if rank == 0:
        A, B, C = synthetic_triple(n, m, p, seed=7)
        chf0 = ControllerHessForm(Ahat=torch.from_numpy(A), Bhat=torch.from_numpy(B),
                                  Chat=torch.from_numpy(C), m=m, n=n, p=p)
    chf = broadcast_chf(chf0, torch.device("cpu"))
    shifts = 1j * np.linspace(1.0, 9.0, 10 * world)

    def stub(chf_, sh, nb, bs, rtol):
        A_ = chf_.Ahat.numpy()
        G = np.concatenate([-chf_.Chat.numpy() @ np.linalg.solve(A_ - s * np.eye(n), chf_.Bhat.numpy())
                            for s in sh], axis=1) if len(sh) else np.zeros((p, 0), complex)
        return G, {}

    t0 = time.perf_counter()
    res = eval_transfer_function_sharded(chf, shifts, nb=8, solver=stub)
    dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64)
    dist.all_reduce(dt, op=dist.ReduceOp.MAX)
    G_ref, _ = stub(chf, shifts, 8, None, None)
    err = float(np.abs(res.G.numpy() - G_ref).max() / np.abs(G_ref).max())
    if rank == 0:
        print(json.dumps({"selftest": "gloo", "n_gpus": world, "shifts": len(shifts),
                          "max_rel_err": err, "ms": float(dt.item()) * 1e3}), flush=True)
    dist.destroy_process_group()
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def main(argv=None):
    args = parse(argv)
    rc = maybe_spawn(args)
    if rc is not None:
        return rc
    if args.selftest_gloo:
        return run_selftest_gloo(args)
    if args.impl == "reference":
        return run_reference(args)

    import ctypes

    import torch
    import torch.distributed as dist

    import paper_1708_06290_b200 as ss
    from paper_1708_06290_b200 import _device as D
    from paper_1708_06290_b200 import _lib
    from paper_1708_06290_b200.distributed import (broadcast_chf, eval_transfer_function_sharded,
                                                   gather_slices)

    world, rank, local = world_info(args)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    cfg = args.cfg
    n, m, p, shifts_loc = workload(cfg, rank, args.shifts)
    s_loc = len(shifts_loc)
    s_total = s_loc * world
    lo = rank * s_loc  # weak scaling: equal contiguous slices

    h = _lib.handle(local)
    L = _lib.load()

    # ---- one-time: synthetic system, GPU reduction on rank 0, broadcast ----
    red_ms = None
    chf0 = None
    circular = n >= 10000
    if args.profile:
        # ncu mode: skip the reduction (tens of thousands of launches at
        # n = 10000); the sweep's cost does not depend on the values
        At, Bt, Ct = synthetic_triple(n, m, p, seed=cfg)
        chf0 = ss.ControllerHessForm(Ahat=torch.from_numpy(At).to(dev), Bhat=torch.from_numpy(Bt).to(dev),
                                     Chat=torch.from_numpy(Ct).to(dev), m=m, n=n, p=p)
        del At, Bt, Ct
    elif rank == 0:
        sysb = ss.random_stable_system(n, m, p, seed=cfg, circular=circular)
        A_d = torch.from_numpy(sysb.A).to(dev)
        B_d = torch.from_numpy(sysb.B).to(dev)
        C_d = torch.from_numpy(sysb.C).to(dev)
        del sysb
        ss.reduce_controller_hessenberg(A_d[:64, :64], B_d[:64, :4], C_d[:2, :64])  # warm
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        chf0 = ss.reduce_controller_hessenberg(A_d, B_d, C_d, block_size=64)
        e1.record()
        torch.cuda.synchronize()
        red_ms = e0.elapsed_time(e1)
        del A_d, B_d, C_d
    chf = broadcast_chf(chf0, dev) if world > 1 else chf0
    A, B, C = chf.Ahat, chf.Bhat, chf.Chat
    sh_d = torch.from_numpy(shifts_loc).to(dev)
    G = torch.empty((s_loc * m, p), dtype=torch.complex128, device=dev).t()
    fail = torch.empty(s_loc, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)
    nan = float("nan")

    def step():
        rc = L.ss_tf_eval(h.ptr, n, m, p, D.ptr(A), D.ld(A), D.ptr(B), D.ld(B), D.ptr(C), D.ld(C),
                          D.ptr(sh_d), s_loc, args.nb, args.batch, nan, D.ptr(G), p,
                          D.ptr(fail), ctypes.c_void_p(stream.cuda_stream))
        D.check(h, rc)
        if world > 1:
            gather_slices(G, {}, lo, s_total, m)

    if args.profile:
        step()
        torch.cuda.synchronize()
        return 0

    # the FP64 peak is the larger of the two measured paths (DFMA on the FP64
    # pipe, DMMA on the tensor pipe); on B200 both measure ~37 TFLOP/s, and
    # the sweep runs on DFMA (north_star: DMMA only in the reduction)
    peak, peak_d = ctypes.c_double(0.0), ctypes.c_double(0.0)
    D.check(h, L.ss_probe_dfma_peak(h.ptr, ctypes.byref(peak)))
    D.check(h, L.ss_probe_dmma_peak(h.ptr, ctypes.byref(peak_d)))
    fp64_peak = max(peak.value, peak_d.value)  # measured TFLOP/s on this box

    clk = Clocks(local)

    def timed(fn, steps):
        """Mean ms per step over `steps` back-to-back calls: CUDA events on
        the launching stream, barrier + synchronize on both sides, max over
        ranks."""
        barrier()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        clk.begin()
        ev0.record(stream)
        for _ in range(steps):
            fn()
        ev1.record(stream)
        torch.cuda.synchronize()
        clk.end()
        barrier()
        return max_over_ranks(ev0.elapsed_time(ev1) / steps)

    clk.start()  # polling thread up before the timed region opens
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- timed region: K steps, no instrumentation ----
    launches0 = h.launches()
    ms = timed(step, args.steps)
    launches = h.launches() - launches0
    value = s_total / (ms * 1e-3)

    # ---- instrumented pass: the same K steps with a CUDA event pair around
    # every kernel on its own stream (deferred resolution, no syncs), for the
    # per-kernel roofline and the reference phase split ----
    L.ss_reset_stats(h.ptr)
    L.ss_set_timing(h.ptr, 1)
    barrier()
    torch.cuda.synchronize()
    ev2, ev3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev2.record(stream)
    for _ in range(args.steps):
        step()
    ev3.record(stream)
    torch.cuda.synchronize()
    L.ss_set_timing(h.ptr, 0)
    ms_instr = ev2.elapsed_time(ev3) / args.steps
    ul, us, ua = ctypes.c_int64(0), ctypes.c_double(0.0), ctypes.c_double(0.0)
    L.ss_update_kernel_stats(h.ptr, ctypes.byref(ul), ctypes.byref(us), ctypes.byref(ua))
    sec5 = (ctypes.c_double * 5)()
    fl5 = (ctypes.c_double * 5)()
    L.ss_phase_stats(h.ptr, sec5, fl5)
    upd_avg_s = us.value / max(ul.value, 1)
    upd_alg = ua.value / max(ul.value, 1)
    achieved = upd_alg / upd_avg_s / 1e12 if upd_avg_s > 0 else 0.0
    step_gpu_s = sum(sec5[1:5])
    share = us.value / step_gpu_s if step_gpu_s > 0 else None
    fa = f_alg(n, m, p)
    sweep_tflops = fa * value / world / 1e12
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", "r2_far_traffic.json")
    if os.path.exists(tpath):
        try:
            rec = json.load(open(tpath)).get(f"cfg{cfg}")
            if rec:
                traffic, traffic_src = rec.get("dram_bytes_per_launch"), rec.get("what")
        except Exception:
            traffic = None

    # ---- the config's second operation: solve_shifted_reduced ----
    reduced = None
    if not args.no_reduced and cfg == 4:
        rng = np.random.default_rng(1000 + rank)
        bd_h = rng.standard_normal((m, s_loc)) + 1j * rng.standard_normal((m, s_loc))
        bd_h /= np.linalg.norm(bd_h, axis=0, keepdims=True)
        bd = torch.from_numpy(np.asfortranarray(bd_h)).to(dev).t().contiguous().t()
        X = torch.empty((s_loc, n), dtype=torch.complex128, device=dev).t()
        fail_r = torch.empty(s_loc, dtype=torch.int32, device=dev)

        def step_red():
            rc = L.ss_solve_reduced(h.ptr, n, m, D.ptr(A), D.ld(A), D.ptr(B), D.ld(B),
                                    D.ptr(sh_d), s_loc, D.ptr(bd), D.ld(bd), args.nb, args.batch,
                                    nan, D.ptr(X), n, D.ptr(fail_r),
                                    ctypes.c_void_p(stream.cuda_stream))
            D.check(h, rc)

        for _ in range(max(1, args.warmup)):
            step_red()
        torch.cuda.synchronize()
        ms_r = timed(step_red, args.steps)
        v_r = s_total / (ms_r * 1e-3)
        fa_r = 2.0 * n * n * m + 4.0 * n * m * (m + 1)  # [I; Ahat]: n identity nonzeros
        reduced = {"op": "solve_shifted_reduced (x_l = (Ahat - sigma_l I)^{-1} Bhat b_l, "
                         "unit-norm complex Gaussian b_dirs)",
                   "value": v_r, "unit": "shifts/s", "ms_per_step": ms_r,
                   "sweep_tflops": fa_r * v_r / world / 1e12,
                   "frac_of_fp64_peak": fa_r * v_r / world / 1e12 / fp64_peak if fp64_peak else None,
                   "failures": int((fail_r >= 0).sum().item())}
        del X, bd

    # ---- SURVEY 8(f) row 1 on the same shifts: solve_shifted_transposed ----
    # (IRKA's left solves; general complex right-hand sides, unit norm)
    transposed = None
    if not args.no_reduced and cfg == 4:
        rng = np.random.default_rng(2000 + rank)
        rhs_h = rng.standard_normal((n, s_loc)) + 1j * rng.standard_normal((n, s_loc))
        rhs_h /= np.linalg.norm(rhs_h, axis=0, keepdims=True)
        rhs = torch.from_numpy(np.asfortranarray(rhs_h)).to(dev).t().contiguous().t()
        del rhs_h
        Xt = torch.empty((s_loc, n), dtype=torch.complex128, device=dev).t()
        fail_t = torch.empty(s_loc, dtype=torch.int32, device=dev)

        def step_tr():
            rc = L.ss_solve_transposed(h.ptr, n, m, D.ptr(A), D.ld(A), D.ptr(sh_d), s_loc, D.ptr(rhs),
                                       D.ld(rhs), 32, args.batch, nan, D.ptr(Xt), n, D.ptr(fail_t),
                                       ctypes.c_void_p(stream.cuda_stream))
            D.check(h, rc)

        step_tr()
        torch.cuda.synchronize()
        k_t = max(1, min(args.steps, 3))
        ms_t = timed(step_tr, k_t)
        v_t = s_total / (ms_t * 1e-3)
        # structural nonzeros of [A^T; -I] (n^2 / 2 + n (m + 1) + n) meet the m + 1
        # state columns once at 4 flops each
        fa_t = 4.0 * (m + 1) * (n * n / 2.0 + n * (m + 2))
        transposed = {"op": "solve_shifted_transposed ((Ahat - sigma_l I)^T x_l = c_l, unit-norm "
                            "complex Gaussian c_l; SURVEY 8(f) row 1)",
                      "value": v_t, "unit": "shifts/s", "ms_per_step": ms_t, "steps": k_t,
                      "sweep_tflops": fa_t * v_t / world / 1e12,
                      "frac_of_fp64_peak": fa_t * v_t / world / 1e12 / fp64_peak if fp64_peak else None,
                      "failures": int((fail_t >= 0).sum().item())}
        del Xt, rhs

    # ---- IRKA on the config-4 system (reduced order 20) ----
    irka = None
    if not args.no_reduced and cfg == 4 and rank == 0:
        r_ord, iters = 20, 3
        ss.irka_iterate(chf, r_ord, maxiter=1, fixed_iters=True, nb=32)  # warm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, ist = ss.irka_iterate(chf, r_ord, maxiter=iters, fixed_iters=True, nb=32)
        torch.cuda.synchronize()
        ms_i = (time.perf_counter() - t0) * 1e3 / iters
        irka = {"op": f"irka_iterate (reduced order {r_ord}, {iters} fixed iterations; per iteration "
                      f"{r_ord} reduced + {r_ord} transposed shifted solves, device bases and "
                      "projections, host r x r pencil)",
                "ms_per_iteration": ms_i, "shifted_solves_per_s": 2 * r_ord / (ms_i * 1e-3),
                "timing": "host wall clock around the host-synchronous call (rank 0)",
                "perturbations": len(ist.perturbations)}

    # ---- e2e through the public API with pinned host buffers ----
    e2e = None
    if not args.no_e2e:
        # column-major pinned host copy: eval_transfer_function streams it to
        # the device in sweep order (ss_tf_eval_stream), overlapped with the sweep
        A_h = A.cpu().t().contiguous().t().pin_memory()
        assert A_h.stride(0) == 1 and A_h.is_pinned()
        B_h = B.cpu().pin_memory()
        C_h = C.cpu().pin_memory()
        sh_all = np.concatenate([workload(cfg, r, args.shifts)[3] for r in range(world)])
        sh_h = torch.from_numpy(sh_all).pin_memory()
        chf_h = ss.ControllerHessForm(Ahat=A_h, Bhat=B_h, Chat=C_h, m=m, n=n, p=p)

        def call():
            if world > 1:
                return eval_transfer_function_sharded(chf_h, sh_h, nb=args.nb, on_singular="mark")
            return ss.eval_transfer_function(chf_h, sh_h, nb=args.nb, on_singular="mark")

        call()
        k_e2e = max(3, min(args.steps, 5))
        barrier()
        torch.cuda.synchronize()
        clk.begin()
        t0 = time.perf_counter()
        for _ in range(k_e2e):
            r = call()
        t1 = time.perf_counter()
        clk.end()
        t_e2e = max_over_ranks((t1 - t0) / k_e2e)  # mean over the (host-synchronous) calls
        h2d = (n * n + n * m + p * n) * 8 + s_loc * 16
        d2h = p * m * s_loc * 16 + s_loc * 4
        e2e = {"value": s_total / t_e2e, "unit": "shifts/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": t_e2e * 1e3, "calls": k_e2e,
               "path": ("paper_1708_06290_b200.eval_transfer_function" if world == 1 else
                        "paper_1708_06290_b200.distributed.eval_transfer_function_sharded") +
                       "(pinned host torch tensors) -> ss_tf_eval_stream (Ahat H2D streamed in "
                       "sweep order on a copy stream, overlapped with the sweep); all inputs H2D "
                       "+ G/failures D2H inside the timed region"}
        del r

    clocks = clk.stop()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(np.asfortranarray(A.cpu().numpy()), np.asfortranarray(B.cpu().numpy()),
                           np.asfortranarray(C.cpu().numpy()), shifts_loc, args.nb, cfg)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "shifts/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64 (complex128 shift arithmetic)",
            "data": ("synthetic: seeded Gaussian A shifted by -1.1 sqrt(n) I (circular law, SURVEY "
                     "8(d) for n >= 10000)" if circular else
                     "synthetic: reference random_stable_system (systems.py:71-86)") +
                    ", Gaussian B, C; reduced on the GPU",
            "config": {"workload": WORKLOADS[cfg], "n": n, "m": m, "p": p,
                       "shifts_per_gpu": s_loc, "nb": args.nb,
                       "l2": "no flush: per-step working set (Ahat + window state) exceeds "
                             "the 126 MB L2",
                       "parallelism": f"shift-sharded x{world} (broadcast once, all-gather G)"},
            "roofline": {"bound": "fp64", "kernel": FAR_KERNEL.get(m, "far-row update (k_far / k_update)"),
                         "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
                         "frac": achieved / fp64_peak if fp64_peak else None,
                         "traffic": traffic, "traffic_source": traffic_src,
                         "peak_source": "max of the measured DFMA and DMMA peaks on this GPU "
                                        f"(ss_probe_dfma_peak {peak.value:.2f}, ss_probe_dmma_peak "
                                        f"{peak_d.value:.2f}); MEASURED_PEAKS.json has no FP64 entry",
                         "alg_flops_per_launch": upd_alg, "avg_launch_ms": upd_avg_s * 1e3,
                         "launches": int(ul.value), "share_of_step": share,
                         "timing": "CUDA event pair around every launch on its stream, in an "
                                   "instrumented repeat of the timed steps "
                                   f"({ms_instr:.2f} ms/step instrumented vs {ms:.2f} clean)"},
            "sweep_roofline": {"bound": "fp64", "achieved": sweep_tflops, "peak": fp64_peak,
                               "unit": "TFLOP/s",
                               "frac": sweep_tflops / fp64_peak if fp64_peak else None,
                               "f_alg_per_shift": fa},
            "reduced": reduced,
            "transposed": transposed,
            "irka": irka,
            "phase_seconds": {k: sec5[i] for i, k in enumerate(ss.counters.ALL_PHASES)},
            "reduction_ms": red_ms,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main() or 0)
