#!/usr/bin/env python
"""Benchmark of the parallel-scan HMM hot path on B200 (one JSON line on rank 0).

A "step" is one pass of the whole hot path over one batch of synthetic input: the parallel
sum-product smoother (filtered + smoothed marginals + log Z, hmm_smooth) followed by the parallel
max-product MAP path (hmm_viterbi) on the same sequence.  Default workload = BASELINE.json configs[4],
the configuration the north-star target is quoted on: one Gilbert-Elliott channel HMM sequence
(PAPER.md:791-836), D=4, T=1e8, partitioned along T across the N GPUs (strong scaling; N=1 runs the
whole sequence on one B200 -- it fits: 1.6 GB in, 3.6 GB out).  `--T 1000000` gives configs[1].

  value   time-steps/s of the device-timed step (CUDA events on the launching stream, inputs resident
          in HBM, L2 flushed between timed steps); N>1: the split-phase smoother + Viterbi with their
          NCCL all-gathers (the method's one exchange step), total T / max-over-ranks step time.
  e2e     the same metric through the public Python API with pinned HOST buffers: H2D of log_lik,
          smooth + viterbi, D2H of log Z / log_prob / info, every step.
  roofline  the dominant kernel vs the measured HBM copy peak (MEASURED_PEAKS.json), plus the Viterbi
          kernel vs the FP32-pipe ALU peak derived in DESIGN.md.
  cpu_baseline  the fp64 oracle (oracle/, sequential C) on the host, bounded sample.

`--impl reference` times the oracle as it stands on the host cores (this tier's reference arm).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "time-steps/sec for smoother and Viterbi at D=4 and D=64; % of HBM/FP32 peak"
UNIT = "time-steps/s"
L2_FLUSH_BYTES = 512 << 20
# Algorithmic work per time step (DESIGN.md §"Roofline accounting").
SMOOTH_BYTES_PER_STEP = lambda D: 12 * D      # read log_lik (4D) + write filtered + smoothed (8D)
VITERBI_BYTES_PER_STEP = lambda D: 4 * D + 4  # read log_lik + write int32 path
VITERBI_ALU_PER_STEP = lambda D: D ** 3 + D * D * ((D - 1 + 1) // 2) + 2 * D * D  # leaf max-plus + sweep


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return dict(hbm=float(d["hbm_gbs"]), sm_mhz=float(d.get("sm_max_mhz", 1965.0)), src="measured")
    return dict(hbm=6650.0, sm_mhz=1965.0, src="fallback")


def ncu_traffic():
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {}


class ClockSampler:
    """Samples SM clock + throttle reasons via NVML during the timed region."""

    def __init__(self, dev_index=0, period=0.01):
        self.samples, self.reasons, self.period, self.dev_index = [], set(), period, dev_index
        self._stop = threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001 - clocks are diagnostics
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {
            getattr(nv, "nvmlClocksEventReasonGpuIdle", 0x1): "gpu_idle",
            getattr(nv, "nvmlClocksEventReasonApplicationsClocksSetting", 0x2): "applications_clocks_setting",
            getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4): "sw_power_cap",
            getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8): "hw_slowdown",
            getattr(nv, "nvmlClocksEventReasonSyncBoost", 0x10): "sync_boost",
            getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20): "sw_thermal_slowdown",
            getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40): "hw_thermal_slowdown",
            getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80): "hw_power_brake_slowdown",
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in names.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def make_workload(args, rank):
    import workloads as W
    if args.workload == "ge":
        cfg = "BASELINE configs[4]" if args.T == 100_000_000 else ("BASELINE configs[1]" if args.T == 1_000_000 else "GE")
        return W.ge(args.T, seed=5), f"{cfg}: Gilbert-Elliott D=4, T={args.T:g}, one sequence, smoother+viterbi"
    if args.workload == "dense":
        return W.dense(args.D, args.T, seed=3 + 1000 * rank), f"dense D={args.D} T={args.T:g} smoother+viterbi"
    raise SystemExit(f"unknown workload {args.workload}")


def cpu_oracle_rate(wl, budget_s):
    """The fp64 oracle as it stands, on bounded samples of the workload (1 core: it is sequential)."""
    import oracle
    T = wl.T
    n = min(T, 200_000)
    ll = np.ascontiguousarray(wl.log_lik[:n])
    done, t0 = 0, time.perf_counter()
    reps = 0
    while True:
        oracle.smooth(wl.log_pi, wl.log_A, ll)
        oracle.viterbi(wl.log_pi, wl.log_A, ll)
        done += n
        reps += 1
        el = time.perf_counter() - t0
        if el >= budget_s:
            break
    return done / el, f"first {n} steps of the workload, smoother+viterbi, {reps} reps, {el:.1f}s", 1


def run_reference(args):
    """--impl reference: the oracle (this tier's reference arm) timed on the host, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    wl, desc = make_workload(args, 0)
    import oracle
    n = min(wl.T, args.ref_sample)
    ll = np.ascontiguousarray(wl.log_lik[:n])
    for _ in range(args.warmup):
        oracle.smooth(wl.log_pi, wl.log_A, ll); oracle.viterbi(wl.log_pi, wl.log_A, ll)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.smooth(wl.log_pi, wl.log_A, ll); oracle.viterbi(wl.log_pi, wl.log_A, ll)
    el = time.perf_counter() - t0
    v = n * args.steps / el
    sample = f"each step = oracle smoother+viterbi on the first {n} of {wl.T} steps"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": desc, "D": wl.D, "T": wl.T, "B": 1},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def run_multi(args, world, rank, local):
    """N > 1: one GE sequence of T steps partitioned along T (rank r owns ~T/N steps); every step
    runs the split-phase smoother and Viterbi with their NCCL all-gathers (the method's exchange step).
    Strong scaling: total work fixed, value = T / max-over-ranks step time."""
    import torch
    import torch.distributed as dist
    import workloads as W
    from paper_2102_05743_b200 import dist as HD

    ndev = torch.cuda.device_count()
    dev = torch.device("cuda", local % max(ndev, 1))
    torch.cuda.set_device(dev)
    if args.dist_backend == "nccl":
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group("gloo")
    Tg = args.T
    wl = W.ge(Tg, seed=5)  # counter-based RNG: every rank simulates the same global chain
    t0, n = HD.partition(Tg, world, rank)
    D = wl.D
    lp = torch.from_numpy(wl.log_pi).to(dev)
    la = torch.from_numpy(wl.log_A).to(dev)
    ll = torch.from_numpy(np.ascontiguousarray(wl.log_lik[t0:t0 + n])).to(dev)
    stream = torch.cuda.current_stream(dev)

    flush_w = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)

    def step():
        # smoother + MAP path of the same slice, 5 library launches and 2 merged NCCL all-gathers
        f, s, lz, info, path, lpr, vinfo = HD.smooth_viterbi_dist(lp, la, ll, t0)
        return lz, info, lpr, vinfo

    for _ in range(args.warmup):
        flush_w.zero_()
        out = step()
    torch.cuda.synchronize()
    assert int(out[1].item()) == 0 and int(out[3].item()) == 0
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    dist.barrier()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(dev.index) as clk:
        for k in range(args.steps):
            flush_w.zero_()  # 512 MiB write: the per-rank slice does not stay in L2 between steps
            evs[k][0].record(stream)
            step()
            evs[k][1].record(stream)
        torch.cuda.synchronize()
    dist.barrier()
    ms = sum(a.elapsed_time(b) for a, b in evs) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if args.dist_backend == "nccl":
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    else:
        tc = t.cpu(); dist.all_reduce(tc, op=dist.ReduceOp.MAX); t = tc
    ms = float(t.item())
    # e2e: H2D of the local slice from pinned memory + the step + D2H of the scalars
    h_ll = torch.from_numpy(np.ascontiguousarray(wl.log_lik[t0:t0 + n])).pin_memory()
    h_out = torch.empty(2, dtype=torch.float64).pin_memory()

    def e2e_step():
        ll.copy_(h_ll, non_blocking=True)
        lz, info, lpr, vinfo = step()
        h_out.copy_(torch.cat([lz, lpr]), non_blocking=True)

    for _ in range(args.warmup):
        e2e_step()
    torch.cuda.synchronize()
    dist.barrier()
    e0.record(stream)
    for _ in range(args.steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    te = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device=dev)
    if args.dist_backend == "nccl":
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    else:
        tc = te.cpu(); dist.all_reduce(tc, op=dist.ReduceOp.MAX); te = tc
    ms_e2e = float(te.item())
    peaks = load_peaks()
    ach = (SMOOTH_BYTES_PER_STEP(D) + VITERBI_BYTES_PER_STEP(D)) * n / (ms * 1e-3) / 1e9  # per GPU, whole step
    if rank == 0:
        cfg = "BASELINE configs[4]: " if Tg == 100_000_000 else ""
        print(json.dumps({
            "metric": METRIC, "value": Tg / (ms * 1e-3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{cfg}Gilbert-Elliott D=4, one sequence of T={Tg:g} steps partitioned along T "
                                   f"across {world} ranks (split-phase smoother+viterbi, NCCL all-gather of rank "
                                   f"aggregates)",
                       "D": D, "T_global": Tg, "T_per_rank": n, "B": 1, "collective": args.dist_backend,
                       "l2": "flushed between timed steps (512 MiB write, outside the events)"},
            "roofline": {"kernel": "whole split-phase step per GPU (smoother+viterbi), algorithmic bytes "
                                   f"{SMOOTH_BYTES_PER_STEP(D) + VITERBI_BYTES_PER_STEP(D)} B/step", "bound": "hbm",
                         "achieved": ach, "peak": peaks["hbm"], "unit": "GB/s", "frac": ach / peaks["hbm"],
                         "traffic": None},
            "cpu_baseline": None,
            "e2e": {"value": Tg / (ms_e2e * 1e-3), "unit": UNIT, "h2d_bytes_per_step": int(h_ll.numel() * 4),
                    "d2h_bytes_per_step": 16, "ms_per_step": ms_e2e},
            "gpu_launches": 7 * args.steps, "clocks": clk.summary(),
            "smoother_viterbi_split": "7 library launches (5 phases + hmm_dist_pack + hmm_dist_combine) + 2 NCCL "
                                      "all-gathers per step (merged collectives)",
        }), flush=True)
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="ge", choices=["ge", "dense"])
    ap.add_argument("--T", type=int, default=100_000_000, help="time steps (1e8 = configs[4], 1e6 = configs[1])")
    ap.add_argument("--D", type=int, default=4)
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--ref-sample", type=int, default=100_000)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo only for single-GPU multi-process smoke runs")
    ap.add_argument("--force-dist", action="store_true",
                    help="run the split-phase (multi-GPU) path even with one rank (tests the NCCL plumbing)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist
    import paper_2102_05743_b200 as H

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 or args.force_dist:
        if not dist.is_initialized() and world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29511")
            os.environ.setdefault("RANK", "0"); os.environ.setdefault("WORLD_SIZE", "1")
        run_multi(args, world, rank, local)
        return
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    wl, desc = make_workload(args, rank)
    D, T = wl.D, wl.T
    lp = torch.from_numpy(wl.log_pi).to(dev)
    la = torch.from_numpy(wl.log_A).to(dev)
    ll = torch.from_numpy(wl.log_lik).to(dev)
    stream = torch.cuda.current_stream(dev)
    out_s = (torch.empty_like(ll), torch.empty_like(ll), torch.empty(1, dtype=torch.float64, device=dev),
             torch.empty(1, dtype=torch.int32, device=dev))
    out_v = (torch.empty(T, dtype=torch.int32, device=dev), torch.empty(1, dtype=torch.float64, device=dev),
             torch.empty(1, dtype=torch.int32, device=dev))
    ws_s = H.workspace(H.HMM_OP_SMOOTH, D, T, 1, dev)
    ws_v = H.workspace(H.HMM_OP_VITERBI, D, T, 1, dev)
    flush_w = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    flush_r = torch.ones(L2_FLUSH_BYTES // 8, dtype=torch.float32, device=dev)
    flush_acc = torch.zeros((), dtype=torch.float32, device=dev)

    def flush_l2():
        # write a buffer 4x the L2 (the contract), then read another 2x-L2 buffer so the dirty lines are
        # written back here rather than inside the next timed kernel: L2 is cold AND clean.
        flush_w.zero_()
        flush_acc.copy_(flush_r.sum())

    def step():
        H.smooth(lp, la, ll, out=out_s, ws=ws_s)
        H.viterbi(lp, la, ll, out=out_v, ws=ws_v)

    for _ in range(args.warmup):
        flush_l2()
        step()
    torch.cuda.synchronize()
    assert int(out_s[3].item()) == 0 and int(out_v[2].item()) == 0

    # ---- device-timed region: K steps, L2 flushed between steps (outside the events)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush_l2()
            ev[k][0].record(stream)
            H.smooth(lp, la, ll, out=out_s, ws=ws_s)
            ev[k][1].record(stream)
            H.viterbi(lp, la, ll, out=out_v, ws=ws_v)
            ev[k][2].record(stream)
        torch.cuda.synchronize()
        # keep sampling a little longer on very short regions
        if len(clk.samples) < 5:
            time.sleep(0.06)
    if world > 1:
        dist.barrier()
    t_s = [ev[k][0].elapsed_time(ev[k][1]) for k in range(args.steps)]
    t_v = [ev[k][1].elapsed_time(ev[k][2]) for k in range(args.steps)]
    ms_step = (sum(t_s) + sum(t_v)) / args.steps
    ms_s, ms_v = sum(t_s) / args.steps, sum(t_v) / args.steps
    if world > 1:
        t = torch.tensor([ms_step, ms_s, ms_v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step, ms_s, ms_v = [float(x) for x in t.cpu()]
    value = T / (ms_step * 1e-3)

    # ---- e2e through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        h_ll = torch.from_numpy(wl.log_lik).pin_memory()
        h_lp = torch.from_numpy(wl.log_pi).pin_memory()
        h_la = torch.from_numpy(wl.log_A).pin_memory()
        h_out = torch.empty(4, dtype=torch.float64).pin_memory()
        d_ll = torch.empty_like(ll); d_lp = torch.empty_like(lp); d_la = torch.empty_like(la)
        d_out = torch.empty(4, dtype=torch.float64, device=dev)

        def e2e_step():
            d_ll.copy_(h_ll, non_blocking=True); d_lp.copy_(h_lp, non_blocking=True)
            d_la.copy_(h_la, non_blocking=True)
            f, s, lz, info = H.smooth(d_lp, d_la, d_ll, out=out_s, ws=ws_s)
            p, lpr, vinfo = H.viterbi(d_lp, d_la, d_ll, out=out_v, ws=ws_v)
            d_out[0] = lz[0]; d_out[1] = lpr[0]; d_out[2] = info[0]; d_out[3] = vinfo[0]
            h_out.copy_(d_out, non_blocking=True)

        for _ in range(args.warmup):
            e2e_step()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        ms_e2e = e0.elapsed_time(e1) / args.steps
        if world > 1:
            t = torch.tensor([ms_e2e], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms_e2e = float(t.item())
        e2e = {"value": T / (ms_e2e * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(h_ll.numel() * 4 + h_lp.numel() * 4 + h_la.numel() * 4),
               "d2h_bytes_per_step": int(h_out.numel() * 8), "ms_per_step": ms_e2e,
               "note": "PCIe-bound: the step's log_lik (16 B/step) crosses the host link every step"}
        del h_ll, d_ll
        # the same GE sequence through the symbol-input API: a GE user holds the
        # channel outputs y (1 B/step) and the emission matrix, not log_lik
        if args.workload == "ge":
            import workloads as W
            wsym = W.ge_symbols(T, seed=5)
            h_y = torch.from_numpy(wsym.y).pin_memory()
            h_lb = torch.from_numpy(wsym.log_B).pin_memory()
            d_y = torch.empty_like(h_y, device=dev); d_lb = torch.empty_like(h_lb, device=dev)

            def e2e_sym_step():
                d_y.copy_(h_y, non_blocking=True); d_lb.copy_(h_lb, non_blocking=True)
                d_lp.copy_(h_lp, non_blocking=True); d_la.copy_(h_la, non_blocking=True)
                f, s, lz, info = H.smooth_symbols(d_lp, d_la, d_lb, d_y)
                p, lpr, vinfo = H.viterbi_symbols(d_lp, d_la, d_lb, d_y)
                d_out[0] = lz[0]; d_out[1] = lpr[0]; d_out[2] = info[0]; d_out[3] = vinfo[0]
                h_out.copy_(d_out, non_blocking=True)

            for _ in range(args.warmup):
                e2e_sym_step()
            torch.cuda.synchronize()
            assert int(h_out[2]) == 0 and int(h_out[3]) == 0
            e0.record(stream)
            for _ in range(args.steps):
                e2e_sym_step()
            e1.record(stream)
            torch.cuda.synchronize()
            ms_sym = e0.elapsed_time(e1) / args.steps
            e2e["symbols"] = {"value": T / (ms_sym * 1e-3), "unit": UNIT, "ms_per_step": ms_sym,
                              "h2d_bytes_per_step": int(h_y.numel() + h_lb.numel() * 4 + h_lp.numel() * 4 +
                                                        h_la.numel() * 4),
                              "d2h_bytes_per_step": int(h_out.numel() * 8),
                              "api": "smooth_symbols + viterbi_symbols (y uint8 + log_B)"}

    # ---- roofline (dominant kernel) + cpu baseline (rank 0, N=1 only)
    peaks = load_peaks()
    traffic = ncu_traffic()
    sm_bytes = SMOOTH_BYTES_PER_STEP(D) * T
    vi_bytes = VITERBI_BYTES_PER_STEP(D) * T
    ach_s = sm_bytes / (ms_s * 1e-3) / 1e9
    ach_v = vi_bytes / (ms_v * 1e-3) / 1e9
    alu_peak = 148 * 128 * peaks["sm_mhz"] * 1e6 / 1e12  # T lane-op/s
    ach_alu = VITERBI_ALU_PER_STEP(D) * T / (ms_v * 1e-3) / 1e12
    kname = lambda op: ("hmm_stream_kernel" if H.plan(op, D, T)["fused"] == 2 else "hmm_small_kernel") + f"<{D},{op}>"
    roof_s = {"kernel": kname(0) + " (smoother)", "bound": "hbm", "achieved": ach_s,
              "peak": peaks["hbm"], "unit": "GB/s", "frac": ach_s / peaks["hbm"],
              "traffic": traffic.get("smooth", {}).get("dram_bytes_per_launch"),
              "peak_source": peaks["src"], "ms_per_launch": ms_s, "algorithmic_bytes_per_launch": sm_bytes}
    roof_v = {"kernel": kname(1) + " (viterbi)", "bound": "alu", "achieved": ach_alu,
              "peak": alu_peak, "unit": "Tlane-op/s", "frac": ach_alu / alu_peak,
              "hbm_achieved_gbs": ach_v, "hbm_frac": ach_v / peaks["hbm"],
              "traffic": traffic.get("viterbi", {}).get("dram_bytes_per_launch"), "ms_per_launch": ms_v}
    dominant = roof_s if ms_s >= ms_v else roof_v
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v, sample, cores = cpu_oracle_rate(wl, args.cpu_budget)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": desc, "D": D, "T": T, "B": 1,
                       "l2": "flushed between timed steps (512 MiB write + 256 MiB read, outside the events)"},
            "smoother_steps_per_s": T / (ms_s * 1e-3),
            "viterbi_steps_per_s": T / (ms_v * 1e-3),
            "roofline": dominant, "roofline_all": [roof_s, roof_v],
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": 2 * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
