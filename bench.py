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


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return dict(hbm=float(d["hbm_gbs"]), sm_mhz=float(d.get("sm_max_mhz", 1965.0)), src="measured",
                    bf16_tflops=d.get("bf16_tflops"))
    return dict(hbm=6650.0, sm_mhz=1965.0, src="fallback", bf16_tflops=None)


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


def host_info():
    """nproc + the CPU model (lscpu), for the cpu_baseline record."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def cpu_oracle_rate(wl, budget_s):
    """The fp64 oracle as it stands, on bounded samples of the workload (1 core: it is sequential).

    The sample is 8 windows of n steps spread evenly over the sequence (window k starts at k*T/8), each
    run as its own sequence (smoother + Viterbi), cycled until the budget is spent."""
    import oracle
    T = wl.T
    n = min(T, 200_000)
    nw = 8 if T >= 8 * n else 1
    wins = [np.ascontiguousarray(wl.log_lik[(k * T) // nw:(k * T) // nw + n]) for k in range(nw)]
    done, t0 = 0, time.perf_counter()
    reps = 0
    while True:
        ll = wins[reps % nw]
        oracle.smooth(wl.log_pi, wl.log_A, ll)
        oracle.viterbi(wl.log_pi, wl.log_A, ll)
        done += n
        reps += 1
        el = time.perf_counter() - t0
        if el >= budget_s:
            break
    return done / el, (f"{nw} windows of {n} steps spread over the T={T:g} workload (window k at k*T/{nw}), "
                       f"smoother+viterbi, {reps} window runs, {el:.1f}s"), 1


def time_ops(H, wl, dev, steps, warmup, flush):
    """Device time (ms, mean over `steps`, CUDA events on the launching stream, L2 flushed between steps
    outside the events) of hmm_smooth and hmm_viterbi on one workload, inputs resident in HBM."""
    import torch
    lp = torch.from_numpy(wl.log_pi).to(dev)
    la = torch.from_numpy(wl.log_A).to(dev)
    ll = torch.from_numpy(wl.log_lik).to(dev)
    batched = ll.dim() == 3
    B = ll.shape[0] if batched else 1
    T, D = ll.shape[-2], ll.shape[-1]
    out_s = (torch.empty_like(ll), torch.empty_like(ll), torch.empty(B, dtype=torch.float64, device=dev),
             torch.empty(B, dtype=torch.int32, device=dev))
    out_v = (torch.empty(ll.shape[:-1], dtype=torch.int32, device=dev),
             torch.empty(B, dtype=torch.float64, device=dev), torch.empty(B, dtype=torch.int32, device=dev))
    ws_s = H.workspace(H.HMM_OP_SMOOTH, D, T, B, dev)
    ws_v = H.workspace(H.HMM_OP_VITERBI, D, T, B, dev)
    stream = torch.cuda.current_stream(dev)
    for _ in range(warmup):
        flush()
        H.smooth(lp, la, ll, out=out_s, ws=ws_s)
        H.viterbi(lp, la, ll, out=out_v, ws=ws_v)
    torch.cuda.synchronize()
    assert int(out_s[3].abs().max().item()) == 0 and int(out_v[2].abs().max().item()) == 0
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
    for k in range(steps):
        flush()
        ev[k][0].record(stream)
        H.smooth(lp, la, ll, out=out_s, ws=ws_s)
        ev[k][1].record(stream)
        H.viterbi(lp, la, ll, out=out_v, ws=ws_v)
        ev[k][2].record(stream)
    torch.cuda.synchronize()
    ms_s = sum(e[0].elapsed_time(e[1]) for e in ev) / steps
    ms_v = sum(e[1].elapsed_time(e[2]) for e in ev) / steps
    del out_s, out_v, ll
    return ms_s, ms_v, B, T, D


def config_lines(H, dev, steps, warmup, flush, peaks):
    """The rest of BASELINE's metric ("at D=4 and D=64"): configs[1] (GE D=4, T=1e6), configs[2] (dense
    D=64, T=1e5) and configs[3] (B=1024, D=16, T=4096), each smoother and Viterbi device-timed with a
    roofline: HBM for the D=4 smoother, the FP32 pipe (effective algorithmic flops) and the
    tensor pipe for the D>=16 sum-product, the derived FADD/FMNMX3 issue ceiling for max-plus."""
    import workloads as W
    clk = peaks["sm_mhz"] * 1e6
    fp32_peak = 2 * 148 * 128 * clk / 1e12                         # TFLOP/s, FFMA
    tf32_peak = peaks["bf16_tflops"] * 0.5 if peaks.get("bf16_tflops") else None  # guide: TF32 = BF16 / 2
    out = {}
    for key, wl, desc in (
            ("configs[1]", W.ge(1_000_000, seed=1), "Gilbert-Elliott D=4, T=1e6, one sequence"),
            ("configs[2]", W.dense(64, 100_000, seed=3), "dense Dirichlet(1) D=64, T=1e5, Gaussian emissions"),
            ("configs[3]", W.dense_batch(1024, 16, 4096), "B=1024 sequences, D=16, T=4096, shared dense model")):
        ms_s, ms_v, B, T, D = time_ops(H, wl, dev, steps, warmup, flush)
        n = B * T
        rec = {"workload": desc, "D": D, "T": T, "B": B,
               "smoother_ms": ms_s, "viterbi_ms": ms_v,
               "smoother_steps_per_s": n / (ms_s * 1e-3), "viterbi_steps_per_s": n / (ms_v * 1e-3),
               "value": n / ((ms_s + ms_v) * 1e-3)}
        vops = D ** 3 + D * D * (D - 1)  # max-plus: D^3 adds + D^2 (D-1) 2-input max comparisons per step
        # issue ceiling: adds as FADD2 (2 lane-adds per lane-issue) and maxima as FMNMX3
        # (2 comparisons per lane-issue) share 128 lane-issues/clk/SM -> clk per step per SM:
        v_clk = (D ** 3 / 2 + D * D * (D - 1) / 2) / 128
        v_ceiling = 148 * clk / v_clk  # steps/s
        rec["viterbi_roofline"] = {"bound": "alu", "achieved": n / (ms_v * 1e-3), "peak": v_ceiling,
                                   "unit": "time-steps/s", "frac": n / (ms_v * 1e-3) / v_ceiling,
                                   "ops_per_step": vops, "ceiling": "FADD2 + FMNMX3 issue, 128 lane-issues/clk/SM"}
        if D <= 8:  # the algorithmic 20 B/step at the HBM peak is the larger floor at small D
            ach = VITERBI_BYTES_PER_STEP(D) * n / (ms_v * 1e-3) / 1e9
            rec["viterbi_roofline"] = {"bound": "hbm", "achieved": ach, "peak": peaks["hbm"], "unit": "GB/s",
                                       "frac": ach / peaks["hbm"], "bytes_per_step": VITERBI_BYTES_PER_STEP(D),
                                       "alu_frac": n / (ms_v * 1e-3) / v_ceiling}
        if D <= 8:
            ach = SMOOTH_BYTES_PER_STEP(D) * n / (ms_s * 1e-3) / 1e9
            rec["smoother_roofline"] = {"bound": "hbm", "achieved": ach, "peak": peaks["hbm"], "unit": "GB/s",
                                        "frac": ach / peaks["hbm"], "bytes_per_step": SMOOTH_BYTES_PER_STEP(D)}
        else:
            flop = 2 * D ** 3 + 4 * D * D  # one semiring product per step + two D^2 sweeps
            ach = flop * n / (ms_s * 1e-3) / 1e12
            r = {"bound": "tensor" if D >= 33 else "fp32", "achieved": ach, "unit": "TFLOP/s",
                 "flop_per_step": flop, "fp32_peak": fp32_peak, "frac_fp32": ach / fp32_peak}
            if D >= 33 and tf32_peak:
                # the contraction runs as TF32x3 (3 MMAs per product): pipe-level achieved = 3x
                r.update({"peak": tf32_peak, "frac": ach / tf32_peak, "tensor_pipe_frac": 3 * ach / tf32_peak,
                          "peak_source": "measured bf16 x 0.5 (TF32/BF16 nominal ratio)"})
            else:
                r.update({"peak": fp32_peak, "frac": ach / fp32_peak})
            if key == "configs[3]":
                # the planner runs the batch-parallel recursions here: they execute
                # ~4 D^2 flop/step (forward + backward dot products), not the scan's 2 D^3; `frac` above is
                # the scan-equivalent rate of SURVEY §8(d), `executed_frac` the rate of the work done
                ex = 4 * D * D
                r.update({"executed_flop_per_step": ex,
                          "executed_frac": ex * n / (ms_s * 1e-3) / 1e12 / fp32_peak,
                          "note": "latency-bound recursions (bidirectional batch plan); frac is scan-equivalent"})
            rec["smoother_roofline"] = r
        out[key] = rec
    return out


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
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample, **host_info()},
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
    ap.add_argument("--no-configs", action="store_true", help="skip the configs[1..3] sub-objects")
    ap.add_argument("--e2e-full-steps", type=int, default=3)
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
            torch.cuda.nvtx.range_push(f"step{k}")  # NVTX ranges for nsys / ncu timelines
            ev[k][0].record(stream)
            torch.cuda.nvtx.range_push("hmm_smooth")
            H.smooth(lp, la, ll, out=out_s, ws=ws_s)
            torch.cuda.nvtx.range_pop()
            ev[k][1].record(stream)
            torch.cuda.nvtx.range_push("hmm_viterbi")
            H.viterbi(lp, la, ll, out=out_v, ws=ws_v)
            torch.cuda.nvtx.range_pop()
            ev[k][2].record(stream)
            torch.cuda.nvtx.range_pop()
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
        # e2e_full: as e2e, plus the step's full results back to pinned host memory every step
        # (filtered + smoothed marginals and the MAP path: what a user who needs the outputs waits for)
        h_f = torch.empty(out_s[0].shape, dtype=torch.float32).pin_memory()
        h_s = torch.empty(out_s[1].shape, dtype=torch.float32).pin_memory()
        h_p = torch.empty(out_v[0].shape, dtype=torch.int32).pin_memory()

        def e2e_full_step():
            e2e_step()
            h_f.copy_(out_s[0], non_blocking=True); h_s.copy_(out_s[1], non_blocking=True)
            h_p.copy_(out_v[0], non_blocking=True)

        nfull = max(1, min(args.steps, args.e2e_full_steps))
        e2e_full_step()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(nfull):
            e2e_full_step()
        e1.record(stream)
        torch.cuda.synchronize()
        ms_full = e0.elapsed_time(e1) / nfull
        e2e["full"] = {"value": T / (ms_full * 1e-3), "unit": UNIT, "ms_per_step": ms_full, "steps": nfull,
                       "h2d_bytes_per_step": e2e["h2d_bytes_per_step"],
                       "d2h_bytes_per_step": int(h_out.numel() * 8 + (h_f.numel() + h_s.numel() + h_p.numel()) * 4),
                       "note": "H2D of log_lik + smooth + viterbi + D2H of filtered, smoothed, path and scalars"}
        del h_ll, d_ll, h_f, h_s, h_p
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
    kname = lambda op: ("hmm_stream_kernel" if H.plan(op, D, T)["fused"] == 2 else "hmm_small_kernel") + f"<{D},{op}>"
    roof_s = {"kernel": kname(0) + " (smoother)", "bound": "hbm", "achieved": ach_s,
              "peak": peaks["hbm"], "unit": "GB/s", "frac": ach_s / peaks["hbm"],
              "traffic": traffic.get("smooth", {}).get("dram_bytes_per_launch"),
              "peak_source": peaks["src"], "ms_per_launch": ms_s, "algorithmic_bytes_per_launch": sm_bytes}
    # Viterbi at D <= 8: of its two floors -- the algorithmic 20 B/step at the HBM peak and the max-plus
    # fold's FADD2 + FMNMX3 issue ceiling (config_lines) -- the HBM one is the larger, so it is the bound.
    v_clk = (D ** 3 / 2 + D * D * (D - 1) / 2) / 128
    v_alu_ceiling = 148 * peaks["sm_mhz"] * 1e6 / v_clk
    roof_v = {"kernel": kname(1) + " (viterbi)", "bound": "hbm", "achieved": ach_v,
              "peak": peaks["hbm"], "unit": "GB/s", "frac": ach_v / peaks["hbm"],
              "alu_frac": (T / (ms_v * 1e-3)) / v_alu_ceiling,
              "traffic": traffic.get("viterbi", {}).get("dram_bytes_per_launch"), "ms_per_launch": ms_v,
              "algorithmic_bytes_per_launch": vi_bytes}
    dominant = roof_s if ms_s >= ms_v else roof_v
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v, sample, cores = cpu_oracle_rate(wl, args.cpu_budget)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample, **host_info()}
    configs = None
    if rank == 0 and world == 1 and not args.no_configs and args.workload == "ge" and T == 100_000_000:
        configs = config_lines(H, dev, max(10, min(args.steps, 50)), args.warmup, flush_l2, peaks)

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
            "configs": configs,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
