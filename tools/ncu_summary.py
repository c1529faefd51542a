"""Compact summary of an `ncu --set full` report (per kernel) + DRAM traffic per launch.

usage: python tools/ncu_summary.py report.ncu-rep [out_traffic.json] [T]
Prints duration, DRAM read/write bytes, achieved DRAM GB/s, issue activity, IPC, top stall reasons.
With out_traffic.json, writes {"smooth"|"viterbi": {"dram_bytes_per_launch": ..., ...}} for bench.py.
"""
import csv, io, json, subprocess, sys

rep = sys.argv[1]
out = sys.argv[2] if len(sys.argv) > 2 else None
T = float(sys.argv[3]) if len(sys.argv) > 3 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
res = {}
for r in data:
    d = dict(zip(hdr, r))
    name = d["Kernel Name"]
    f = lambda k: float(d[k].replace(",", "")) if d.get(k, "") not in ("", "n/a") else float("nan")
    dur_ns = f("gpu__time_duration.sum")
    rd, wr = f("dram__bytes_read.sum"), f("dram__bytes_write.sum")
    u = dict(zip(hdr, units))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    rd *= scale.get(u.get("dram__bytes_read.sum", "byte"), 1)
    wr *= scale.get(u.get("dram__bytes_write.sum", "byte"), 1)
    dscale = {"nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}
    dur_ns *= dscale.get(u.get("gpu__time_duration.sum", "nsecond"), 1)
    stalls = {}
    for h, v in d.items():
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                stalls[h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(v)
            except ValueError:
                pass
    top = sorted(stalls.items(), key=lambda kv: -kv[1])[:6]
    s = {
        "kernel": name, "duration_us": dur_ns / 1e3, "dram_read_bytes": rd, "dram_write_bytes": wr,
        "dram_bytes_per_launch": rd + wr, "dram_gbs": (rd + wr) / dur_ns,
        "issue_active_pct": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "ipc": f("sm__inst_executed.avg.per_cycle_active"),
        "warp_instructions": f("smsp__inst_executed.sum"),
        "sm_ghz": f("sm__cycles_elapsed.avg.per_second"),
        "top_stalls_per_issue": top,
        "pipe_active_pct": {h.split("__")[1].split(".")[0]: f(h) for h in hdr
                            if ("pipe_tensor" in h or "pipe_fma_cycles" in h or "pipe_alu_cycles" in h
                                or "pipe_fmaheavy_cycles" in h or "pipe_xu" in h)
                            and h.endswith("pct_of_peak_sustained_active")},
    }
    if T:
        s["dram_bytes_per_step"] = (rd + wr) / T
        s["warp_instructions_per_step"] = s["warp_instructions"] / T
    if "hmm_stream_kernel" in name:
        key = "smooth" if ", 0>" in name else ("viterbi" if ", 1>" in name else name)
    else:
        key = name
    res[key] = s
    print(json.dumps(s, indent=1))
if out:
    with open(out, "w") as fh:
        json.dump(res, fh, indent=1)
