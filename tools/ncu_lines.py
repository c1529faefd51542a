"""Aggregate ncu source-page metrics (stall samples, instructions) per CUDA source line.

usage: python tools/ncu_lines.py report.ncu-rep [kernel-substring] [topN]
"""
import csv, io, subprocess, sys, collections

rep = sys.argv[1]; ksub = sys.argv[2] if len(sys.argv) > 2 else ""; top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
fname = func = None; hdr = None
agg = collections.defaultdict(lambda: [0, 0, 0, ""])
stalls = collections.defaultdict(collections.Counter)
tot = [0, 0]
for row in csv.reader(io.StringIO(out)):
    if not row: continue
    if row[0] == "File Path": fname = row[1].split("/")[-1]; continue
    if row[0] == "Function Name": func = row[1]; continue
    if row[0] == "Line No": hdr = row; continue
    if hdr is None or ksub not in (func or ""): continue
    if len(row) < len(hdr) or not row[0].strip(): continue
    d = dict(zip(hdr[:2], row[:2])); m = dict(zip(hdr[2:], row[2:]))
    try:
        s = int(m.get("Warp Stall Sampling (All Samples)", "0") or 0)
        ins = int(m.get("Instructions Executed", "0") or 0)
    except ValueError:
        continue
    key = (fname, int(d["Line No"]))
    a = agg[key]; a[0] += s; a[1] += ins; a[3] = d["Source"][:90]
    tot[0] += s; tot[1] += ins
    for k, v in m.items():
        if k.startswith("stall_") and "Not Issued" not in k and v not in ("", "0"):
            try: stalls[key][k[6:]] += int(v)
            except ValueError: pass
print(f"total samples {tot[0]}  warp-instructions {tot[1]}")
for key, (s, ins, _, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    st = ", ".join(f"{k}:{v}" for k, v in stalls[key].most_common(3))
    print(f"{s/tot[0]*100:5.1f}% smp {ins/tot[1]*100:5.1f}% ins  {key[0]}:{key[1]:<5} {src:<70} [{st}]")
