"""Thread-instructions per time step, per CUDA source line (ncu source page)."""
import subprocess, csv, io, collections, sys
rep, ksub, T = sys.argv[1], sys.argv[2], float(sys.argv[3]) if len(sys.argv) > 3 else 1e6
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"], capture_output=True, text=True).stdout
func = hdr = fname = None; agg = collections.Counter(); src = {}
for row in csv.reader(io.StringIO(out)):
    if not row: continue
    if row[0] == "File Path": fname = row[1].split('/')[-1]; continue
    if row[0] == "Function Name": func = row[1]; continue
    if row[0] == "Line No": hdr = row; continue
    if not hdr or ksub not in (func or "") or not row[0].strip() or len(row) < len(hdr): continue
    v = row[hdr.index("Thread Instructions Executed")]
    if not v.isdigit(): continue
    k = (fname, int(row[0])); agg[k] += int(v); src[k] = row[1][:90]
tot = sum(agg.values()); print(f"thread-instr per step {tot/T:.1f}")
for k, v in agg.most_common(top): print(f"{v/T:7.1f}/step {k[0]}:{k[1]:<5} {src[k]}")
