"""Per-CUDA-source-line instruction / stall shares of one kernel in an .ncu-rep:
python tools/ncu_lines.py rep [kernel-regex] [top]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else "."
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", "regex:" + kre], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, data, hdr = "?", [], None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or r[0] == "":
        continue
    ie = hdr.index("Instructions Executed")
    ws = hdr.index("Warp Stall Sampling (All Samples)")
    try:
        data.append((int(r[ie] or 0), int(r[ws] or 0), f"{fname}:{r[0]}", r[1][:90]))
    except ValueError:
        pass
tot = sum(d[0] for d in data) or 1
tw = sum(d[1] for d in data) or 1
print(f"total warp instructions {tot:.3e}")
for d in sorted(data, reverse=True)[:top]:
    print(f"{100 * d[0] / tot:5.1f}%  stall {100 * d[1] / tw:5.1f}%  {d[2]:>20s}  {d[3]}")
