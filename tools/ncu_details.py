"""Selected details-page metrics of an .ncu-rep: python tools/ncu_details.py rep [regex]"""
import csv, io, re, subprocess, sys
rep = sys.argv[1]
pat = re.compile(sys.argv[2] if len(sys.argv) > 2 else
                 r"Duration|DRAM Throughput|Memory Throughput|Achieved Occupancy|Theoretical Occupancy|"
                 r"Registers Per Thread|Block Limit|Waves Per SM|Compute \(SM\) Throughput|L2 Hit Rate|"
                 r"Executed Ipc Active|Grid Size|Shared Memory Configuration Size|Dynamic Shared|Static Shared")
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
ki, sn, mn, mu, mv = (h.index(x) for x in ("Kernel Name", "Section Name", "Metric Name", "Metric Unit", "Metric Value"))
seen = set()
for r in rows[1:]:
    if len(r) <= mv or not pat.search(r[mn]):
        continue
    key = (r[ki][:30], r[mn])
    if key in seen:
        continue
    seen.add(key)
    print(f"{r[ki][:28]:28s} {r[mn]:45s} {r[mv]:>14s} {r[mu]}")
