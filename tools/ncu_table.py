"""Per-kernel table from a full ncu capture: duration, DRAM bytes, achieved GB/s, IPC, occupancy."""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]
out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
def col(name):
    return h.index(name) if name in h else None
ki = col('Kernel Name'); du = col('gpu__time_duration.sum'); dr = col('dram__bytes_read.sum'); dw = col('dram__bytes_write.sum')
ipc = col('sm__inst_executed.avg.per_cycle_active'); occ = col('sm__warps_active.avg.pct_of_peak_sustained_active')
units = rows[1]
def val(r, i, unit_row=units):
    if i is None: return float('nan')
    v = float(r[i].replace(',', ''))
    u = unit_row[i]
    scale = {'ns': 1e-9, 'us': 1e-6, 'usecond': 1e-6, 'ms': 1e-3, 'msecond': 1e-3, 'nsecond': 1e-9, 's': 1,
             'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'KB': 1e3, 'MB': 1e6, 'GB': 1e9}.get(u, 1)
    return v * scale
agg = collections.OrderedDict()
for r in rows[2:]:
    n = r[ki].split('(')[0].replace('void ', '').replace('cr::', '')
    n = n.split('<')[0] + ('<' + r[ki].split('<')[1].split('>')[0].replace(' ', '') + '>' if '<' in r[ki].split('(')[0] else '')
    a = agg.setdefault(n, [0, 0.0, 0.0, 0.0, 0.0, 0.0])
    a[0] += 1; a[1] += val(r, du); a[2] += val(r, dr) + val(r, dw); a[3] += val(r, ipc); a[4] += val(r, occ)
lt = col('lts__t_bytes.sum')
print(f"{'kernel':40s} {'n':>3s} {'time ms':>9s} {'DRAM GB':>8s} {'GB/s':>8s} {'IPC':>5s} {'occ%':>5s}")
for n, (c, t, b, i, o, _) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n[:40]:40s} {c:3d} {t*1e3:9.3f} {b/1e9:8.3f} {b/t/1e9 if t else 0:8.0f} {i/c:5.2f} {o/c:5.1f}")
