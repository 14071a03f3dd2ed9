"""Summarise tools/prof_ablation.sh outputs into a markdown table."""
import csv, sys, glob, io
rows_out = []
for f in sorted(glob.glob(sys.argv[1])):
    txt = open(f).read()
    i = txt.index('"ID"')
    rows = list(csv.reader(io.StringIO(txt[i:])))
    h = rows[0]
    mi, vi, ui = h.index('Metric Name'), h.index('Metric Value'), h.index('Metric Unit')
    m = {r[mi]: (float(r[vi].replace(',', '')), r[ui]) for r in rows[1:] if len(r) > vi}
    rows_out.append((f, m))
def g(m, k):
    return m.get(k, (float('nan'), ''))[0]
print("| variant | time | DRAM bytes | L2 bytes | warp exec eff. (thr/inst) | global ld sectors/request | IPC | warp instructions |")
print("|---|---|---|---|---|---|---|---|")
names = {'k0_r1': 'staged (B200), remap', 'k1_r1': 'paper thread/subpixel, remap', 'k1_r0': 'paper thread/subpixel, raster order (w/o remap)'}
for f, m in rows_out:
    key = f.split('_')[-2] + '_' + f.split('_')[-1].replace('.csv', '')
    t = m['gpu__time_duration.sum']
    sec = g(m, 'l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum') / max(1.0, g(m, 'l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum'))
    print(f"| {names.get(key, key)} | {t[0]:.2f} {t[1]} | {g(m,'dram__bytes_read.sum')+g(m,'dram__bytes_write.sum'):.3g} | {g(m,'lts__t_bytes.sum'):.3g} | {g(m,'smsp__thread_inst_executed_per_inst_executed.ratio'):.1f} | {sec:.2f} | {g(m,'sm__inst_executed.avg.per_cycle_active'):.2f} | {g(m,'smsp__inst_executed.sum'):.3g} |")
