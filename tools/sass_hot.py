"""Hot SASS blocks of one kernel in an .ncu-rep: python tools/sass_hot.py rep.ncu-rep [regex] [threshold]"""
import csv, subprocess, sys, io, collections
rep = sys.argv[1]; kre = sys.argv[2] if len(sys.argv) > 2 else '.'; thr = float(sys.argv[3]) if len(sys.argv) > 3 else 0.02
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass', '-k', 'regex:' + kre], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
si = h.index('Source'); ie = h.index('Instructions Executed'); ws = h.index('Warp Stall Sampling (All Samples)'); at = h.index('Avg. Threads Executed'); ai = h.index('Address')
data = []
for r in rows[2:]:
    try: data.append((r[ai], r[si], int(r[ie] or 0), int(r[ws] or 0), float(r[at] or 0)))
    except Exception: pass
tot = sum(d[2] for d in data); totw = sum(d[3] for d in data) or 1
print('total warp instr %.3e  stall samples %d' % (tot, totw))
op = collections.Counter()
for a, s, i, w, t in data:
    o = s.split()[0] if s else ''
    if o.startswith('@'): o = s.split()[1]
    op[o.split('.')[0]] += i
print(' '.join(f"{o}:{100*c/tot:.1f}%" for o, c in op.most_common(14)))
prev = None; blocks = []
for a, s, i, w, t in data:
    if i != prev:
        blocks.append([a, 0, i, s, 0, t]); prev = i
    blocks[-1][1] += 1; blocks[-1][4] += w
for b in blocks:
    if b[2] * b[1] > thr * tot or b[4] > thr * totw:
        print(b[0][-5:], 'n=%3d' % b[1], 'exec=%10d' % b[2], 'inst%%=%4.1f' % (100 * b[1] * b[2] / tot), 'stall%%=%4.1f' % (100 * b[4] / totw), 'thr=%4.1f' % b[5], b[3][:50])
