"""Experiment: two contexts on two streams driven by two host threads (same
scene/rig, so the shared __constant__ rig is identical) -> frame throughput."""
import sys, os, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_04509_b200 import CoherentRaster, synthetic as sy
c = sy.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C"]
scene, cams = c.make_scene(), c.make_rig()
nctx = int(sys.argv[2]) if len(sys.argv) > 2 else 2
ctxs = []
for q in range(nctx):
    st = torch.cuda.Stream()
    r = CoherentRaster(0, stream=st)
    r.upload_gaussians(scene)
    r.set_display(c.W, c.H, c.N, c.lens_pitch, c.slant, c.center_offset, c.view_cone)
    r.set_camera_rig(cams)
    out = torch.empty(r.band_shape(), dtype=torch.uint8, device="cuda")
    ctxs.append((r, st, out))
def work(q, n):
    r, st, out = ctxs[q]
    with torch.cuda.stream(st):
        for _ in range(n):
            r.render(8, out=out)
        st.synchronize()
for q in range(nctx):
    work(q, 3)
torch.cuda.synchronize()
F = 30
t0 = time.perf_counter()
th = [threading.Thread(target=work, args=(q, F)) for q in range(nctx)]
for t in th: t.start()
for t in th: t.join()
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"{nctx} contexts: {nctx * F} frames in {dt:.3f} s -> {nctx * F / dt:.1f} frames/s")
