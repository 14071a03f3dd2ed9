import faulthandler, sys
faulthandler.enable(all_threads=True)
sys.path.insert(0, '.')
import numpy as np, torch
print('threads', __import__('os').cpu_count(), flush=True)
from paper_2605_04509_b200 import CoherentRaster, synthetic as sy
c = sy.CONFIGS['A']
scene, cams = c.make_scene(), c.make_rig()
g = CoherentRaster(0); print('ctx', flush=True)
g.upload_gaussians(scene); print('upload', flush=True)
g.set_display(c.W, c.H, c.N, c.lens_pitch, c.slant, c.center_offset); print('display', flush=True)
g.set_camera_rig(cams); print('rig', flush=True)
img = g.render(8, output_format='float', stats=True); torch.cuda.synchronize(); print('render', g.last_stats, flush=True)
img = img.cpu().numpy(); print(img.mean(), flush=True)
k, p = g.sorted_pairs(); print('pairs', k.shape, flush=True)
import oracle
o = oracle.Oracle(); print('oracle threads', o.threads, flush=True)
o.set_scene(scene); o.set_display(c.W, c.H, c.N, c.lens_pitch, slant=c.slant, center_offset=c.center_offset); o.set_rig(cams)
o.render(s=8); print('oracle render', o.num_pairs, flush=True)
ko, po = o.pairs(); print('eq keys', np.array_equal(k, ko), np.array_equal(p, po), flush=True)
print('maxdiff', np.abs(img - o.image()).max(), flush=True)
g.close(); print('closed', flush=True)
