"""One warm-up + one profiled solve of a BASELINE config, for ncu captures:

  ncu --set full -k regex:hm2_leaf -s <skip> -c 1 python tools/one_solve.py C2
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import datagen  # noqa: E402
import paper_1601_06274_b200 as dmm  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
c = datagen.CONFIGS[cfg]
W, H, K, iters = c["W"], c["H"], c["K"], c["iters"]
nf = c.get("frames", 1)
pairs = [datagen.pair(c["kind"], W, H, K, seed=s) for s in range(min(nf, 8))]
lt = torch.stack([torch.from_numpy(pairs[s % len(pairs)][0]) for s in range(nf)]).cuda()
rt = torch.stack([torch.from_numpy(pairs[s % len(pairs)][1]) for s in range(nf)]).cuda()
ctx = dmm.Context(width=W, height=H, d_min=0, d_max=K - 1, w=3, T=4, frac_bits=4, max_iters=iters, batch=nf)
for _ in range(reps):
    ctx.cost_volume_frames(lt, rt)
    ctx.solve(iters, nframes=nf)
torch.cuda.synchronize()
print(cfg, ctx.result())
