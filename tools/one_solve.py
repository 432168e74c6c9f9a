"""One warm-up + one profiled solve of a BASELINE config, for ncu captures:

  ncu --set full -k regex:hm2_leaf -s <skip> -c 1 python tools/one_solve.py C2
  python tools/one_solve.py C2 2 refine      # + the continuous refinement after each solve
  python tools/one_solve.py C2 1 general     # NEXT-3 penalty 8,16,2,80 + edge weights (or: iterative)
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
mode = sys.argv[3] if len(sys.argv) > 3 else ""
refine = mode == "refine"
extra = {"general": dict(pen=(8, 16, 2, 80), edge_weights=True), "iterative": dict(minorant="iterative")}.get(mode, {})
c = datagen.CONFIGS[cfg]
W, H, K, iters = c["W"], c["H"], c["K"], c["iters"]
if c["kind"] == "flow":                       # configs[3]: two K-label layers of one context
    i1, i2, _, _ = datagen.flow_pair(W, H, -c["d_min"], seed=0)
    ctx = dmm.Context(width=W, height=H, d_min=c["d_min"], d_max=c["d_min"] + K - 1, w=3, T=4, frac_bits=4,
                      max_iters=iters, batch=2)
    t1, t2 = torch.from_numpy(i1).cuda(), torch.from_numpy(i2).cuda()
    for _ in range(reps):
        ctx.flow_cost_volume(t1, t2, c["d_min"])
        ctx.solve(iters, nframes=2)
        if refine:
            ctx.flow_refine(c["d_min"], C=4.0)
    torch.cuda.synchronize()
    print(cfg, ctx.result(0), ctx.result(1))
    sys.exit(0)
nf = c.get("frames", 1)
pairs = [datagen.pair(c["kind"], W, H, K, seed=s) for s in range(min(nf, 8))]
lt = torch.stack([torch.from_numpy(pairs[s % len(pairs)][0]) for s in range(nf)]).cuda()
rt = torch.stack([torch.from_numpy(pairs[s % len(pairs)][1]) for s in range(nf)]).cuda()
ctx = dmm.Context(width=W, height=H, d_min=0, d_max=K - 1, w=3, T=4, frac_bits=4, max_iters=iters, batch=nf, **extra)
for _ in range(reps):
    ctx.cost_volume_frames(lt, rt)
    ctx.solve(iters, nframes=nf)
    if refine:
        for f in range(nf):
            ctx.refine(frame=f)
torch.cuda.synchronize()
print(cfg, ctx.result())
