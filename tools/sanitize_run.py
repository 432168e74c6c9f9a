"""Small invocations of every kernel family for compute-sanitizer runs:
C1 (pair kernels + int32 kernels), flow, refinement, general model, iterative
minorant, ROWCOL world 1 (NCCL not required: external transport)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import datagen  # noqa: E402
import paper_1601_06274_b200 as dmm  # noqa: E402

W, H, K = 64, 48, 16
l, r, _ = datagen.pair("rd", W, H, K, seed=0)
lt, rt = torch.from_numpy(l).cuda(), torch.from_numpy(r).cuda()
for pair in (True, False):
    c = dmm.Context(width=W, height=H, d_min=0, d_max=K - 1, max_iters=5)
    c.set_pair(pair)
    c.cost_volume(lt, rt)
    c.solve(5)
    print("C1", c.kernel_family(), c.result()[:2])
c = dmm.Context(width=96, height=40, d_min=0, d_max=127, max_iters=3)
l2, r2, _ = datagen.pair("wt-kitti", 96, 40, 128, seed=1)
c.cost_volume(torch.from_numpy(l2).cuda(), torch.from_numpy(r2).cuda())
c.solve(3)
print("K128", c.result()[:2])
print("refine", c.refine(warps=2, iters=5)[1])
i1, i2, _, _ = datagen.flow_pair(80, 40, 16, seed=0)
f = dmm.Context(width=80, height=40, d_min=-16, d_max=15, batch=2, max_iters=2)
f.flow_cost_volume(torch.from_numpy(i1).cuda(), torch.from_numpy(i2).cuda(), -16)
f.solve(2, nframes=2)
print("flow", f.result(0)[:2], f.result(1)[:2])
g = dmm.Context(width=W, height=H, d_min=0, d_max=K - 1, max_iters=2, pen=(8, 16, 2, 80), edge_weights=True)
g.cost_volume(lt, rt)
g.solve(2)
print("general", g.result()[:2])
it = dmm.Context(width=W, height=H, d_min=0, d_max=K - 1, max_iters=2, minorant="iterative")
it.cost_volume(lt, rt)
it.solve(2)
print("iterative", it.result()[:2])
torch.cuda.synchronize()
