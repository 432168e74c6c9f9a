"""Multi-GPU sharding of the Dual MM hot path.

Two modes, one process per GPU:

* frames  -- independent frames are assigned round-robin to ranks; no data-path
  collective (``frames_for_rank``; bench.py's default, weak scaling).
* bands   -- one large frame (configs[2]): rank r owns the row band
  ``bands(H)[r]`` for the H half-steps and the column band ``bands(W)[r]`` for
  the V half-steps.  Everything of the data plane is behind the C ABI
  (``dmm_shard``, include/dmm.h): the library owns the NCCL communicator, the
  all-to-all transposes of the dual records between half-steps (grouped
  ncclSend / ncclRecv straight out of / into the kernels' record arrays), the
  int64 all-reduce of the bound history and energy, and the labelling
  all-gather.  Python only creates the communicator id on rank 0 and
  broadcasts its 128 bytes (``rowcol_setup``).

Chains of one orientation are independent ("decoupled for all
horizontal (resp. vertical) chains"), which is why the only exchange is the
transpose; the sharded result is bit-identical to the unsharded solve.
"""
from __future__ import annotations

from typing import List, Tuple


def bands(n: int, world: int) -> List[Tuple[int, int]]:
    """Contiguous [start, stop) bands of n items over world ranks (sizes differ
    by <= 1, the first n % world bands one longer) -- the split the C ABI uses."""
    if world < 1:
        raise ValueError("world must be >= 1")
    q, r = divmod(n, world)
    out, s = [], 0
    for k in range(world):
        e = s + q + (1 if k < r else 0)
        out.append((s, e))
        s = e
    return out


def frames_for_rank(n_frames: int, world: int, rank: int) -> List[int]:
    """Round-robin frame assignment (frames mode)."""
    return list(range(rank, n_frames, world))


def broadcast_nccl_id(group=None) -> bytes:
    """Rank 0 creates an NCCL id (dmm_nccl_unique_id); every rank returns it."""
    import torch
    import torch.distributed as dist

    import paper_1601_06274_b200 as dmm
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else "cpu"
    buf = torch.zeros(128, dtype=torch.uint8, device=dev)
    if dist.get_rank(group) == 0:
        buf.copy_(torch.frombuffer(bytearray(dmm.nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(buf, src=0, group=group)
    return bytes(buf.cpu().numpy().tobytes())


def rowcol_setup(ctx, group=None):
    """Shard `ctx` (created with the whole frame's config) in row / column
    bands over the ranks of `group`, with the library's own NCCL communicator."""
    import torch.distributed as dist

    import paper_1601_06274_b200 as dmm
    nid = broadcast_nccl_id(group)
    ctx.shard(nid, dist.get_rank(group), dist.get_world_size(group), dmm.SHARD_ROWCOL)
    return ctx
