"""Multi-GPU sharding of the Dual MM hot path.

Two modes, one process per GPU:

* frames  -- independent frames are assigned round-robin to ranks; no data-path
  collective (``frames_for_rank``; used by bench.py, weak scaling).
* bands   -- one large frame: rank r owns the row band ``bands(H)[r]`` for the H
  half-steps and the column band ``bands(W)[r]`` for the V half-steps.  Chains of
  one orientation are independent ("decoupled for all horizontal (resp.
  vertical) chains"), so each half-step is local; between half-steps the
  minorant records are transposed with one all-to-all:
  after H, the f_ records (the V pass's unaries) go row band -> column band;
  after V, the D*2^F + g_ records (the H pass's unaries) go back.
  The bounds are sums over chains, hence an all-reduce of per-rank partial
  sums; the labels are all-gathered.  The result is bit-identical to the
  unsharded solve (integer arithmetic; the exchange is a permutation).

The exchange is written against a tiny ``Exchanger`` interface so the same
driver runs over ``torch.distributed`` (NCCL on B200s, gloo on CPU for tests)
or in-process (``lockstep_band_dmm``: all ranks' states held by one process and
advanced in lockstep -- pure data movement between the ranks' buffers, no
kernels waiting on each other -- for single-GPU / CPU checks of the band logic).
"""
from __future__ import annotations

from typing import List, Sequence, Tuple


def bands(n: int, world: int) -> List[Tuple[int, int]]:
    """Contiguous [start, stop) bands of n items over world ranks (sizes differ by <= 1)."""
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


# --------------------------------------------------------------- exchangers
class DistExchanger:
    """all-to-all over torch.distributed (one rank per process)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def exchange(self, sends: Sequence, recv_shapes: Sequence[Tuple[int, ...]]):
        """sends[s] goes to rank s; returns recvs[s] (shape recv_shapes[s])
        received from rank s -- one all_to_all_single of the flattened blocks."""
        import torch
        flat_in = torch.cat([s.reshape(-1) for s in sends]) if sends else None
        in_splits = [s.numel() for s in sends]
        out_splits = [int(torch.tensor(sh).prod().item()) if len(sh) else 1 for sh in recv_shapes]
        flat_out = torch.empty(sum(out_splits), dtype=sends[0].dtype, device=sends[0].device)
        self.dist.all_to_all_single(flat_out, flat_in, output_split_sizes=out_splits,
                                    input_split_sizes=in_splits, group=self.group)
        outs, o = [], 0
        for sh, n in zip(recv_shapes, out_splits):
            outs.append(flat_out[o:o + n].view(*sh))
            o += n
        return outs

    def all_reduce_sum(self, t):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return t

    def all_gather(self, t):
        import torch
        outs = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(outs, t.contiguous(), group=self.group)
        return outs


# ------------------------------------------------------------- transposes
def rows_to_cols_sends(rowband, col_bands):
    """rowband (Hb, W, E) -> per destination s the block (Hb, cols_s, E)."""
    return [rowband[:, c0:c1, :].contiguous() for (c0, c1) in col_bands]


def cols_to_rows_sends(colband, row_bands):
    """colband (H, Wb, E) -> per destination s the block (rows_s, Wb, E)."""
    return [colband[r0:r1, :, :].contiguous() for (r0, r1) in row_bands]


def transpose_rows_to_cols(exch, rowband, row_bands, col_bands, rank):
    """All-to-all: my row band of every column -> my column band of every row."""
    import torch
    Wb = col_bands[rank][1] - col_bands[rank][0]
    E = rowband.shape[2]
    recv_shapes = [((r1 - r0), Wb, E) for (r0, r1) in row_bands]
    recvs = exch.exchange(rows_to_cols_sends(rowband, col_bands), recv_shapes)
    return torch.cat(recvs, dim=0)


def transpose_cols_to_rows(exch, colband, row_bands, col_bands, rank):
    """All-to-all back: my column band of every row -> my row band of every column."""
    import torch
    Hb = row_bands[rank][1] - row_bands[rank][0]
    E = colband.shape[2]
    recv_shapes = [(Hb, (c1 - c0), E) for (c0, c1) in col_bands]
    recvs = exch.exchange(cols_to_rows_sends(colband, row_bands), recv_shapes)
    return torch.cat(recvs, dim=1)


# ---------------------------------------------------------------- driver
def band_dmm(engine, exch, iterations: int):
    """Algorithm 2 on a band-sharded frame.

    ``engine`` provides, for this rank:
      half_h(t, iterations)          H half-step on the row band
      half_v(t, iterations)          V half-step on the column band
      fv_rows() / set_fv_cols(x)     f_ records: row-band view / column-band store
      fh_cols() / set_fh_rows(x)     D*2^F + g_ records: column-band view / row-band store
      row_bands, col_bands, rank
    """
    rb, cb, r = engine.row_bands, engine.col_bands, engine.rank
    for t in range(iterations):
        engine.half_h(t, iterations)
        engine.set_fv_cols(transpose_rows_to_cols(exch, engine.fv_rows(), rb, cb, r))
        engine.half_v(t, iterations)
        if t + 1 < iterations:
            engine.set_fh_rows(transpose_cols_to_rows(exch, engine.fh_cols(), rb, cb, r))


# ------------------------------------------------------- CUDA band engine
class CudaBandEngine:
    """Band engine on the CUDA path: three contexts per rank -- the full frame
    (census + cost volume need image halos and full-width right codes), the
    row band (H half-steps) and the column band (V half-steps).  Records move
    between them as uint8 tensors of REC bytes per pixel."""

    def __init__(self, W: int, H: int, world: int, rank: int, device=None, **cfg):
        import paper_1601_06274_b200 as dmm
        self.dmm = dmm
        self.W, self.H, self.world, self.rank = W, H, world, rank
        self.row_bands, self.col_bands = bands(H, world), bands(W, world)
        (self.r0, self.r1), (self.c0, self.c1) = self.row_bands[rank], self.col_bands[rank]
        max_iters = cfg.pop("max_iters", 16)
        self.full = dmm.Context(width=W, height=H, max_iters=max_iters, device=device, **cfg)
        self.rb = dmm.Context(width=W, height=self.r1 - self.r0, max_iters=max_iters, device=device, **cfg)
        self.cb = dmm.Context(width=self.c1 - self.c0, height=H, max_iters=max_iters, device=device, **cfg)
        self.frac_bits = self.full.frac_bits

    def cost_volume(self, left, right):
        self.full.cost_volume(left, right)
        D = self.full.cost_volume_tensor()
        self.rb.import_cost_volume(D[self.r0:self.r1].contiguous())
        self.cb.import_cost_volume(D[:, self.c0:self.c1].contiguous())

    def half_h(self, t, iterations):
        self.rb.half_step(t, 0, iterations)

    def half_v(self, t, iterations):
        self.cb.half_step(t, 1, iterations)

    def fv_rows(self):
        return self.rb.buffer(self.dmm.BUF_FV)

    def set_fv_cols(self, x):
        self.cb.buffer(self.dmm.BUF_FV).copy_(x)

    def fh_cols(self):
        return self.cb.buffer(self.dmm.BUF_FH)

    def set_fh_rows(self, x):
        self.rb.buffer(self.dmm.BUF_FH).copy_(x)

    def partial_bounds(self, iterations):
        """This rank's per-half-step partial bounds (H slots from the row band,
        V slots from the column band), int64 CUDA tensor [2*iterations]."""
        import torch
        hb = self.rb.bound_slots()[: 2 * iterations]
        vb = self.cb.bound_slots()[: 2 * iterations]
        idx = torch.arange(2 * iterations, device=hb.device)
        return torch.where(idx % 2 == 0, hb, vb).clone()

    def labels_cols(self):
        return self.cb.buffer(self.dmm.BUF_LABELS)[:, :, 0]


def solve_bands(engine: CudaBandEngine, exch, left, right, iterations: int):
    """Band-sharded solve of one frame; returns (labels (H, W) CUDA uint8 on
    every rank, bound history list of ints, energy int) -- all scaled by 2^F
    like Context.result()."""
    import torch
    engine.cost_volume(left, right)
    band_dmm(engine, exch, iterations)
    hist = exch.all_reduce_sum(engine.partial_bounds(iterations))
    labels = torch.cat(_gather_label_cols(exch, engine), dim=1)
    engine.full.buffer(engine.dmm.BUF_LABELS)[:, :, 0].copy_(labels)
    energy = engine.full.energy()
    return labels, [int(v) for v in hist.tolist()], energy


def _gather_label_cols(exch, engine):
    """All-gather of the column-band labels (bands may differ in width by one:
    pad to the widest band for the collective)."""
    import torch
    lab = engine.labels_cols()
    wmax = max(c1 - c0 for c0, c1 in engine.col_bands)
    pad = torch.zeros((engine.H, wmax), dtype=lab.dtype, device=lab.device)
    pad[:, : lab.shape[1]] = lab
    outs = exch.all_gather(pad)
    return [o[:, : (c1 - c0)] for o, (c0, c1) in zip(outs, engine.col_bands)]


def lockstep_band_dmm(engines: Sequence, iterations: int):
    """Run band_dmm for all ranks of one process in lockstep (single-GPU or
    CPU emulation of the band decomposition; each half-step is launched rank
    after rank, the transposes are pure data movement between the ranks'
    buffers)."""
    import torch
    rb, cb = engines[0].row_bands, engines[0].col_bands
    world = len(engines)
    for t in range(iterations):
        for e in engines:
            e.half_h(t, iterations)
        sends = [rows_to_cols_sends(e.fv_rows(), cb) for e in engines]
        for r, e in enumerate(engines):
            e.set_fv_cols(torch.cat([sends[s][r] for s in range(world)], dim=0))
        for e in engines:
            e.half_v(t, iterations)
        if t + 1 < iterations:
            sends = [cols_to_rows_sends(e.fh_cols(), rb) for e in engines]
            for r, e in enumerate(engines):
                e.set_fh_rows(torch.cat([sends[s][r] for s in range(world)], dim=1))


def solve_bands_lockstep(engines: Sequence[CudaBandEngine], left, right, iterations: int):
    """lockstep_band_dmm + the same reductions as solve_bands, in one process."""
    import torch
    for e in engines:
        e.cost_volume(left, right)
    lockstep_band_dmm(engines, iterations)
    hist = sum(e.partial_bounds(iterations) for e in engines)
    labels = torch.cat([e.labels_cols() for e in engines], dim=1)
    e0 = engines[0]
    e0.full.buffer(e0.dmm.BUF_LABELS)[:, :, 0].copy_(labels)
    return labels, [int(v) for v in hist.tolist()], e0.full.energy()
