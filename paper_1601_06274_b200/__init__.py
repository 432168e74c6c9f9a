"""B200-native (sm_100a) hot path of arXiv 1601.06274: census cost volume + Dual MM
with hierarchical minorants.

This module is the thin Python face of the C ABI in ``include/dmm.h``
(``_lib/libdmm_b200.so``): argument marshalling only.  Every step of the path
runs in the CUDA kernels of ``csrc/``; PyTorch provides device memory (the
workspace), streams and ``torch.distributed``.  There is no CPU fallback: if the
shared library or a CUDA device is missing, construction raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

__all__ = ["Context", "DmmError", "library_path", "load_library", "EXPORTS"]

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.environ.get("DMM_B200_LIB") or os.path.join(_HERE, "_lib", "libdmm_b200.so")
_lib = None

# every entry point declared in include/dmm.h
EXPORTS = (
    "dmm_workspace_bytes", "dmm_create", "dmm_destroy", "dmm_cost_volume", "dmm_solve",
    "dmm_result", "dmm_copy_labels", "dmm_copy_codes", "dmm_copy_cost_volume", "dmm_copy_dual",
    "dmm_run_host", "dmm_launch_count", "dmm_status_str", "dmm_last_error",
    "dmm_set_profiling", "dmm_read_profile", "dmm_set_tuning", "dmm_msg", "dmm_handshake",
    "dmm_buffer_ptr", "dmm_import_cost_volume", "dmm_half_step", "dmm_energy",
    "dmm_cost_volume_frames", "dmm_run_host_frames", "dmm_energy_of",
    "dmm_flow_cost_volume", "dmm_refine", "dmm_flow_refine", "dmm_nccl_unique_id", "dmm_shard", "dmm_shard_workspace_bytes", "dmm_shard_plan", "dmm_shard_locate",
)
SHARD_FRAMES, SHARD_ROWCOL = 0, 1
LOC_FV_H, LOC_FH_H, LOC_FV_V, LOC_FH_V, LOC_LABEL_V, LOC_BOUNDS = range(6)
BUF_D, BUF_FV, BUF_FH, BUF_LABELS, BUF_BOUNDS = 0, 1, 2, 3, 4
TUNE_STOP_AFTER_H = 2
TUNE_PAIR = 3
TUNE_QUERY_PAIR = 4
PROFILE_CLASSES = ("census", "cost_volume", "hm_h", "hm_v", "energy", "refine")


class DmmError(RuntimeError):
    pass


class DmmConfig(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in (
        "width", "height", "d_min", "d_max", "census_radius", "w_h", "w_v", "trunc",
        "frac_bits", "oob_cost", "batch", "max_iters", "pen_e1", "pen_e2", "pen_delta", "pen_c", "edge_weights",
        "minorant", "iter_passes", "iter_gshift")]


class DmmRefineParams(ctypes.Structure):
    _fields_ = [("eps", ctypes.c_double), ("delta", ctypes.c_double), ("C", ctypes.c_double),
                ("h", ctypes.c_double), ("tau", ctypes.c_double), ("sigma", ctypes.c_double),
                ("warps", ctypes.c_int32), ("iters", ctypes.c_int32)]


class DmmXfer(ctypes.Structure):
    _fields_ = [("peer", ctypes.c_int32), ("send_offset", ctypes.c_int64), ("send_bytes", ctypes.c_int64),
                ("recv_offset", ctypes.c_int64), ("recv_bytes", ctypes.c_int64)]


def make_config(width, height, d_min=0, d_max=127, w=3, T=4, frac_bits=4, census_radius=2, oob_cost=-1,
                batch=1, max_iters=16, w_h=None, w_v=None, pen=None, edge_weights=False, minorant="hierarchical",
                iter_passes=3, iter_gshift=2) -> DmmConfig:
    p = pen if pen is not None else (0, 0, 0, 0)
    mi = {"hierarchical": 0, "iterative": 1}[minorant]
    return DmmConfig(width, height, d_min, d_max, census_radius, w if w_h is None else w_h,
                     w if w_v is None else w_v, T, frac_bits, oob_cost, batch, max_iters, *p, int(bool(edge_weights)),
                     mi, iter_passes if mi else 0, iter_gshift if mi else 0)


def library_path() -> str:
    return _LIB_PATH


def load_library():
    """Load libdmm_b200.so (raises if it was not built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"{_LIB_PATH} missing: run __graft_entry__.build() "
                          "(python -m paper_1601_06274_b200._build)")
    lib = ctypes.CDLL(_LIB_PATH)
    P, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    C = ctypes.POINTER(DmmConfig)
    sig = {
        "dmm_workspace_bytes": (ctypes.c_size_t, [C]),
        "dmm_create": (ctypes.c_int, [C, P, ctypes.c_size_t, ctypes.c_int, ctypes.POINTER(P)]),
        "dmm_destroy": (None, [P]),
        "dmm_cost_volume": (ctypes.c_int, [P, ctypes.c_int, P, P, i64, P]),
        "dmm_solve": (ctypes.c_int, [P, ctypes.c_int, ctypes.c_int, i32, P]),
        "dmm_result": (ctypes.c_int, [P, ctypes.c_int, P, P, P, P]),
        "dmm_copy_labels": (ctypes.c_int, [P, ctypes.c_int, P, P]),
        "dmm_copy_codes": (ctypes.c_int, [P, ctypes.c_int, ctypes.c_int, P, P]),
        "dmm_copy_cost_volume": (ctypes.c_int, [P, ctypes.c_int, P, P]),
        "dmm_copy_dual": (ctypes.c_int, [P, ctypes.c_int, ctypes.c_int, P, P]),
        "dmm_run_host": (ctypes.c_int, [P, ctypes.c_int, P, P, i32, P, P, P, P]),
        "dmm_cost_volume_frames": (ctypes.c_int, [P, ctypes.c_int, ctypes.c_int, P, P, i64, P]),
        "dmm_run_host_frames": (ctypes.c_int, [P, ctypes.c_int, ctypes.c_int, P, P, i32, P, P, P, P]),
        "dmm_launch_count": (i64, [P]),
        "dmm_status_str": (ctypes.c_char_p, [ctypes.c_int]),
        "dmm_last_error": (ctypes.c_char_p, [P]),
        "dmm_set_profiling": (ctypes.c_int, [P, ctypes.c_int]),
        "dmm_read_profile": (ctypes.c_int, [P, P, P]),
        "dmm_set_tuning": (ctypes.c_int, [P, ctypes.c_int, i64]),
        "dmm_msg": (ctypes.c_int, [P, P, ctypes.c_int, ctypes.c_int, i32, i32, P]),
        "dmm_handshake": (ctypes.c_int, [P, P, P, P, P, P, ctypes.c_int, ctypes.c_int, i32, i32, P]),
        "dmm_buffer_ptr": (ctypes.c_int, [P, ctypes.c_int, ctypes.c_int, ctypes.POINTER(P),
                                          ctypes.POINTER(ctypes.c_size_t), ctypes.POINTER(ctypes.c_int)]),
        "dmm_import_cost_volume": (ctypes.c_int, [P, ctypes.c_int, P, P]),
        "dmm_half_step": (ctypes.c_int, [P, ctypes.c_int, ctypes.c_int, i32, ctypes.c_int, i32, P]),
        "dmm_energy": (ctypes.c_int, [P, ctypes.c_int, ctypes.POINTER(i64), P]),
        "dmm_energy_of": (ctypes.c_int, [P, ctypes.c_int, P, ctypes.POINTER(i64), P]),
        "dmm_flow_cost_volume": (ctypes.c_int, [P, ctypes.c_int, P, P, i64, i32, P]),
        "dmm_refine": (ctypes.c_int, [P, ctypes.c_int, ctypes.POINTER(DmmRefineParams), P,
                                      ctypes.POINTER(ctypes.c_double), P]),
        "dmm_flow_refine": (ctypes.c_int, [P, ctypes.c_int, i32, ctypes.POINTER(DmmRefineParams), P, P,
                                           ctypes.POINTER(ctypes.c_double), P]),
        "dmm_nccl_unique_id": (ctypes.c_int, [P]),
        "dmm_shard": (ctypes.c_int, [P, P, ctypes.c_int, ctypes.c_int, ctypes.c_int]),
        "dmm_shard_workspace_bytes": (ctypes.c_size_t, [C, ctypes.c_int, ctypes.c_int, ctypes.c_int]),
        "dmm_shard_plan": (ctypes.c_int, [C, ctypes.c_int, ctypes.c_int, ctypes.c_int, P, ctypes.c_int]),
        "dmm_shard_locate": (i64, [C, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def nccl_unique_id() -> bytes:
    """A fresh NCCL communicator id (dmm_nccl_unique_id), to broadcast to the other ranks."""
    buf = (ctypes.c_uint8 * 128)()
    _prim_check(load_library().dmm_nccl_unique_id(buf))
    return bytes(buf)


def shard_workspace_bytes(cfg: DmmConfig, rank: int, world: int, mode: int = SHARD_ROWCOL) -> int:
    return int(load_library().dmm_shard_workspace_bytes(ctypes.byref(cfg), rank, world, mode))


def shard_plan(cfg: DmmConfig, rank: int, world: int, phase: int):
    """dmm_shard_plan (host only): [(peer, send_off, send_bytes, recv_off, recv_bytes)] of one all-to-all."""
    out = (DmmXfer * world)()
    n = load_library().dmm_shard_plan(ctypes.byref(cfg), rank, world, phase, out, world)
    if n < 0:
        raise DmmError("dmm_shard_plan: invalid arguments")
    return [(x.peer, x.send_offset, x.send_bytes, x.recv_offset, x.recv_bytes) for x in out[:n]]


def shard_locate(cfg: DmmConfig, rank: int, world: int, which: int, y: int, x: int) -> int:
    """dmm_shard_locate (host only): byte offset of pixel (y, x)'s record / label, -1 if not owned."""
    return int(load_library().dmm_shard_locate(ctypes.byref(cfg), rank, world, which, y, x))


def torch_int64():
    import torch
    return torch.int64


def _stream_handle(stream, device=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return s.cuda_stream


def _prim_check(st):
    if st != 0:
        raise DmmError(load_library().dmm_status_str(st).decode())


def msg(a, ws: int, T: int, stream=None):
    """Device Msg (Eq. msg-pass) on int32 CUDA tensor a[count, K]."""
    import torch
    a = a.contiguous()
    out = torch.empty_like(a)
    count, K = a.shape
    _prim_check(load_library().dmm_msg(ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                       count, K, ws, T, _stream_handle(stream)))
    return out


def handshake(Fi, Fj, phiL, phiR, ws: int, T: int, stream=None):
    """Device Handshake (Alg.5) on int32 CUDA tensors [count, K];
    returns (phi_ij, phi_ji')."""
    import torch
    Fi, Fj, phiL, phiR = (t.contiguous() for t in (Fi, Fj, phiL, phiR))
    oij = torch.empty_like(Fi)
    oji = torch.empty_like(Fi)
    count, K = Fi.shape
    _prim_check(load_library().dmm_handshake(*(ctypes.c_void_p(t.data_ptr()) for t in (Fi, Fj, phiL, phiR, oij, oji)),
                                             count, K, ws, T, _stream_handle(stream)))
    return oij, oji


class Context:
    """One problem shape (W x H, disparities d_min..d_max) and `batch` frames.

    Energies / bounds are returned as exact ints in units of 2**-frac_bits
    (``value / 2**frac_bits`` is the real-valued energy of Eq.3)."""

    def __init__(self, width: int, height: int, d_min: int = 0, d_max: int = 127, w: int = 3,
                 T: int = 4, frac_bits: int = 4, census_radius: int = 2, oob_cost: int = -1,
                 batch: int = 1, max_iters: int = 16, w_h: int | None = None,
                 w_v: int | None = None, device=None, shard_world: int = 0, pen=None, edge_weights: bool = False,
                 minorant: str = "hierarchical", iter_passes: int = 3, iter_gshift: int = 2):
        import torch
        if not torch.cuda.is_available():
            raise DmmError("no CUDA device: the DMM hot path has no CPU fallback")
        self._lib = load_library()
        self.device = torch.device(device if device is not None else f"cuda:{torch.cuda.current_device()}")
        self.cfg = make_config(width, height, d_min, d_max, w, T, frac_bits, census_radius, oob_cost, batch,
                               max_iters, w_h, w_v, pen, edge_weights, minorant, iter_passes, iter_gshift)
        self.W, self.H, self.K = width, height, d_max - d_min + 1
        self.batch, self.frac_bits, self.max_iters = batch, frac_bits, max_iters
        nbytes = self._lib.dmm_workspace_bytes(ctypes.byref(self.cfg))
        if nbytes == 0:
            raise DmmError("invalid dmm_config")
        if shard_world >= 1:
            # room for a later ROWCOL shard() over shard_world ranks, any rank
            nbytes = max([nbytes] + [int(self._lib.dmm_shard_workspace_bytes(ctypes.byref(self.cfg), r,
                                                                             shard_world, SHARD_ROWCOL))
                                     for r in range(shard_world)])
        self.workspace = torch.empty(nbytes + 256, dtype=torch.uint8, device=self.device)
        base = self.workspace.data_ptr()
        aligned = (base + 255) & ~255
        self._base_off = aligned - base
        h = ctypes.c_void_p()
        self._check(self._lib.dmm_create(ctypes.byref(self.cfg), ctypes.c_void_p(aligned), nbytes,
                                         self.device.index, ctypes.byref(h)), None)
        self._h = h
        self._iters = [0] * batch

    # ---------------------------------------------------------------- plumbing
    def _check(self, st: int, h):
        if st != 0:
            msg = self._lib.dmm_status_str(st).decode()
            if h is not None:
                msg += ": " + self._lib.dmm_last_error(h).decode()
            raise DmmError(msg)

    def _call(self, name, *args):
        self._check(getattr(self._lib, name)(self._h, *args), self._h)

    def close(self):
        if getattr(self, "_h", None):
            self._lib.dmm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launch_count(self) -> int:
        return int(self._lib.dmm_launch_count(self._h))

    def set_profiling(self, enable: bool = True):
        """Record CUDA events around every kernel launch (on its stream)."""
        self._call("dmm_set_profiling", 1 if enable else 0)

    def set_stop_after_h(self, enable: bool = True):
        """Debug: the next solve stops after the first H half-step (f_ tap only)."""
        self._call("dmm_set_tuning", TUNE_STOP_AFTER_H, 1 if enable else 0)

    def set_pair(self, enable: bool = True):
        """Chain-pair packed 16-bit kernels (default on; used only when the
        configuration passes the 16-bit range check) or the int32 kernels."""
        self._call("dmm_set_tuning", TUNE_PAIR, 1 if enable else 0)

    def kernel_family(self) -> str:
        """'pair' or 'int32': the half-step kernels the next solve runs."""
        self._call("dmm_set_tuning", TUNE_QUERY_PAIR, 0)
        return self._lib.dmm_last_error(self._h).decode()

    def read_profile(self):
        """{class: (total_ms, launches)} since the last read (synchronises)."""
        n = len(PROFILE_CLASSES)
        ms = (ctypes.c_double * n)()
        cnt = (ctypes.c_int64 * n)()
        self._call("dmm_read_profile", ms, cnt)
        return {c: (float(ms[i]), int(cnt[i])) for i, c in enumerate(PROFILE_CLASSES)}

    # ------------------------------------------------------------------- path
    def cost_volume(self, left, right, frame: int = 0, stream=None):
        """left/right: torch.uint8 (H, W) (row pitch allowed) on this device."""
        for t in (left, right):
            if t.dtype.itemsize != 1 or t.device != self.device or t.dim() != 2 or t.stride(1) != 1:
                raise DmmError("images must be uint8 (H, W) row-major tensors on the context device")
            if tuple(t.shape) != (self.H, self.W):
                raise DmmError(f"image shape {tuple(t.shape)} != {(self.H, self.W)}")
        if left.stride(0) != right.stride(0):
            raise DmmError("left/right row pitch differ")
        self._call("dmm_cost_volume", frame, ctypes.c_void_p(left.data_ptr()),
                   ctypes.c_void_p(right.data_ptr()), left.stride(0), _stream_handle(stream, self.device))

    def refine(self, eps: float = 1.0, delta: float = 1.0, C: float | None = None, h: float = 1.0,
               tau: float = 0.35, sigma: float = 0.35, warps: int = 5, iters: int = 40, frame: int = 0,
               stream=None, energy: bool = True):
        """Continuous refinement (dmm_refine) of the frame's labelling; returns
        (u, energy): u = torch.float32 (H, W) refined disparities on the device,
        energy = E(u) (float, or None if energy=False).  C defaults to T."""
        import torch
        prm = DmmRefineParams(eps, delta, float(self.cfg.trunc if C is None else C), h, tau, sigma, warps, iters)
        out = torch.empty((self.H, self.W), dtype=torch.float32, device=self.device)
        e = ctypes.c_double()
        self._call("dmm_refine", frame, ctypes.byref(prm), ctypes.c_void_p(out.data_ptr()),
                   ctypes.byref(e) if energy else None, _stream_handle(stream, self.device))
        return out, (float(e.value) if energy else None)

    def flow_refine(self, v_min: int, eps: float = 1.0, delta: float = 1.0, C: float | None = None, h: float = 1.0,
                    tau: float = 0.35, sigma: float = 0.35, warps: int = 5, iters: int = 40, frame: int = 0,
                    stream=None, energy: bool = True):
        """Continuous refinement of the flow of layers (frame, frame + 1)
        (dmm_flow_refine): returns (u1, u2, energy), float32 (H, W) on the device."""
        import torch
        prm = DmmRefineParams(eps, delta, float(self.cfg.trunc if C is None else C), h, tau, sigma, warps, iters)
        u1 = torch.empty((self.H, self.W), dtype=torch.float32, device=self.device)
        u2 = torch.empty_like(u1)
        e = ctypes.c_double()
        self._call("dmm_flow_refine", frame, v_min, ctypes.byref(prm), ctypes.c_void_p(u1.data_ptr()),
                   ctypes.c_void_p(u2.data_ptr()), ctypes.byref(e) if energy else None,
                   _stream_handle(stream, self.device))
        return u1, u2, (float(e.value) if energy else None)

    def flow_cost_volume(self, left, right, v_min: int, frame: int = 0, stream=None):
        """Optical flow, discrete stage (dmm_flow_cost_volume): the decoupled
        costs f1 (horizontal u1 = d_min + label) into frame `frame` and f2
        (vertical u2 = v_min + label) into frame `frame + 1`; then
        solve(iterations, frame, nframes=2) solves both layers."""
        for t in (left, right):
            if t.dtype.itemsize != 1 or t.device != self.device or t.dim() != 2 or t.stride(1) != 1:
                raise DmmError("images must be uint8 (H, W) row-major tensors on the context device")
            if tuple(t.shape) != (self.H, self.W):
                raise DmmError(f"image shape {tuple(t.shape)} != {(self.H, self.W)}")
        if left.stride(0) != right.stride(0):
            raise DmmError("left/right row pitch differ")
        self._call("dmm_flow_cost_volume", frame, ctypes.c_void_p(left.data_ptr()), ctypes.c_void_p(right.data_ptr()),
                   left.stride(0), v_min, _stream_handle(stream, self.device))
        self._iters[frame] = self._iters[frame + 1] = 0

    def cost_volume_frames(self, left, right, frame: int = 0, stream=None):
        """left/right: torch.uint8 (nframes, H, W) contiguous stacks on this device:
        census + cost volume of frames [frame, frame + nframes) in one launch each."""
        for t in (left, right):
            if (t.dtype.itemsize != 1 or t.device != self.device or t.dim() != 3 or not t.is_contiguous()
                    or tuple(t.shape[1:]) != (self.H, self.W)):
                raise DmmError("images must be contiguous uint8 (nframes, H, W) tensors on the context device")
        if left.shape[0] != right.shape[0]:
            raise DmmError("left/right frame counts differ")
        self._call("dmm_cost_volume_frames", frame, int(left.shape[0]), ctypes.c_void_p(left.data_ptr()),
                   ctypes.c_void_p(right.data_ptr()), self.W, _stream_handle(stream, self.device))

    def solve(self, iterations: int = 4, frame: int = 0, nframes: int = 1, stream=None):
        self._call("dmm_solve", frame, nframes, iterations, _stream_handle(stream, self.device))
        for f in range(frame, frame + nframes):
            self._iters[f] = iterations

    def result(self, frame: int = 0, stream=None):
        """(energy, bound, bound_history) as exact ints scaled by 2**frac_bits."""
        it = self._iters[frame]
        e = ctypes.c_int64()
        b = ctypes.c_int64()
        hist = (ctypes.c_int64 * max(2 * it, 1))()
        self._call("dmm_result", frame, ctypes.byref(e), ctypes.byref(b), hist, _stream_handle(stream, self.device))
        return int(e.value), int(b.value), [int(v) for v in hist[: 2 * it]]

    def labels(self, frame: int = 0, stream=None):
        import torch
        out = torch.empty((self.H, self.W), dtype=torch.uint8, device=self.device)
        self._call("dmm_copy_labels", frame, ctypes.c_void_p(out.data_ptr()), _stream_handle(stream, self.device))
        return out

    def codes(self, which: int, frame: int = 0, stream=None):
        import torch
        out = torch.empty((self.H, self.W), dtype=torch.int32, device=self.device)
        self._call("dmm_copy_codes", frame, which, ctypes.c_void_p(out.data_ptr()), _stream_handle(stream, self.device))
        return out

    def cost_volume_tensor(self, frame: int = 0, stream=None):
        import torch
        out = torch.empty((self.H, self.W, self.K), dtype=torch.uint8, device=self.device)
        self._call("dmm_copy_cost_volume", frame, ctypes.c_void_p(out.data_ptr()), _stream_handle(stream, self.device))
        return out

    def dual(self, which: int, frame: int = 0, stream=None):
        """which 0: f_ after the last H half-step; 1: g_ after the last V half-step."""
        import torch
        out = torch.empty((self.H, self.W, self.K), dtype=torch.int32, device=self.device)
        self._call("dmm_copy_dual", frame, which, ctypes.c_void_p(out.data_ptr()), _stream_handle(stream, self.device))
        return out

    # --------------------------------------------------------- multi-GPU
    def shard(self, nccl_id: bytes | None, rank: int, world: int, mode: int = SHARD_ROWCOL):
        """dmm_shard: make this context rank `rank` of `world` (ROWCOL: one frame
        in row / column bands, the all-to-all transposes and reductions done
        by the library over NCCL).  nccl_id None: no communicator (the caller
        moves the bytes of shard_plan between dmm_half_step calls)."""
        idbuf = None if nccl_id is None else (ctypes.c_uint8 * 128).from_buffer_copy(nccl_id)
        self._call("dmm_shard", idbuf, rank, world, mode)
        self.rank, self.world, self.shard_mode = rank, world, mode

    def ws_view(self, offset: int, nbytes: int):
        """uint8 view of `nbytes` bytes at byte `offset` of the (aligned) workspace."""
        o = self._base_off + offset
        return self.workspace[o: o + nbytes]

    # ------------------------------------------------ sharding building blocks
    def buffer(self, which: int, frame: int = 0):
        """uint8 CUDA tensor view (H, W, bytes_per_pixel) of one of the frame's
        arrays inside the workspace (BUF_D, BUF_FV, BUF_FH, BUF_LABELS)."""
        ptr = ctypes.c_void_p()
        nbytes = ctypes.c_size_t()
        bpp = ctypes.c_int()
        self._call("dmm_buffer_ptr", frame, which, ctypes.byref(ptr), ctypes.byref(nbytes), ctypes.byref(bpp))
        off = ptr.value - self.workspace.data_ptr()
        flat = self.workspace[off: off + nbytes.value]
        if which == BUF_BOUNDS:
            return flat.view(torch_int64())
        return flat.view(self.H, self.W, max(bpp.value, 1))

    def import_cost_volume(self, D, frame: int = 0, stream=None):
        """Load a dense uint8 (H, W, K) CUDA tensor as the frame's cost volume."""
        D = D.contiguous()
        if tuple(D.shape) != (self.H, self.W, self.K):
            raise DmmError(f"cost volume shape {tuple(D.shape)} != {(self.H, self.W, self.K)}")
        self._call("dmm_import_cost_volume", frame, ctypes.c_void_p(D.data_ptr()), _stream_handle(stream, self.device))
        self._iters[frame] = 0

    def half_step(self, t: int, vertical: int, iterations: int, frame: int = 0, nframes: int = 1, stream=None):
        """One half-step of Algorithm 2 (H if vertical == 0, else V) of iteration t."""
        self._call("dmm_half_step", frame, nframes, t, vertical, iterations, _stream_handle(stream, self.device))
        if vertical and t == iterations - 1:
            for f in range(frame, frame + nframes):
                self._iters[f] = iterations

    def bound_slots(self, frame: int = 0):
        """int64 CUDA tensor view of the frame's bound history slots."""
        return self.buffer(BUF_BOUNDS, frame)

    def energy(self, frame: int = 0, stream=None, labels=None) -> int:
        """Primal energy (Eq.3, scaled by 2**frac_bits) of the frame's
        current labels, or of `labels` (uint8 (H, W) label indices on this
        device) against the frame's cost volume.  Synchronises."""
        e = ctypes.c_int64()
        if labels is None:
            self._call("dmm_energy", frame, ctypes.byref(e), _stream_handle(stream, self.device))
        else:
            if (labels.dtype.itemsize != 1 or labels.device != self.device or tuple(labels.shape) != (self.H, self.W)
                    or not labels.is_contiguous()):
                raise DmmError("labels must be a contiguous uint8 (H, W) tensor on the context device")
            self._call("dmm_energy_of", frame, ctypes.c_void_p(labels.data_ptr()), ctypes.byref(e),
                       _stream_handle(stream, self.device))
        return int(e.value)

    def run_host_frames(self, left, right, iterations: int = 4, labels_out=None, frame: int = 0, stream=None):
        """run_host for a stack of frames: host uint8 (nframes, H, W) buffers
        (contiguous, preferably pinned).  Returns (labels, energies, bounds)."""
        import torch
        n = int(left.shape[0])
        for t in (left, right):
            if t.device.type != "cpu" or not t.is_contiguous() or tuple(t.shape) != (n, self.H, self.W):
                raise DmmError("run_host_frames expects contiguous host (nframes, H, W) uint8 buffers")
        if labels_out is None:
            labels_out = torch.empty((n, self.H, self.W), dtype=torch.uint8).pin_memory()
        e = (ctypes.c_int64 * n)()
        b = (ctypes.c_int64 * n)()
        self._call("dmm_run_host_frames", frame, n, ctypes.c_void_p(left.data_ptr()),
                   ctypes.c_void_p(right.data_ptr()), iterations, ctypes.c_void_p(labels_out.data_ptr()), e, b,
                   _stream_handle(stream, self.device))
        for f in range(frame, frame + n):
            self._iters[f] = iterations
        return labels_out, [int(v) for v in e], [int(v) for v in b]

    def run_host(self, left, right, iterations: int = 4, labels_out=None, frame: int = 0, stream=None):
        """End-to-end through the C ABI with HOST buffers (numpy or CPU tensors,
        preferably pinned): H2D, cost volume, solve, energy, D2H.  Returns
        (labels_host, energy, bound)."""
        import torch

        def host_ptr(a):
            if isinstance(a, np.ndarray):
                a = np.ascontiguousarray(a, dtype=np.uint8)
                return a, a.ctypes.data
            if a.device.type != "cpu" or not a.is_contiguous():
                raise DmmError("run_host expects contiguous host buffers")
            return a, a.data_ptr()

        l, lp = host_ptr(left)
        r, rp = host_ptr(right)
        if labels_out is None:
            labels_out = torch.empty((self.H, self.W), dtype=torch.uint8).pin_memory()
        _, op = host_ptr(labels_out)
        e = ctypes.c_int64()
        b = ctypes.c_int64()
        self._call("dmm_run_host", frame, ctypes.c_void_p(lp), ctypes.c_void_p(rp), iterations,
                   ctypes.c_void_p(op), ctypes.byref(e), ctypes.byref(b), _stream_handle(stream, self.device))
        self._iters[frame] = iterations
        return labels_out, int(e.value), int(b.value)
