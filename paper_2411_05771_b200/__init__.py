"""paper_2411_05771_b200 — B200-native sketched Equivariant Imaging operator pass.

Thin Python binding over the C ABI of include/skei.h (libskei.so, hand-written CUDA for
sm_100a).  Argument marshalling only: every step of the pass runs in the library's
kernels.  torch supplies device memory and the current CUDA stream.  There is no CPU
fallback: if libskei.so is missing or no sm_100 device is present the calls raise.

Names follow the C ABI (and the paper's notation, arXiv 2411.05771 Algorithm 1):
    draw, draw_device        a1  (g, S) ~ G x sketches
    rotate                   a2  x2 = T_g x1                       L120
    radon_fwd                a3  A_S x                             L92, L283
    ramp_filter              a4  Ram-Lak ramp (FFT)                L283 (iradon)
    fbp                      a4+a5  A_S^+ = (pi/2m) A_S^T ramp     L92, L102
    radon_adj                a5/a8  A_S^T p                        L122
    ei_residual              a7  r, ||y_S - A_S x1||^2, ||x2-x3||^2  L122
    sketched_pass            the whole pass (skei_pass)
    sketched_pass_host       the whole pass from host buffers (skei_pass_host)
"""
from __future__ import annotations

import ctypes
import os
import threading

import torch

__all__ = [
    "Plan", "SkeiError", "lib", "lib_path", "draw", "draw_device", "rotate", "radon_fwd",
    "radon_adj", "ramp_filter", "fbp", "ei_residual", "sketched_pass", "sketched_pass_host",
    "sketched_pass_profiled", "sketched_pass_draw", "smem_probe", "l2_probe", "alloc_pass_outputs",
    "workspace_bytes", "MODE_INTERLEAVED", "MODE_UNIFORM", "SHARED_IMAGE", "version",
]

MODE_INTERLEAVED, MODE_UNIFORM = 0, 1
SHARED_IMAGE = (1 << 64) - 1

_HERE = os.path.dirname(os.path.abspath(__file__))
lib_path = os.environ.get("SKEI_LIB") or os.path.join(_HERE, "libskei.so")  # override: A/B diagnostics
_lib = None
_lock = threading.Lock()


class SkeiError(RuntimeError):
    pass


class _Geom(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("n_det", ctypes.c_int32), ("n_full", ctypes.c_int32),
                ("fft_len", ctypes.c_int32)]


class _PassOut(ctypes.Structure):
    _fields_ = [(k, ctypes.c_void_p) for k in ("x2", "p1", "p2", "q", "xfbp", "r", "grad", "mc", "ei")]


class _DrawSpec(ctypes.Structure):  # skei_draw_spec
    _fields_ = [("seed", ctypes.c_uint64), ("iter", ctypes.c_uint64), ("image0", ctypes.c_uint64),
                ("shared", ctypes.c_int32), ("mode", ctypes.c_int32)]


def lib():
    """Load libskei.so (raises if the CUDA extension has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(lib_path):
            raise SkeiError(f"CUDA extension missing: {lib_path} (run __graft_entry__.build())")
        L = ctypes.CDLL(lib_path)
        vp, i32, u64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint64, ctypes.c_size_t
        st = ctypes.c_int
        sig = {
            "skei_plan_create": ([ctypes.POINTER(_Geom), ctypes.c_int, ctypes.POINTER(vp)], st),
            "skei_plan_destroy": ([vp], None),
            "skei_plan_geometry": ([vp, ctypes.POINTER(_Geom)], st),
            "skei_status_string": ([st], ctypes.c_char_p),
            "skei_last_cuda_error": ([], ctypes.c_char_p),
            "skei_workspace_bytes": ([vp, i32, i32], sz),
            "skei_draw": ([u64, u64, u64, i32, i32, i32, vp, vp], st),
            "skei_draw_device": ([u64, u64, u64, i32, i32, i32, i32, i32, vp, vp, vp], st),
            "skei_rotate": ([vp, vp, vp, i32, vp, i32, vp], st),
            "skei_rotate_adjoint": ([vp, vp, vp, i32, vp, i32, vp], st),
            "skei_ei_grad": ([vp, i32, vp, vp, vp, i32, vp, i32, i32, vp, vp, sz, vp], st),
            "skei_fbp_adjoint": ([vp, vp, vp, i32, vp, i32, i32, i32, vp, sz, vp], st),
            "skei_pass_rei": ([vp, i32, vp, vp, vp, i32, vp, i32, i32, ctypes.c_float, u64, u64,
                               u64, vp, vp, sz, vp], st),
            "skei_sketch_deviation": ([vp, i32, vp, i32, i32, i32, vp, vp, vp, sz, vp], st),
            "skei_ramp_allgather": ([vp, i32, vp, vp, i32, i32, i32, vp, vp, vp, i32, vp], st),
            "skei_backproject_band": ([vp, i32, vp, vp, vp, i32, i32, i32, vp, i32, i32, vp, vp,
                                       vp, vp, sz, vp], st),
            "skei_rs_recv_floats": ([vp, i32, i32], sz),
            "skei_backproject_scatter": ([vp, i32, vp, vp, vp, i32, i32, i32, vp, i32, i32, vp],
                                         st),
            "skei_band_reduce": ([vp, i32, vp, i32, i32, vp, vp, vp, vp, vp, sz, vp], st),
            "skei_radon_fwd": ([vp, vp, vp, i32, vp, i32, i32, vp, sz, vp], st),
            "skei_radon_adj": ([vp, vp, vp, i32, vp, i32, i32, ctypes.c_float, vp], st),
            "skei_ramp_filter": ([vp, vp, vp, i32, vp], st),
            "skei_fbp": ([vp, vp, vp, i32, vp, i32, i32, i32, vp, sz, vp], st),
            "skei_ei_residual": ([vp, vp, vp, vp, i32, i32, vp, vp, i32, vp, vp, vp, vp, sz, vp], st),
            "skei_pass": ([vp, i32, vp, vp, vp, i32, vp, i32, i32, vp, ctypes.POINTER(_PassOut),
                           vp, sz, vp], st),
            "skei_pass_host": ([vp, i32, vp, vp, vp, i32, vp, i32, i32, vp, vp, vp, vp,
                                ctypes.POINTER(_PassOut), vp, vp, vp, vp, sz, vp], st),
            "skei_pass_profiled": ([vp, i32, vp, vp, vp, i32, vp, i32, i32, ctypes.POINTER(_PassOut),
                                    vp, sz, ctypes.POINTER(vp), i32, vp], st),
            "skei_pass_draw": ([vp, i32, vp, vp, ctypes.POINTER(_DrawSpec), i32, vp, vp,
                                ctypes.POINTER(_PassOut), vp, sz, ctypes.POINTER(vp), i32, vp], st),
            "skei_smem_probe": ([vp, i32, i32, vp], st),
            "skei_l2_probe": ([vp, ctypes.c_int64, vp, i32, i32, vp], st),
            "skei_version": ([], ctypes.c_char_p),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def version() -> str:
    return lib().skei_version().decode()


def _check(status: int, what: str):
    if status != 0:
        msg = lib().skei_status_string(status).decode()
        if status == 4:
            msg += ": " + lib().skei_last_cuda_error().decode()
        raise SkeiError(f"{what}: {msg} (status {status})")


def _stream(t: torch.Tensor):
    return ctypes.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def _ptr(t: torch.Tensor | None, dtype=torch.float32, name="tensor"):
    if t is None:
        return None
    if not t.is_cuda:
        raise SkeiError(f"{name}: expected a CUDA tensor")
    if t.dtype != dtype:
        raise SkeiError(f"{name}: expected {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise SkeiError(f"{name}: expected a contiguous tensor")
    return ctypes.c_void_p(t.data_ptr())


class Plan:
    """skei_plan: immutable geometry tables on one device (fp64 trig, ramp spectrum, twiddles)."""

    _cache: dict = {}

    def __init__(self, n: int, n_det: int, n_full: int, fft_len: int = 0, device: int | None = None):
        if device is None:
            device = torch.cuda.current_device()
        g = _Geom(n, n_det, n_full, fft_len)
        h = ctypes.c_void_p()
        _check(lib().skei_plan_create(ctypes.byref(g), int(device), ctypes.byref(h)), "skei_plan_create")
        self._h = h
        out = _Geom()
        _check(lib().skei_plan_geometry(h, ctypes.byref(out)), "skei_plan_geometry")
        self.n, self.n_det, self.n_full, self.fft_len = out.n, out.n_det, out.n_full, out.fft_len
        self.device = int(device)

    @classmethod
    def get(cls, n, n_det, n_full, fft_len=0, device=None):
        if device is None:
            device = torch.cuda.current_device()
        key = (n, n_det, n_full, fft_len, device)
        if key not in cls._cache:
            cls._cache[key] = cls(n, n_det, n_full, fft_len, device)
        return cls._cache[key]

    @property
    def handle(self):
        return self._h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            try:
                _lib.skei_plan_destroy(h)
            except Exception:
                pass
            self._h = None

    def workspace(self, B: int, m: int) -> torch.Tensor:
        nbytes = workspace_bytes(self, B, m)
        return torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{self.device}")


def workspace_bytes(plan: Plan, B: int, m: int) -> int:
    return int(lib().skei_workspace_bytes(plan.handle, B, m))


def draw(seed: int, it: int, image: int, n_full: int, m: int, mode: int = MODE_UNIFORM):
    """Host draw (skei_draw): returns (g_deg, list of m ascending angle indices)."""
    g = ctypes.c_int32(0)
    idx = (ctypes.c_int32 * m)()
    _check(lib().skei_draw(seed, it, image, n_full, m, mode, ctypes.byref(g), idx), "skei_draw")
    return g.value, list(idx)


def draw_device(seed: int, it: int, image0: int, count: int, shared: bool, n_full: int, m: int,
                mode: int = MODE_UNIFORM, g: torch.Tensor | None = None,
                idx: torch.Tensor | None = None, device=None):
    """Device draws (skei_draw_device) into int32 tensors g[count], idx[count, m]."""
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    if g is None:
        g = torch.empty(count, dtype=torch.int32, device=dev)
    if idx is None:
        idx = torch.empty(count, m, dtype=torch.int32, device=dev)
    _check(lib().skei_draw_device(seed, it, image0, count, int(bool(shared)), n_full, m, mode,
                                  _ptr(g, torch.int32, "g"), _ptr(idx, torch.int32, "idx"), _stream(g)),
           "skei_draw_device")
    return g, idx


def _idx_stride(idx: torch.Tensor, B: int, m: int) -> int:
    if idx.dim() == 1 or idx.shape[0] == 1:
        return 0
    if idx.shape[0] != B:
        raise SkeiError(f"idx: expected [m] or [B, m], got {tuple(idx.shape)}")
    return m


def rotate(plan: Plan, x: torch.Tensor, g: torch.Tensor, out: torch.Tensor | None = None):
    B = x.shape[0]
    out = torch.empty_like(x) if out is None else out
    g_stride = 0 if g.numel() == 1 else 1
    _check(lib().skei_rotate(plan.handle, _ptr(x, name="x"), _ptr(out, name="out"), B,
                             _ptr(g, torch.int32, "g"), g_stride, _stream(x)), "skei_rotate")
    return out


def rotate_adjoint(plan: Plan, y: torch.Tensor, g: torch.Tensor, out: torch.Tensor | None = None):
    """skei_rotate_adjoint: T_g^T y (the transpose of `rotate`)."""
    B = y.shape[0]
    out = torch.empty_like(y) if out is None else out
    g_stride = 0 if g.numel() == 1 else 1
    _check(lib().skei_rotate_adjoint(plan.handle, _ptr(y, name="y"), _ptr(out, name="out"), B,
                                     _ptr(g, torch.int32, "g"), g_stride, _stream(y)),
           "skei_rotate_adjoint")
    return out


def fbp_adjoint(plan: Plan, x: torch.Tensor, idx: torch.Tensor, m_total: int | None = None,
                out: torch.Tensor | None = None, ws: torch.Tensor | None = None):
    """skei_fbp_adjoint: (pi / 2 m_total) ramp(A_S x), the transpose of `fbp`."""
    B, m = x.shape[0], idx.shape[-1]
    p = torch.empty(B, m, plan.n_det, dtype=torch.float32, device=x.device) if out is None else out
    ws = plan.workspace(B, m) if ws is None else ws
    _check(lib().skei_fbp_adjoint(plan.handle, _ptr(x, name="x"), _ptr(p, name="p"), B,
                                  _ptr(idx, torch.int32, "idx"), m, _idx_stride(idx, B, m),
                                  int(m_total or m), _ptr(ws, torch.uint8, "ws"), ws.numel(),
                                  _stream(x)), "skei_fbp_adjoint")
    return p


def ramp_allgather(plan: Plan, p: torch.Tensor, r: torch.Tensor, row0: int, m_total: int,
                   peer_q: list, peer_r: list, q_local: torch.Tensor | None = None):
    """skei_ramp_allgather: q_local = ramp(p) and, fused in the same kernel, every row of q and
    of r stored into rows row0.. of each peer buffer (device pointers, ints)."""
    B, m_local = p.shape[0], p.shape[1]
    q_local = torch.empty_like(p) if q_local is None else q_local
    n = len(peer_q)
    arr_q = (ctypes.c_void_p * n)(*[ctypes.c_void_p(int(x)) for x in peer_q])
    arr_r = (ctypes.c_void_p * n)(*[ctypes.c_void_p(int(x)) for x in peer_r])
    _check(lib().skei_ramp_allgather(plan.handle, B, _ptr(p, name="p"), _ptr(r, name="r"), m_local,
                                     int(row0), int(m_total), _ptr(q_local, name="q_local"), arr_q,
                                     arr_r, n, _stream(p)), "skei_ramp_allgather")
    return q_local


def backproject_band(plan: Plan, q: torch.Tensor, r: torch.Tensor, idx: torch.Tensor,
                     x2: torch.Tensor, row0: int, rows: int, m_total: int | None = None,
                     ws: torch.Tensor | None = None):
    """skei_backproject_band: (x_fbp band, grad band, ei band partial) for output rows
    [row0, row0 + rows) from the whole filtered sinogram q and residual r."""
    B, m = q.shape[0], idx.shape[-1]
    xf = torch.empty(B, rows, plan.n, dtype=torch.float32, device=q.device)
    gr = torch.empty_like(xf)
    ei = torch.empty(B, dtype=torch.float32, device=q.device)
    ws = plan.workspace(B, m) if ws is None else ws
    _check(lib().skei_backproject_band(plan.handle, B, _ptr(q, name="q"), _ptr(r, name="r"),
                                       _ptr(idx, torch.int32, "idx"), m, _idx_stride(idx, B, m),
                                       int(m_total or m), _ptr(x2, name="x2"), int(row0),
                                       int(rows), _ptr(xf, name="xfbp"), _ptr(gr, name="grad"),
                                       _ptr(ei, name="ei"), _ptr(ws, torch.uint8, "ws"),
                                       ws.numel(), _stream(q)), "skei_backproject_band")
    return xf, gr, ei


def rs_recv_floats(plan: Plan, B: int, world: int) -> int:
    """skei_rs_recv_floats: floats of one rank's receive buffer [world][2][B][bmax][n]."""
    return int(lib().skei_rs_recv_floats(plan.handle, int(B), int(world)))


def backproject_scatter(plan: Plan, q: torch.Tensor, r: torch.Tensor, idx: torch.Tensor,
                        m_total: int, peer_recv: list, rank: int):
    """skei_backproject_scatter: this rank's angle-shard partials of x_fbp and grad, every
    output row stored by the kernel's epilogue into its band owner's receive buffer (device
    pointers, ints; slot `rank`)."""
    B, m = q.shape[0], idx.shape[-1]
    n = len(peer_recv)
    arr = (ctypes.c_void_p * n)(*[ctypes.c_void_p(int(x)) for x in peer_recv])
    _check(lib().skei_backproject_scatter(plan.handle, B, _ptr(q, name="q"), _ptr(r, name="r"),
                                          _ptr(idx, torch.int32, "idx"), m,
                                          _idx_stride(idx, B, m), int(m_total), arr, n,
                                          int(rank), _stream(q)), "skei_backproject_scatter")


def band_reduce(plan: Plan, recv: torch.Tensor, world: int, rank: int, x2: torch.Tensor,
                ws: torch.Tensor | None = None):
    """skei_band_reduce: (x_fbp band, grad band, ei band partial) of `rank` from its receive
    buffer (the world slots summed in rank order)."""
    B, n = x2.shape[0], plan.n
    q, rem = divmod(n, world)
    rows = q + (1 if rank < rem else 0)
    xf = torch.empty(B, rows, n, dtype=torch.float32, device=x2.device)
    gr = torch.empty_like(xf)
    ei = torch.empty(B, dtype=torch.float32, device=x2.device)
    ws = plan.workspace(B, 1) if ws is None else ws
    _check(lib().skei_band_reduce(plan.handle, B, _ptr(recv, name="recv"), int(world), int(rank),
                                  _ptr(x2, name="x2"), _ptr(xf, name="xfbp"), _ptr(gr, name="grad"),
                                  _ptr(ei, name="ei"), _ptr(ws, torch.uint8, "ws"), ws.numel(),
                                  _stream(x2)), "skei_band_reduce")
    return xf, gr, ei


def sketch_deviation(plan: Plan, idx: torch.Tensor, v: torch.Tensor, iters: int,
                     ws: torch.Tensor | None = None):
    """skei_sketch_deviation: ||A^T (S^T S - I) A||_2 by power iteration from the start images
    v [B][n][n] (overwritten by the last iterate).  Returns lambda [B]."""
    B, m = v.shape[0], idx.shape[-1]
    lam = torch.empty(B, dtype=torch.float32, device=v.device)
    ws = plan.workspace(B, plan.n_full) if ws is None else ws
    _check(lib().skei_sketch_deviation(plan.handle, B, _ptr(idx, torch.int32, "idx"), m,
                                       _idx_stride(idx, B, m), int(iters), _ptr(v, name="v"),
                                       _ptr(lam, name="lambda"), _ptr(ws, torch.uint8, "ws"),
                                       ws.numel(), _stream(v)), "skei_sketch_deviation")
    return lam


def ei_grad(plan: Plan, x2: torch.Tensor, x3: torch.Tensor, g: torch.Tensor, idx: torch.Tensor,
            out: torch.Tensor | None = None, ws: torch.Tensor | None = None):
    """skei_ei_grad: d ||x2 - x3||^2 / d x1 for x2 = T_g x1 and the identity network
    x3 = (pi/2m) A_S^T ramp A_S x2 (pass x2 and xfbp of the same draw)."""
    B, m = x2.shape[0], idx.shape[-1]
    out = torch.empty_like(x2) if out is None else out
    ws = plan.workspace(B, m) if ws is None else ws
    _check(lib().skei_ei_grad(plan.handle, B, _ptr(x2, name="x2"), _ptr(x3, name="x3"),
                              _ptr(g, torch.int32, "g"), 0 if g.numel() == 1 else 1,
                              _ptr(idx, torch.int32, "idx"), m, _idx_stride(idx, B, m),
                              _ptr(out, name="grad"), _ptr(ws, torch.uint8, "ws"), ws.numel(),
                              _stream(x2)), "skei_ei_grad")
    return out


def radon_fwd(plan: Plan, x: torch.Tensor, idx: torch.Tensor, out: torch.Tensor | None = None,
              ws: torch.Tensor | None = None):
    B, m = x.shape[0], idx.shape[-1]
    p = torch.empty(B, m, plan.n_det, dtype=torch.float32, device=x.device) if out is None else out
    ws = plan.workspace(B, m) if ws is None else ws
    _check(lib().skei_radon_fwd(plan.handle, _ptr(x, name="x"), _ptr(p, name="p"), B,
                                _ptr(idx, torch.int32, "idx"), m, _idx_stride(idx, B, m),
                                _ptr(ws, torch.uint8, "ws"), ws.numel(), _stream(x)),
           "skei_radon_fwd")
    return p


def radon_adj(plan: Plan, p: torch.Tensor, idx: torch.Tensor, scale: float = 1.0,
              out: torch.Tensor | None = None):
    B, m = p.shape[0], p.shape[1]
    x = torch.empty(B, plan.n, plan.n, dtype=torch.float32, device=p.device) if out is None else out
    _check(lib().skei_radon_adj(plan.handle, _ptr(p, name="p"), _ptr(x, name="x"), B,
                                _ptr(idx, torch.int32, "idx"), m, _idx_stride(idx, B, m),
                                ctypes.c_float(scale), _stream(p)), "skei_radon_adj")
    return x


def ramp_filter(plan: Plan, p: torch.Tensor, out: torch.Tensor | None = None):
    rows = p.numel() // plan.n_det
    q = torch.empty_like(p) if out is None else out
    _check(lib().skei_ramp_filter(plan.handle, _ptr(p, name="p"), _ptr(q, name="q"), rows, _stream(p)),
           "skei_ramp_filter")
    return q


def fbp(plan: Plan, p: torch.Tensor, idx: torch.Tensor, m_total: int | None = None,
        out: torch.Tensor | None = None, ws: torch.Tensor | None = None):
    B, m = p.shape[0], p.shape[1]
    x = torch.empty(B, plan.n, plan.n, dtype=torch.float32, device=p.device) if out is None else out
    ws = plan.workspace(B, m) if ws is None else ws
    _check(lib().skei_fbp(plan.handle, _ptr(p, name="p"), _ptr(x, name="x"), B,
                          _ptr(idx, torch.int32, "idx"), m, _idx_stride(idx, B, m), int(m_total or m),
                          _ptr(ws, torch.uint8, "ws"), ws.numel(), _stream(p)), "skei_fbp")
    return x


def ei_residual(plan: Plan, p1, y, idx, x2, x3, r: torch.Tensor | None = None, want_r: bool = True,
                ws: torch.Tensor | None = None):
    """(mc, ei, r).  p1 = y = None computes only ei; x2 = x3 = None only (mc, r)."""
    ref = p1 if p1 is not None else x2
    B, m = ref.shape[0], idx.shape[-1]
    dev = ref.device
    mc = torch.empty(B, dtype=torch.float32, device=dev) if p1 is not None else None
    ei = torch.empty(B, dtype=torch.float32, device=dev) if x2 is not None else None
    if p1 is None:
        want_r = False
    if want_r and r is None:
        r = torch.empty_like(p1)
    ws = plan.workspace(B, m) if ws is None else ws
    _check(lib().skei_ei_residual(plan.handle, _ptr(p1, name="p1"), _ptr(y, name="y"),
                                  _ptr(idx, torch.int32, "idx"), m, _idx_stride(idx, B, m),
                                  _ptr(x2, name="x2"), _ptr(x3, name="x3"), B, _ptr(mc), _ptr(ei),
                                  _ptr(r) if want_r else None, _ptr(ws, torch.uint8, "ws"),
                                  ws.numel(), _stream(ref)), "skei_ei_residual")
    return mc, ei, r


def alloc_pass_outputs(plan: Plan, B: int, m: int, device) -> dict:
    f = dict(dtype=torch.float32, device=device)
    img = (B, plan.n, plan.n)
    sino = (B, m, plan.n_det)
    return {"x2": torch.empty(img, **f), "p1": torch.empty(sino, **f), "p2": torch.empty(sino, **f),
            "q": torch.empty(sino, **f), "xfbp": torch.empty(img, **f), "r": torch.empty(sino, **f),
            "grad": torch.empty(img, **f), "mc": torch.empty(B, **f), "ei": torch.empty(B, **f)}


def _pass_out(o: dict) -> _PassOut:
    return _PassOut(*[ctypes.c_void_p(o[k].data_ptr()) for k in
                      ("x2", "p1", "p2", "q", "xfbp", "r", "grad", "mc", "ei")])


def sketched_pass(plan: Plan, x1, y, g, idx, x3=None, out: dict | None = None,
                  ws: torch.Tensor | None = None):
    """skei_pass: the whole sketched-EI operator pass.  Returns the dict of outputs."""
    B, m = x1.shape[0], idx.shape[-1]
    out = alloc_pass_outputs(plan, B, m, x1.device) if out is None else out
    ws = plan.workspace(B, m) if ws is None else ws
    po = _pass_out(out)
    _check(lib().skei_pass(plan.handle, B, _ptr(x1, name="x1"), _ptr(y, name="y"),
                           _ptr(g, torch.int32, "g"), 0 if g.numel() == 1 else 1,
                           _ptr(idx, torch.int32, "idx"), m, _idx_stride(idx, B, m),
                           _ptr(x3, name="x3"), ctypes.byref(po), _ptr(ws, torch.uint8, "ws"),
                           ws.numel(), _stream(x1)), "skei_pass")
    return out


def sketched_pass_rei(plan: Plan, x1, y, g, idx, sigma: float, noise_seed: int, noise_iter: int,
                      image0: int = 0, out: dict | None = None, ws: torch.Tensor | None = None):
    """skei_pass_rei: the REI pass, q = ramp(p2 + sigma eps)."""
    B, m = x1.shape[0], idx.shape[-1]
    out = alloc_pass_outputs(plan, B, m, x1.device) if out is None else out
    ws = plan.workspace(B, m) if ws is None else ws
    po = _pass_out(out)
    _check(lib().skei_pass_rei(plan.handle, B, _ptr(x1, name="x1"), _ptr(y, name="y"),
                               _ptr(g, torch.int32, "g"), 0 if g.numel() == 1 else 1,
                               _ptr(idx, torch.int32, "idx"), m, _idx_stride(idx, B, m),
                               float(sigma), int(noise_seed), int(noise_iter), int(image0),
                               ctypes.byref(po), _ptr(ws, torch.uint8, "ws"), ws.numel(),
                               _stream(x1)), "skei_pass_rei")
    return out


def sketched_pass_profiled(plan: Plan, x1, y, g, idx, events, out: dict, ws: torch.Tensor):
    """skei_pass_profiled: skei_pass with up to 6 caller-owned torch.cuda.Events (None =
    skipped) recorded at the stage boundaries: 0 start, 1 after rotate+pack, 2 after the
    forward (with fused MC residual), 3 after the ramp, 4 after the backprojections (with
    fused EI residual), 5 end."""
    B, m = x1.shape[0], idx.shape[-1]
    po = _pass_out(out)
    for e in events:  # torch creates the cudaEvent_t lazily, on its first record()
        if e is not None and e.cuda_event == 0:
            e.record()
    ev = (ctypes.c_void_p * len(events))(*[ctypes.c_void_p(e.cuda_event if e is not None else 0)
                                            for e in events])
    _check(lib().skei_pass_profiled(plan.handle, B, _ptr(x1, name="x1"), _ptr(y, name="y"),
                                    _ptr(g, torch.int32, "g"), 0 if g.numel() == 1 else 1,
                                    _ptr(idx, torch.int32, "idx"), m, _idx_stride(idx, B, m),
                                    ctypes.byref(po), _ptr(ws, torch.uint8, "ws"), ws.numel(), ev,
                                    len(events), _stream(x1)), "skei_pass_profiled")
    return out


def _events_arg(events):
    if events is None:
        return None, 0
    for e in events:  # torch creates the cudaEvent_t lazily, on its first record()
        if e is not None and e.cuda_event == 0:
            e.record()
    ev = (ctypes.c_void_p * len(events))(*[ctypes.c_void_p(e.cuda_event if e is not None else 0)
                                            for e in events])
    return ev, len(events)


def sketched_pass_draw(plan: Plan, x1, y, seed: int, it: int, m: int, mode: int = MODE_UNIFORM,
                       shared: bool = True, image0: int = 0, g: torch.Tensor | None = None,
                       idx: torch.Tensor | None = None, out: dict | None = None,
                       ws: torch.Tensor | None = None, events=None):
    """skei_pass_draw: the device draw (a1) and the pass on it in one call; the draw is
    written to g [1 or B] and idx [1 or B, m].  events: None or >= 6 stage events as in
    sketched_pass_profiled (event 0 before the draw).  Returns (out, g, idx)."""
    B = x1.shape[0]
    nd = 1 if shared else B
    if g is None:
        g = torch.empty(nd, dtype=torch.int32, device=x1.device)
    if idx is None:
        idx = torch.empty(nd, m, dtype=torch.int32, device=x1.device)
    if g.numel() != nd or idx.numel() != nd * m:
        raise SkeiError(f"g, idx: expected [{nd}] and [{nd}, {m}]")
    out = alloc_pass_outputs(plan, B, m, x1.device) if out is None else out
    ws = plan.workspace(B, m) if ws is None else ws
    po = _pass_out(out)
    spec = _DrawSpec(int(seed), int(it), int(image0), int(bool(shared)), int(mode))
    ev, nev = _events_arg(events)
    _check(lib().skei_pass_draw(plan.handle, B, _ptr(x1, name="x1"), _ptr(y, name="y"),
                                ctypes.byref(spec), m, _ptr(g, torch.int32, "g"),
                                _ptr(idx, torch.int32, "idx"), ctypes.byref(po),
                                _ptr(ws, torch.uint8, "ws"), ws.numel(), ev, nev, _stream(x1)),
           "skei_pass_draw")
    return out, g, idx


def l2_probe(buf: torch.Tensor, blocks: int, iters: int, sink: torch.Tensor):
    """skei_l2_probe (diagnostic): L2 read bandwidth; bytes = blocks*buf.numel()*4*iters."""
    _check(lib().skei_l2_probe(_ptr(buf, name="buf"), buf.numel(), _ptr(sink, name="sink"), blocks,
                               iters, _stream(sink)), "skei_l2_probe")


def smem_probe(blocks: int, iters: int, sink: torch.Tensor):
    """skei_smem_probe (diagnostic): shared-memory read bandwidth; bytes = blocks*1024*16*32*iters."""
    _check(lib().skei_smem_probe(_ptr(sink, name="sink"), blocks, iters, _stream(sink)), "skei_smem_probe")


def sketched_pass_host(plan: Plan, h_x1, h_y, h_g, h_idx, d: dict, h_mc, h_ei, ws, stream_tensor,
                       h_ystage=None):
    """skei_pass_host: H2D of (x1, y_S or y, g, idx) from (pinned) host tensors into d['x1'],
    d['y'], d['g'], d['idx'], the pass, and D2H of mc/ei into h_mc/h_ei (asynchronous).
    h_ystage: optional pinned host staging tensor (>= B*m*n_det floats) for the gathered y_S."""
    B, m = h_x1.shape[0], h_idx.shape[-1]
    po = _pass_out(d)
    g_stride = 0 if h_g.numel() == 1 else 1
    idx_stride = 0 if (h_idx.dim() == 1 or h_idx.shape[0] == 1) else m
    hp = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    _check(lib().skei_pass_host(plan.handle, B, hp(h_x1), hp(h_y), hp(h_g), g_stride, hp(h_idx), m,
                                idx_stride, hp(d["x1"]), hp(d["y"]), hp(d["g"]), hp(d["idx"]),
                                ctypes.byref(po), hp(h_mc), hp(h_ei),
                                hp(h_ystage) if h_ystage is not None else None, hp(ws), ws.numel(),
                                _stream(stream_tensor)), "skei_pass_host")
