"""oracle — TEST INFRASTRUCTURE ONLY.

Python (ctypes + numpy) front end of oracle/oracle.c, the plain fp64 CPU
implementation of the sketched-EI CT operator pass (arXiv 2411.05771, Algorithm 1,
PAPER.md L108-L129).  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` leg may import this package.  It shares no code
with the CUDA path (paper_2411_05771_b200/) and never imports it.

All arrays are converted to C-contiguous fp64 before the call; every function is a
thin marshalling wrapper around the C routine of the same name (see oracle.c for
the cited definitions).  Pins: tests/test_oracle_pins.py; none is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

STREAM_ROT, STREAM_SKETCH, STREAM_NOISE, STREAM_PHANTOM = 1, 2, 3, 4
SHARED_IMAGE = (1 << 64) - 1
MODE_INTERLEAVED, MODE_UNIFORM = 0, 1


def build(force: bool = False) -> str:
    """Compile oracle.c with plain -O2 (no fast-math, no OpenMP)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fno-fast-math",
                               "-ffp-contract=off", "-o", _LIB_PATH, _SRC, "-lm"])
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        u64, i32 = ctypes.c_uint64, ctypes.c_int
        dp, ip = ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int)
        lib.oracle_word.restype = u64
        lib.oracle_word.argtypes = [u64, u64]
        lib.oracle_key.restype = u64
        lib.oracle_key.argtypes = [u64, u64, u64, u64]
        lib.oracle_draw.restype = i32
        lib.oracle_draw.argtypes = [u64, u64, u64, i32, i32, i32, ip, ip]
        lib.oracle_rotate.argtypes = [dp, dp, i32, i32]
        lib.oracle_rotate_adj.argtypes = [dp, dp, i32, i32]
        lib.oracle_rei_noise.argtypes = [u64, u64, u64, i32, i32, dp]
        lib.oracle_sketch_deviation.argtypes = [i32, i32, i32, ip, i32, i32, dp, dp,
                                                ctypes.POINTER(ctypes.c_double)]
        lib.oracle_pass_rei.argtypes = [dp, dp, i32, i32, i32, i32, ip, i32, ctypes.c_double,
                                        u64, u64, u64, dp, dp, dp, dp, dp, dp, dp,
                                        ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
        lib.oracle_ei_grad.argtypes = [dp, i32, i32, i32, i32, ip, i32, dp]
        lib.oracle_fwd.argtypes = [dp, dp, i32, i32, i32, ip, i32]
        lib.oracle_adj.argtypes = [dp, dp, i32, i32, i32, ip, i32, ctypes.c_double]
        lib.oracle_ramp.argtypes = [dp, dp, i32, i32]
        lib.oracle_fbp.argtypes = [dp, dp, i32, i32, i32, ip, i32, i32]
        lib.oracle_residual.argtypes = [dp, dp, ip, i32, i32, dp, dp, i32, dp, dp, dp]
        lib.oracle_pass.argtypes = [dp, dp, i32, i32, i32, i32, ip, i32, dp,
                                    dp, dp, dp, dp, dp, dp, dp, dp, dp]
        _lib = lib
    return _lib


def _d(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _dp(a):
    return None if a is None else a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _ip(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int))


def word(key: int, i: int) -> int:
    return int(_load().oracle_word(key, i))


def key(seed: int, stream: int, it: int, image: int) -> int:
    return int(_load().oracle_key(seed, stream, it, image))


def draw(seed: int, it: int, image: int, n_full: int, m: int, mode: int = MODE_UNIFORM):
    """(g_deg, idx[m]) — SURVEY §8(c) O-1.  image = SHARED_IMAGE for a per-pass draw."""
    g = ctypes.c_int(0)
    idx = np.zeros(m, dtype=np.int32)
    st = _load().oracle_draw(seed, it, image, n_full, m, mode, ctypes.byref(g), _ip(idx))
    if st != 0:
        raise ValueError(f"oracle_draw: config error (n_full={n_full}, m={m}, mode={mode})")
    return g.value, idx


def rotate(x, g: int):
    x = _d(x)
    out = np.empty_like(x)
    N = x.shape[-1]
    flat_in, flat_out = x.reshape(-1, N, N), out.reshape(-1, N, N)
    for b in range(flat_in.shape[0]):
        _load().oracle_rotate(_dp(flat_in[b]), _dp(flat_out[b]), N, int(g))
    return out


def rotate_adj(y, g: int):
    """T_g^T y (oracle.c oracle_rotate_adj) for one image or a batch sharing g."""
    y = _d(y)
    out = np.empty_like(y)
    N = y.shape[-1]
    flat_in, flat_out = y.reshape(-1, N, N), out.reshape(-1, N, N)
    for b in range(flat_in.shape[0]):
        _load().oracle_rotate_adj(_dp(flat_in[b]), _dp(flat_out[b]), N, int(g))
    return out


def ei_grad(x1, g: int, idx, n_full: int, n_det: int):
    """d ||x2 - x3||^2 / d x1 for one image, identity network (oracle.c oracle_ei_grad)."""
    x1, idx = _d(x1), _i(idx)
    N = x1.shape[-1]
    out = np.empty((N, N))
    _load().oracle_ei_grad(_dp(x1), N, n_det, n_full, int(g), _ip(idx), len(idx), _dp(out))
    return out


def fwd(x, idx, n_full: int, n_det: int):
    """A_S x for one image [N, N] or a batch [B, N, N] sharing idx."""
    x = _d(x)
    idx = _i(idx)
    N = x.shape[-1]
    xs = x.reshape(-1, N, N)
    out = np.empty((xs.shape[0], len(idx), n_det))
    for b in range(xs.shape[0]):
        _load().oracle_fwd(_dp(xs[b]), _dp(out[b]), N, n_det, n_full, _ip(idx), len(idx))
    return out.reshape(x.shape[:-2] + (len(idx), n_det))


def adj(p, idx, n_full: int, N: int, scale: float = 1.0):
    p = _d(p)
    idx = _i(idx)
    m, n_det = p.shape[-2], p.shape[-1]
    ps = p.reshape(-1, m, n_det)
    out = np.empty((ps.shape[0], N, N))
    for b in range(ps.shape[0]):
        _load().oracle_adj(_dp(ps[b]), _dp(out[b]), N, n_det, n_full, _ip(idx), m, float(scale))
    return out.reshape(p.shape[:-2] + (N, N))


def ramp(p):
    p = _d(p)
    n_det = p.shape[-1]
    ps = p.reshape(-1, n_det)
    out = np.empty_like(ps)
    _load().oracle_ramp(_dp(ps), _dp(out), ps.shape[0], n_det)
    return out.reshape(p.shape)


def fbp(p, idx, n_full: int, N: int, m_total: int | None = None):
    p = _d(p)
    idx = _i(idx)
    m, n_det = p.shape[-2], p.shape[-1]
    ps = p.reshape(-1, m, n_det)
    out = np.empty((ps.shape[0], N, N))
    for b in range(ps.shape[0]):
        _load().oracle_fbp(_dp(ps[b]), _dp(out[b]), N, n_det, n_full, _ip(idx), m,
                           int(m_total or m))
    return out.reshape(p.shape[:-2] + (N, N))


def residual(p1, y, idx, x2, x3):
    """One image: (mc, ei, r)."""
    p1, y, x2, x3, idx = _d(p1), _d(y), _d(x2), _d(x3), _i(idx)
    m, n_det = p1.shape
    r = np.empty_like(p1)
    mc, ei = ctypes.c_double(0), ctypes.c_double(0)
    _load().oracle_residual(_dp(p1), _dp(y), _ip(idx), m, n_det, _dp(x2), _dp(x3),
                            x2.shape[-1], ctypes.byref(mc), ctypes.byref(ei), _dp(r))
    return mc.value, ei.value, r


def sketched_pass(x1, y, g: int, idx, n_full: int, x3=None):
    """The whole pass for one image (oracle.c oracle_pass).  Returns a dict of fp64 arrays."""
    x1, y, idx = _d(x1), _d(y), _i(idx)
    N = x1.shape[-1]
    n_det = y.shape[-1]
    m = len(idx)
    out = {k: np.empty((N, N)) for k in ("x2", "xfbp", "grad")}
    out.update({k: np.empty((m, n_det)) for k in ("p1", "p2", "q", "r")})
    mc, ei = ctypes.c_double(0), ctypes.c_double(0)
    x3d = None if x3 is None else _d(x3)
    _load().oracle_pass(_dp(x1), _dp(y), N, n_det, n_full, int(g), _ip(idx), m, _dp(x3d),
                        _dp(out["x2"]), _dp(out["p1"]), _dp(out["p2"]), _dp(out["q"]),
                        _dp(out["xfbp"]), _dp(out["r"]), _dp(out["grad"]),
                        ctypes.byref(mc), ctypes.byref(ei))
    out["mc"], out["ei"] = mc.value, ei.value
    return out


def rei_noise(seed: int, it: int, image: int, m: int, n_det: int):
    """eps [m][n_det] ~ N(0,1) of the REI pass (oracle.c oracle_rei_noise)."""
    out = np.empty((m, n_det))
    _load().oracle_rei_noise(seed, it, image, m, n_det, _dp(out))
    return out


def sketched_pass_rei(x1, y, g: int, idx, n_full: int, sigma: float, seed: int, it: int,
                      image: int):
    """The REI pass for one image (oracle.c oracle_pass_rei): q = ramp(p2 + sigma eps)."""
    x1, y, idx = _d(x1), _d(y), _i(idx)
    N = x1.shape[-1]
    n_det = y.shape[-1]
    m = len(idx)
    out = {k: np.empty((N, N)) for k in ("x2", "xfbp", "grad")}
    out.update({k: np.empty((m, n_det)) for k in ("p1", "p2", "q", "r")})
    mc, ei = ctypes.c_double(0), ctypes.c_double(0)
    _load().oracle_pass_rei(_dp(x1), _dp(y), N, n_det, n_full, int(g), _ip(idx), m, float(sigma),
                            seed, it, image, _dp(out["x2"]), _dp(out["p1"]), _dp(out["p2"]),
                            _dp(out["q"]), _dp(out["xfbp"]), _dp(out["r"]), _dp(out["grad"]),
                            ctypes.byref(mc), ctypes.byref(ei))
    out["mc"], out["ei"] = mc.value, ei.value
    return out


def sketch_deviation(v0, idx, n_full: int, n_det: int, iters: int):
    """(lambda, v): power-iteration estimate of ||A^T (S^T S - I) A||_2 (oracle.c
    oracle_sketch_deviation) from the start image v0 [N, N]."""
    v0, idx = _d(v0), _i(idx)
    N = v0.shape[-1]
    v = np.empty((N, N))
    lam = ctypes.c_double(0)
    _load().oracle_sketch_deviation(N, n_det, n_full, _ip(idx), len(idx), int(iters), _dp(v0),
                                    _dp(v), ctypes.byref(lam))
    return lam.value, v

