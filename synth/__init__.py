"""synth — seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the method's arithmetic (no discrete projector, no ramp
filter, no backprojection, no rotation).  It only produces *inputs*:

* random-ellipse phantoms x† (the stand-in for the paper's CT100 slice, PAPER.md
  L283-L284, §3.1 "Sparse-view CT imaging": one 512×512 slice), rasterised with
  4×4 supersampling;
* the measured data y = (continuous Radon transform of the ellipses, sampled at the
  detector centres) + Gaussian noise, i.e. y = A x† + ε of PAPER.md L36-L39 (Eq. 1)
  generated from the *continuous* object, not from the discrete operator A under
  test (no inverse crime, and no dependence on either implementation);
* seeded random arrays for operator-level parity cases.

Geometry conventions used for the analytic
sinogram: pixel centres u_c = c-(N-1)/2, v_r = (N-1)/2-r; detector s_j = j-(n_det-1)/2;
θ_i = iπ/n_full.  Every phantom is a sum of ellipses (Shepp-Logan convention, additive
intensities), rescaled by one constant so that the rasterised image lies in [0, 1];
the analytic sinogram is rescaled by the same constant (the Radon transform is linear).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

__all__ = [
    "Config", "CONFIGS", "phantom_params", "rasterize", "analytic_sinogram",
    "make_phantoms", "make_measurements", "make_workload", "rand_images", "rand_sinograms",
]


@dataclasses.dataclass(frozen=True)
class Config:
    """One BASELINE.json config (configs[0..4]); `name` is cfg1..cfg5."""
    name: str
    N: int            # image side
    B: int            # batch (images per pass)
    n_full: int       # full angle set θ_i = iπ/n_full
    n_det: int        # detector bins, Δs = 1 px
    m: int            # sketch size
    fft_len: int      # ramp FFT length P (pow2 ≥ 2 n_det − 1)
    phantom: str      # "ellipses" | "nested"
    K: int            # ellipses per phantom
    noise: float      # σ = noise·max|y_clean| per image
    per_image_draws: bool  # fresh (g, S) per image (cfg4) or one shared draw per pass


CONFIGS = {
    "cfg1": Config("cfg1", 64, 2, 32, 91, 8, 256, "ellipses", 5, 0.01, False),
    "cfg2": Config("cfg2", 256, 8, 128, 363, 32, 1024, "ellipses", 10, 0.01, False),
    "cfg3": Config("cfg3", 512, 16, 360, 725, 90, 2048, "nested", 20, 0.005, False),
    "cfg4": Config("cfg4", 512, 64, 720, 725, 180, 2048, "ellipses", 20, 0.005, True),
    "cfg5": Config("cfg5", 1024, 1, 1024, 1449, 256, 4096, "ellipses", 40, 0.005, False),
}


def phantom_params(kind: str, K: int, seed: int, image: int) -> np.ndarray:
    """Ellipse table [K, 6] = (X0, Y0, a, b, phi, rho) in normalised coordinates
    X = u/(N/2), Y = v/(N/2).  Recipe: DESIGN.md §3 (SURVEY §8(d) "Synthetic inputs")."""
    rng = np.random.default_rng([seed, image, 4])
    out = np.zeros((K, 6))
    if kind == "ellipses":
        rad = 0.6 * np.sqrt(rng.random(K))
        ang = 2 * np.pi * rng.random(K)
        out[:, 0] = rad * np.cos(ang)
        out[:, 1] = rad * np.sin(ang)
        out[:, 2] = rng.uniform(0.05, 0.35, K)
        out[:, 3] = rng.uniform(0.05, 0.35, K)
        out[:, 4] = rng.uniform(0, np.pi, K)
        out[:, 5] = rng.random(K)
    elif kind == "nested":
        # Shepp-Logan-like: bright shell, darker body, then K-2 random interior features.
        out[0] = (0.0, 0.0, 0.69, 0.92, 0.0, 1.0)
        out[1] = (0.0, -0.0184, 0.6624, 0.874, 0.0, -0.8)
        k = K - 2
        rad = 0.5 * np.sqrt(rng.random(k))
        ang = 2 * np.pi * rng.random(k)
        out[2:, 0] = 0.55 * rad * np.cos(ang)
        out[2:, 1] = 0.8 * rad * np.sin(ang)
        out[2:, 2] = rng.uniform(0.03, 0.2, k)
        out[2:, 3] = rng.uniform(0.03, 0.2, k)
        out[2:, 4] = rng.uniform(0, np.pi, k)
        out[2:, 5] = rng.uniform(0.0, 0.3, k)
    elif kind == "disk":
        out = np.array([[0.0, 0.0, 1.0, 1.0, 0.0, 1.0]])
    else:
        raise ValueError(f"unknown phantom kind {kind!r}")
    return out


def _pixel_params(params: np.ndarray, N: int):
    half = N / 2.0
    for X0, Y0, a, b, phi, rho in params:
        yield X0 * half, Y0 * half, a * half, b * half, phi, rho


def rasterize(params: np.ndarray, N: int, ss: int = 4) -> np.ndarray:
    """Additive ellipse image [N, N] (fp64), ss×ss supersampled partial-volume inside tests."""
    img = np.zeros((N, N))
    h = (N - 1) / 2.0
    offs = (np.arange(ss) + 0.5) / ss - 0.5
    for u0, v0, A, Bq, phi, rho in _pixel_params(params, N):
        R = max(A, Bq) + 1.0
        c_lo = max(0, int(math.floor(u0 + h - R)))
        c_hi = min(N - 1, int(math.ceil(u0 + h + R)))
        r_lo = max(0, int(math.floor(h - v0 - R)))
        r_hi = min(N - 1, int(math.ceil(h - v0 + R)))
        if c_lo > c_hi or r_lo > r_hi:
            continue
        cs = np.arange(c_lo, c_hi + 1)
        rs = np.arange(r_lo, r_hi + 1)
        u = (cs[None, :, None, None] - h) + offs[None, None, None, :]
        v = (h - rs[:, None, None, None]) - offs[None, None, :, None]
        du, dv = u - u0, v - v0
        cph, sph = math.cos(phi), math.sin(phi)
        xp = du * cph + dv * sph
        yp = -du * sph + dv * cph
        inside = (xp / A) ** 2 + (yp / Bq) ** 2 <= 1.0
        img[r_lo:r_hi + 1, c_lo:c_hi + 1] += rho * inside.mean(axis=(2, 3))
    return img


def analytic_sinogram(params: np.ndarray, N: int, n_full: int, n_det: int) -> np.ndarray:
    """Continuous parallel-beam Radon transform of the additive ellipses, [n_full, n_det] fp64:
    p(θ, s) = Σ 2ρAB·sqrt(w² − (s−s0)²)/w², w² = A²cos²(θ−φ) + B²sin²(θ−φ)."""
    th = np.arange(n_full) * np.pi / n_full
    s = np.arange(n_det) - (n_det - 1) / 2.0
    out = np.zeros((n_full, n_det))
    for u0, v0, A, Bq, phi, rho in _pixel_params(params, N):
        w2 = (A * np.cos(th - phi)) ** 2 + (Bq * np.sin(th - phi)) ** 2
        s0 = u0 * np.cos(th) + v0 * np.sin(th)
        d2 = w2[:, None] - (s[None, :] - s0[:, None]) ** 2
        out += np.where(d2 > 0, 2 * rho * A * Bq * np.sqrt(np.maximum(d2, 0)) / w2[:, None], 0.0)
    return out


def _scale(params: np.ndarray, N: int, img: np.ndarray) -> float:
    mx = float(img.max()) if img.size else 0.0
    return 1.0 / mx if mx > 1.0 else 1.0


def make_phantoms(cfg: Config, seed: int = 0, images=None):
    """fp32 phantoms [len(images), N, N] in [0, 1] plus the per-image scale constants."""
    images = range(cfg.B) if images is None else images
    xs, scales, params = [], [], []
    for i in images:
        p = phantom_params(cfg.phantom, cfg.K, seed, i)
        img = rasterize(p, cfg.N)
        sc = _scale(p, cfg.N, img)
        xs.append(img * sc)
        scales.append(sc)
        params.append(p)
    return np.stack(xs).astype(np.float32), scales, params


def make_measurements(cfg: Config, params, scales, seed: int = 0, images=None):
    """y = analytic Radon(x†) + ε, σ_b = noise·max|y_clean,b| (BASELINE.json configs), fp32
    [len(images), n_full, n_det]."""
    images = range(cfg.B) if images is None else images
    ys = []
    for i, p, sc in zip(images, params, scales):
        yc = analytic_sinogram(p, cfg.N, cfg.n_full, cfg.n_det) * sc
        sigma = cfg.noise * float(np.abs(yc).max())
        rng = np.random.default_rng([seed, i, 3])
        ys.append(yc + sigma * rng.standard_normal(yc.shape))
    return np.stack(ys).astype(np.float32)


def make_workload(cfg: Config, seed: int = 0, images=None):
    """(x1, y): x1 = the phantom batch (the network output F_θ(z) of Alg. 1 step 3 is OUT
    of the hot path; the ideal network output x† stands in for it), y = measured data."""
    x, scales, params = make_phantoms(cfg, seed, images)
    y = make_measurements(cfg, params, scales, seed, images)
    return x, y


def rand_images(B: int, N: int, seed: int) -> np.ndarray:
    return np.random.default_rng([seed, 11]).standard_normal((B, N, N)).astype(np.float32)


def rand_sinograms(B: int, rows: int, n_det: int, seed: int) -> np.ndarray:
    return np.random.default_rng([seed, 12]).standard_normal((B, rows, n_det)).astype(np.float32)
