"""Pins of the fp64 oracle (oracle/oracle.c) against things other than itself.

Each test names what fixes the expected value: a published reference vector, a closed
form, an invariant of the mathematics, a special case that reduces to a library
routine (numpy / scipy), or brute force on tiny inputs.  Tolerances and the readings
they rest on are listed in DESIGN.md §4.  CPU only (no GPU marker).
"""
import math
import os

import numpy as np
import pytest
import scipy.ndimage as ndi
import scipy.stats as st

import oracle
import synth

SH = oracle.SHARED_IMAGE


# ----------------------------------------------------------------------------- draws
def test_splitmix64_reference_vector(golden_dir):
    """Published SplitMix64 outputs for seed 1234567 (golden fixture, cited in the file)."""
    vals = [int(l) for l in open(os.path.join(golden_dir, "splitmix64_seed1234567.txt"))
            if l.strip() and not l.startswith("#")]
    assert [oracle.word(1234567, i) for i in range(5)] == vals


# SURVEY §8(c) O-1 written out in plain Python integers (mod 2^64), independently of both C
# implementations (oracle/oracle.c and the library's csrc/sm64.h): the key chain, the
# multiply-high range reduction U(n) and the partial Fisher-Yates word order.
_M64 = (1 << 64) - 1
_GAMMA = 0x9E3779B97F4A7C15
_STREAM_ROT, _STREAM_SKETCH = 1, 2


def _o1_mix(z):
    z = (z + _GAMMA) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def _o1_key(seed, stream, it, image):
    return _o1_mix(_o1_mix(_o1_mix(_o1_mix(seed) ^ stream) ^ it) ^ image)


def _o1_word(key, i):
    return _o1_mix((key + i * _GAMMA) & _M64)


def _o1_u(w, n):
    return (w * n) >> 64  # floor(w n / 2^64)


def _o1_draw(seed, it, image, n_full, m, mode):
    kr = _o1_key(seed, _STREAM_ROT, it, image)
    g = 1 + _o1_u(_o1_word(kr, 0), 360)
    ks = _o1_key(seed, _STREAM_SKETCH, it, image)
    if mode == oracle.MODE_INTERLEAVED:
        step = n_full // m
        b = _o1_u(_o1_word(ks, 0), step)
        return g, [b + k * step for k in range(m)]
    perm = list(range(n_full))
    for i in range(m):
        j = i + _o1_u(_o1_word(ks, i), n_full - i)
        perm[i], perm[j] = perm[j], perm[i]
    return g, sorted(perm[:m])


def test_o1_mix_is_splitmix64_stream():
    """The i-th word of key k is the i-th output of a standard SplitMix64 generator seeded with
    k; the published vector (seed 1234567) pins the finaliser and the increment order."""
    vals = [int(l) for l in open(os.path.join(os.path.dirname(__file__), "golden",
                                              "splitmix64_seed1234567.txt"))
            if l.strip() and not l.startswith("#")]
    assert [_o1_word(1234567, i) for i in range(5)] == vals


@pytest.mark.parametrize("seed,it,image", [(0, 0, SH), (0, 1, SH), (0, 17, SH), (1, 0, 0),
                                           (7, 11, 3), (12345, 999, SH), (2**63 + 5, 2, 63),
                                           (0, 0, 0), (0, 0, 1), (3, 4, 2**32 + 1)])
@pytest.mark.parametrize("n_full,m", [(32, 8), (128, 32), (360, 90), (720, 180), (1024, 256),
                                      (12, 12), (5, 1)])
def test_o1_draw_rederived_in_python_integers(seed, it, image, n_full, m):
    """oracle.draw equals O-1 re-derived here in Python integers: the key chain
    mix(mix(mix(mix(seed) ^ stream) ^ iter) ^ image), U(n) = floor(w n / 2^64), g from word 0
    of ROT, the interleaved offset from word 0 of SKETCH and the Fisher-Yates target of step i
    from word i."""
    for mode in (oracle.MODE_UNIFORM, oracle.MODE_INTERLEAVED):
        if mode == oracle.MODE_INTERLEAVED and n_full % m:
            continue
        g, idx = oracle.draw(seed, it, image, n_full, m, mode)
        rg, ridx = _o1_draw(seed, it, image, n_full, m, mode)
        assert g == rg and list(idx) == ridx, (mode, g, rg)
    assert oracle.key(seed, _STREAM_SKETCH, it, image) == _o1_key(seed, _STREAM_SKETCH, it, image)


def test_interleave_rule_examples():
    """SPEC S:164 example (4 angles, 2 minibatches) -> [[0,2],[1,3]]
    'interleaved angles'; and the (100, 10) example S:165: batch i = {i, i+10, ..., i+90}."""
    seen = set()
    for it in range(200):
        g, idx = oracle.draw(7, it, SH, 4, 2, oracle.MODE_INTERLEAVED)
        assert tuple(idx) in {(0, 2), (1, 3)}
        assert 1 <= g <= 360
        seen.add(tuple(idx))
    assert seen == {(0, 2), (1, 3)}
    for it in range(50):
        _, idx = oracle.draw(3, it, SH, 100, 10, oracle.MODE_INTERLEAVED)
        b = idx[0]
        assert list(idx) == [b + 10 * k for k in range(10)] and 0 <= b < 10


def test_draw_config_errors():
    with pytest.raises(ValueError):
        oracle.draw(0, 0, SH, 10, 11)
    with pytest.raises(ValueError):
        oracle.draw(0, 0, SH, 10, 3, oracle.MODE_INTERLEAVED)  # 3 does not divide 10


def test_uniform_subset_properties_and_uniformity():
    """Uniform m-subset: ascending, distinct, in range; each index included with
    probability m/n_full (chi-square at alpha = 0.01); m = n_full gives all angles."""
    n_full, m, T = 36, 9, 4000
    counts = np.zeros(n_full)
    for it in range(T):
        _, idx = oracle.draw(11, it, SH, n_full, m)
        assert np.all(np.diff(idx) > 0) and idx[0] >= 0 and idx[-1] < n_full
        counts[idx] += 1
    exp = T * m / n_full
    chi = ((counts - exp) ** 2 / exp).sum()
    assert chi < st.chi2.ppf(0.99, n_full - 1)
    _, idx = oracle.draw(5, 1, SH, 32, 32)
    assert list(idx) == list(range(32))


def test_rotation_draw_chi_square():
    """1e5 draws of g from |G| = 360 pass chi-square at alpha = 0.01; g in 1..360."""
    T = 100_000
    gs = np.array([oracle.draw(2024, it, SH, 4, 1)[0] for it in range(T)])
    assert gs.min() >= 1 and gs.max() <= 360
    counts = np.bincount(gs - 1, minlength=360)
    exp = T / 360
    assert ((counts - exp) ** 2 / exp).sum() < st.chi2.ppf(0.99, 359)


def test_draw_streams_independent_per_image_and_iter():
    a = oracle.draw(0, 0, 0, 720, 180)
    b = oracle.draw(0, 0, 1, 720, 180)
    c = oracle.draw(0, 1, 0, 720, 180)
    assert not np.array_equal(a[1], b[1]) and not np.array_equal(a[1], c[1])
    assert np.array_equal(a[1], oracle.draw(0, 0, 0, 720, 180)[1])


# -------------------------------------------------------------------------- rotation
def test_rotation_identity_and_quarter_turns_exact():
    """g = 360 is the identity; g = 90/180/270 are exact index
    permutations equal to numpy.rot90 (counter-clockwise content rotation)."""
    x = synth.rand_images(1, 33, 1)[0].astype(np.float64)
    assert np.array_equal(oracle.rotate(x, 360), x)
    for g, k in ((90, 1), (180, 2), (270, 3)):
        assert np.array_equal(oracle.rotate(x, g), np.rot90(x, k))
    y = synth.rand_images(1, 32, 2)[0].astype(np.float64)
    assert np.array_equal(oracle.rotate(y, 90), np.rot90(y, 1))


@pytest.mark.parametrize("g", [1, 37, 123, 200, 301, 359])
def test_rotation_equals_scipy_bilinear(g):
    """Bilinear interpolation with zero padding reduces to scipy.ndimage.map_coordinates
    (order=1, mode='grid-constant'); the sample positions are those of the centre
    rotation (u, v) -> (u cos g + v sin g, -u sin g + v cos g)."""
    N = 40
    x = synth.rand_images(1, N, g)[0].astype(np.float64)
    h = (N - 1) / 2
    r, c = np.meshgrid(np.arange(N), np.arange(N), indexing="ij")
    u, v = c - h, h - r
    cg, sg = math.cos(math.radians(g)), math.sin(math.radians(g))
    us, vs = u * cg + v * sg, -u * sg + v * cg
    ref = ndi.map_coordinates(x, [h - vs, us + h], order=1, mode="grid-constant", cval=0.0)
    assert np.max(np.abs(oracle.rotate(x, g) - ref)) < 1e-12


def test_rotation_round_trip_psnr():
    """g = 37 then g = 323 recovers a smooth disk-masked image to >= 40 dB."""
    N = 128
    h = (N - 1) / 2
    r, c = np.meshgrid(np.arange(N), np.arange(N), indexing="ij")
    u, v = c - h, h - r
    img = np.exp(-((u - 10) ** 2 + (v + 5) ** 2) / (2 * 15 ** 2)) + 0.5 * np.exp(
        -((u + 20) ** 2 + (v - 12) ** 2) / (2 * 9 ** 2))
    mask = u ** 2 + v ** 2 <= (0.4 * N) ** 2
    back = oracle.rotate(oracle.rotate(img, 37), 323)
    mse = np.mean((back - img)[mask] ** 2)
    assert 10 * np.log10(img.max() ** 2 / mse) >= 40


# --------------------------------------------------------------------------- forward
def _dense_A(N, n_det, n_full, idx):
    """Brute-force dense matrix from the north_star formula, entry by entry (broadcast)."""
    h, hd = (N - 1) / 2, (n_det - 1) / 2
    th = np.asarray(idx) * np.pi / n_full
    k, j, r, c = np.meshgrid(np.arange(len(idx)), np.arange(n_det), np.arange(N),
                             np.arange(N), indexing="ij")
    t = (c - h) * np.cos(th[k]) + (h - r) * np.sin(th[k])
    s = j - hd
    return np.maximum(0.0, 1.0 - np.abs(t - s)).reshape(len(idx) * n_det, N * N)


def test_dense_8x8_forward_and_adjoint():
    """Brute force on 8x8 (n_det = 12, all 8 angles): A x and A^T y from the dense matrix."""
    N, n_det, n_full = 8, 12, 8
    idx = np.arange(n_full)
    A = _dense_A(N, n_det, n_full, idx)
    rng = np.random.default_rng(0)
    x = rng.standard_normal((N, N))
    y = rng.standard_normal((n_full, n_det))
    assert np.max(np.abs(oracle.fwd(x, idx, n_full, n_det).ravel() - A @ x.ravel())) < 1e-13
    assert np.max(np.abs(oracle.adj(y, idx, n_full, N).ravel() - A.T @ y.ravel())) < 1e-13


def test_forward_mass_conservation():
    """Hats form a partition of unity and every pixel projects inside the detector
    (n_det = ceil(N sqrt 2)): sum_j p[k][j] = sum x at every angle."""
    cfg = synth.CONFIGS["cfg1"]
    x = synth.rand_images(1, cfg.N, 5)[0].astype(np.float64)
    p = oracle.fwd(x, np.arange(cfg.n_full), cfg.n_full, cfg.n_det)
    assert np.max(np.abs(p.sum(axis=1) - x.sum())) <= 1e-12 * np.abs(x).sum()
    e = np.zeros((cfg.N, cfg.N))
    e[31, 40] = 1.0
    pe = oracle.fwd(e, np.arange(cfg.n_full), cfg.n_full, cfg.n_det)
    assert np.allclose(pe.sum(axis=1), 1.0, atol=1e-15)
    assert np.all(oracle.fwd(np.zeros((16, 16)), [0, 3], 8, 23) == 0)


def _hat_smoothed_disk(s, r):
    """Analytic projection of a radius-r unit disk, 2 sqrt(r^2 - s^2), convolved with the
    unit hat (what an ideal line integral through a linear-interpolating detector gives)."""
    off = np.linspace(-1, 1, 257)
    w = 1 - np.abs(off)
    vals = 2 * np.sqrt(np.maximum(r ** 2 - (s[:, None] + off[None, :]) ** 2, 0))
    return np.trapezoid(vals * w, off, axis=1)


def test_forward_closed_form_disk():
    """Closed-form disk projection (north_star pin).  Pixel-driven aliasing at exactly
    45/135 degrees is a property of the discretisation, hence the
    angle-aware bounds: median rel-L2 <= 0.5%, every angle off 45+-1/135+-1 <= 2%,
    45/135 <= 10%."""
    N, n_full, n_det, rad = 256, 360, 363, 60.0
    params = np.array([[0, 0, rad / (N / 2), rad / (N / 2), 0, 1.0]])
    x = synth.rasterize(params, N, ss=8)
    p = oracle.fwd(x, np.arange(n_full), n_full, n_det)
    s = np.arange(n_det) - (n_det - 1) / 2
    ref = _hat_smoothed_disk(s, rad)
    err = np.linalg.norm(p - ref[None, :], axis=1) / np.linalg.norm(ref)
    deg = np.arange(n_full) * 180 / n_full
    diag = (np.abs(deg - 45) <= 1) | (np.abs(deg - 135) <= 1)
    assert np.median(err) <= 5e-3
    assert err[~diag].max() <= 2e-2
    assert err[diag].max() <= 1e-1


def test_forward_rotation_commutation():
    """A_th(T_90 x) = A_{th-90} x (wrapping th-90 < 0 to th+90 with s -> -s) and
    A_th(T_180 x) = flip_s A_th x.  Pins the joint orientation of
    the rotation and the projector; a flipped convention fails at O(0.1)."""
    N, n_full, n_det = 48, 32, 69
    x = synth.rand_images(1, N, 9)[0].astype(np.float64)
    idx = np.arange(n_full)
    p = oracle.fwd(x, idx, n_full, n_det)
    p90 = oracle.fwd(oracle.rotate(x, 90), idx, n_full, n_det)
    p180 = oracle.fwd(oracle.rotate(x, 180), idx, n_full, n_det)
    half = n_full // 2
    scale = np.abs(p).max()
    for i in range(n_full):
        ref = p[i - half] if i >= half else p[i + half][::-1]
        assert np.max(np.abs(p90[i] - ref)) <= 1e-12 * scale
        assert np.max(np.abs(p180[i] - p[i][::-1])) <= 1e-12 * scale


# --------------------------------------------------------------------------- adjoint
def test_adjoint_identity_and_negative_control():
    """<A x, y> = <x, A^T y> to 1e-10 relative (north_star); a deliberately wrong
    adjoint (angles reflected th -> pi - th) gives a defect >= 0.1 on y = A x."""
    cfg = synth.CONFIGS["cfg1"]
    rng = np.random.default_rng(3)
    idx = np.sort(rng.choice(cfg.n_full, 12, replace=False))
    for trial in range(5):
        x = rng.standard_normal((cfg.N, cfg.N))
        y = rng.standard_normal((12, cfg.n_det))
        Ax = oracle.fwd(x, idx, cfg.n_full, cfg.n_det)
        lhs = float((Ax * y).sum())
        rhs = float((x * oracle.adj(y, idx, cfg.n_full, cfg.N)).sum())
        denom = np.linalg.norm(Ax) * np.linalg.norm(y)
        assert abs(lhs - rhs) / denom <= 1e-10
        # negative control on a correlated pair (y = A x), where <Ax, y> = ||Ax||^2
        wrong = oracle.adj(Ax, (cfg.n_full - idx) % cfg.n_full, cfg.n_full, cfg.N)
        defect = abs(float((Ax * Ax).sum()) - float((x * wrong).sum())) / np.linalg.norm(Ax) ** 2
        assert defect >= 0.1


# ------------------------------------------------------------------------------ ramp
def test_ramp_impulse_response():
    """Impulse response = the Ram-Lak (Kak-Slaney) kernel doubled: 1/2 at 0, 0 at even
    offsets, -2/(pi^2 n^2) at odd n; rows are independent; linear."""
    n_det = 31
    p = np.zeros((2, n_det))
    p[0, 15] = 1.0
    q = oracle.ramp(p)
    ref = np.zeros(n_det)
    for j in range(n_det):
        n = j - 15
        ref[j] = 0.5 if n == 0 else (0.0 if n % 2 == 0 else -2.0 / (math.pi ** 2 * n * n))
    assert np.max(np.abs(q[0] - ref)) < 1e-15
    assert np.all(q[1] == 0)


@pytest.mark.parametrize("f", [0.05, 0.125, 0.25, 0.37])
def test_ramp_frequency_response_is_2f(f):
    """sum_{odd n>=1} cos(n x)/n^2 = (pi/4)(pi/2 - |x|) gives an infinite-length response
    of exactly 2|f| on |f| <= 1/2.  At the centre of a long row the truncated tails cost
    <= sum_{|n|>L} 2/(pi^2 n^2) ~ 2/(pi^2 L)."""
    n_det = 4001
    j = np.arange(n_det)
    p = np.cos(2 * np.pi * f * (j - 2000))[None, :]
    q = oracle.ramp(p)[0]
    assert abs(q[2000] - 2 * f) <= 2 * 2 / (np.pi ** 2 * 2000)


def test_ramp_equals_zero_padded_fft_when_long_enough():
    """App. A.1: with P >= 2 n_det - 1 the P-point circular convolution with the wrapped
    kernel equals the linear convolution (the identity the GPU's FFT path relies on);
    with P too short it does not."""
    rng = np.random.default_rng(4)
    for n_det, P in ((91, 256), (363, 1024), (363, 2048)):
        p = rng.standard_normal((3, n_det))
        idx = np.arange(P)
        lag = np.where(idx <= P // 2, idx, idx - P)
        hP = np.where(lag == 0, 0.5, np.where(lag % 2 == 0, 0.0, -2 / (np.pi ** 2 * np.maximum(np.abs(lag), 1) ** 2)))
        R = np.fft.fft(hP).real
        qf = np.fft.ifft(np.fft.fft(p, P, axis=1) * R[None, :], axis=1).real[:, :n_det]
        assert np.max(np.abs(qf - oracle.ramp(p))) < 1e-13
        if P == 1024:
            R2 = np.fft.fft(hP[np.r_[0:256, P - 256:P]]).real  # 512 points < 2*363-1
            q2 = np.fft.ifft(np.fft.fft(p, 512, axis=1) * R2[None, :], axis=1).real[:, :n_det]
            assert np.max(np.abs(q2 - oracle.ramp(p))) > 1e-6


# ------------------------------------------------------------------------------- FBP
def _disk_interior(N, rad, margin):
    h = (N - 1) / 2
    r, c = np.meshgrid(np.arange(N), np.arange(N), indexing="ij")
    return (c - h) ** 2 + (h - r) ** 2 <= (rad - margin) ** 2


def _psnr(a, ref, peak=1.0):
    return 10 * np.log10(peak ** 2 / np.mean((a - ref) ** 2))


def test_fbp_of_analytic_disk_sinogram():
    """FBP recovery of a disk phantom (north_star pin), independent of projector aliasing:
    the analytic sinogram 2 sqrt(r^2 - s^2) (seen through the unit-hat detector response)
    through ramp + backprojection with the
    pi/(2m) scale: interior max|err| <= 0.01, PSNR >= 33 dB."""
    N, n_full, n_det, rad = 256, 128, 363, 80.0
    params = np.array([[0, 0, rad / (N / 2), rad / (N / 2), 0, 1.0]])
    s = np.arange(n_det) - (n_det - 1) / 2
    sino = np.tile(_hat_smoothed_disk(s, rad), (n_full, 1))
    rec = oracle.fbp(sino, np.arange(n_full), n_full, N)
    truth = synth.rasterize(params, N, ss=8)
    inner = _disk_interior(N, rad, 4)
    assert np.max(np.abs(rec - truth)[inner]) <= 0.01
    assert _psnr(rec, truth) >= 33


def test_fbp_of_discrete_projection_of_disk():
    """Full discrete operator: FBP(A x_disk).  Without the aliased 45/135 degree views:
    PSNR >= 28 dB and interior mean within 1%; with all views interior mean within 2%."""
    N, n_full, n_det, rad = 256, 128, 363, 80.0
    params = np.array([[0, 0, rad / (N / 2), rad / (N / 2), 0, 1.0]])
    truth = synth.rasterize(params, N, ss=8)
    inner = _disk_interior(N, rad, 4)
    allv = np.arange(n_full)
    no_diag = allv[(allv != 32) & (allv != 96)]
    for views, check_psnr, tol in ((no_diag, True, 0.01), (allv, False, 0.02)):
        rec = oracle.fbp(oracle.fwd(truth, views, n_full, n_det), views, n_full, N)
        assert abs(rec[inner].mean() - 1.0) <= tol
        if check_psnr:
            assert _psnr(rec, truth) >= 28


# ------------------------------------------------------------------ residuals / grad
def test_partition_identity_and_zero_ei():
    """||Ax - y||^2 = sum_i ||S_i A x - S_i y||^2 over the interleaved
    minibatches; x2 = x3 gives ei = 0 exactly."""
    cfg = synth.CONFIGS["cfg1"]
    rng = np.random.default_rng(8)
    x = rng.standard_normal((cfg.N, cfg.N))
    y = rng.standard_normal((cfg.n_full, cfg.n_det))
    full = np.arange(cfg.n_full)
    mc_full, ei, _ = oracle.residual(oracle.fwd(x, full, cfg.n_full, cfg.n_det), y, full, x, x)
    assert ei == 0.0
    nb = cfg.n_full // cfg.m
    tot = 0.0
    for b in range(nb):
        S = np.arange(b, cfg.n_full, nb)
        tot += oracle.residual(oracle.fwd(x, S, cfg.n_full, cfg.n_det), y, S, x, x)[0]
    assert abs(tot - mc_full) <= 1e-12 * mc_full


def test_mc_expectation_under_noise():
    """x1 = x_true, y = A x_true + N(0, s^2): E[mc] = m n_det s^2 (within 4 sd)."""
    N, n_full, n_det, m, sig = 64, 32, 91, 32, 0.3
    rng = np.random.default_rng(12)
    x = rng.random((N, N))
    full = np.arange(n_full)
    y = oracle.fwd(x, full, n_full, n_det) + sig * rng.standard_normal((n_full, n_det))
    mc, _, _ = oracle.residual(oracle.fwd(x, full, n_full, n_det), y, full, x, x)
    ratio = mc / (m * n_det * sig ** 2)
    assert abs(ratio - 1) <= 4 * math.sqrt(2 / (m * n_det))


def test_mc_gradient_finite_difference():
    """d/dx1 ||A_S x1 - y_S||^2 = 2 A_S^T r; mc is quadratic so central differences are
    exact up to rounding."""
    N, n_full, n_det = 12, 16, 17
    idx = np.array([0, 3, 5, 8, 13])
    rng = np.random.default_rng(6)
    x = rng.standard_normal((N, N))
    y = rng.standard_normal((n_full, n_det))
    out = oracle.sketched_pass(x, y, 37, idx, n_full)

    def mc(z):
        return oracle.residual(oracle.fwd(z, idx, n_full, n_det), y, idx, z, z)[0]

    eps = 1e-3
    for (r, c) in ((0, 0), (5, 7), (11, 3), (6, 6)):
        e = np.zeros((N, N))
        e[r, c] = eps
        fd = (mc(x + e) - mc(x - e)) / (2 * eps)
        assert abs(fd - out["grad"][r, c]) <= 1e-8 * max(1.0, abs(fd))


# ------------------------------------------------------------------------ whole pass
def test_whole_pass_dense_8x8():
    """Brute force: compose dense T_g (scipy bilinear applied to basis images), dense A_S
    (formula), dense H2 (Toeplitz of the closed-form kernel) and A_S^T; compare every
    output of oracle_pass (SPEC S:441 'unrolled x1, x2, x3 oracle on 8x8')."""
    N, n_det, n_full, g = 8, 12, 8, 37
    idx = np.array([1, 2, 5, 7])
    m = len(idx)
    h = (N - 1) / 2
    r, c = np.meshgrid(np.arange(N), np.arange(N), indexing="ij")
    u, v = c - h, h - r
    cg, sg = math.cos(math.radians(g)), math.sin(math.radians(g))
    coords = [h - (-u * sg + v * cg), u * cg + v * sg + h]
    T = np.stack([ndi.map_coordinates(np.eye(N * N)[i].reshape(N, N), coords, order=1,
                                      mode="grid-constant").ravel() for i in range(N * N)], 1)
    A = _dense_A(N, n_det, n_full, idx)
    lag = np.arange(n_det)[:, None] - np.arange(n_det)[None, :]
    H = np.where(lag == 0, 0.5, np.where(lag % 2 == 0, 0.0,
                                         -2 / (np.pi ** 2 * np.maximum(np.abs(lag), 1) ** 2)))
    Hb = np.kron(np.eye(m), H)
    rng = np.random.default_rng(1)
    x1 = rng.standard_normal(N * N)
    y = rng.standard_normal((n_full, n_det))
    yS = y[idx].ravel()
    x2 = T @ x1
    p2 = A @ x2
    q = Hb @ p2
    xf = (np.pi / (2 * m)) * A.T @ q
    p1 = A @ x1
    rr = p1 - yS
    out = oracle.sketched_pass(x1.reshape(N, N), y, g, idx, n_full)
    for name, ref in (("x2", x2), ("p2", p2), ("q", q), ("xfbp", xf), ("p1", p1), ("r", rr),
                      ("grad", 2 * A.T @ rr)):
        assert np.max(np.abs(out[name].ravel() - ref)) < 1e-12, name
    assert abs(out["mc"] - rr @ rr) < 1e-12 * (rr @ rr)
    assert abs(out["ei"] - np.sum((x2 - xf) ** 2)) < 1e-12 * np.sum((x2 - xf) ** 2)


# ------------------------------------------------- EI-branch backward
def _dense_T(N, g):
    """Dense bilinear rotation from scipy (map_coordinates, order 1, zeros outside) applied
    to the basis images — independent of oracle_rotate."""
    h = (N - 1) / 2
    r, c = np.meshgrid(np.arange(N), np.arange(N), indexing="ij")
    u, v = c - h, h - r
    cg, sg = math.cos(math.radians(g)), math.sin(math.radians(g))
    coords = [h - (-u * sg + v * cg), u * cg + v * sg + h]
    return np.stack([ndi.map_coordinates(np.eye(N * N)[i].reshape(N, N), coords, order=1,
                                         mode="grid-constant").ravel() for i in range(N * N)], 1)


@pytest.mark.parametrize("g", [37, 123, 211, 300])
def test_rotation_transpose_dense_8x8(g):
    """T_g^T: oracle_rotate_adj applied to every basis image equals the transpose of the
    dense scipy rotation matrix (brute force)."""
    N = 8
    T = _dense_T(N, g)
    TT = np.stack([oracle.rotate_adj(np.eye(N * N)[i].reshape(N, N), g).ravel()
                   for i in range(N * N)], 1)
    assert np.max(np.abs(TT - T.T)) < 1e-14


@pytest.mark.parametrize("g", [1, 45, 89, 137, 359])
def test_rotation_transpose_adjoint_identity(g):
    """<T_g x, y> = <x, T_g^T y> for random x, y (33 x 33, odd size: the centre is a pixel)."""
    rng = np.random.default_rng(g)
    x, y = rng.standard_normal((33, 33)), rng.standard_normal((33, 33))
    lhs = float(np.sum(oracle.rotate(x, g) * y))
    rhs = float(np.sum(x * oracle.rotate_adj(y, g)))
    assert abs(lhs - rhs) <= 1e-12 * np.linalg.norm(x) * np.linalg.norm(y)


def test_rotation_transpose_quarter_turns_exact():
    """The quarter turns are permutations, so their transposes are the inverse turns:
    T_360^T = I, T_90^T = numpy rot90(., -1), T_180^T = rot90(., 2), T_270^T = rot90(., 1)."""
    y = np.random.default_rng(3).standard_normal((16, 16))
    assert np.array_equal(oracle.rotate_adj(y, 360), y)
    assert np.array_equal(oracle.rotate_adj(y, 90), np.rot90(y, -1))
    assert np.array_equal(oracle.rotate_adj(y, 180), np.rot90(y, 2))
    assert np.array_equal(oracle.rotate_adj(y, 270), np.rot90(y, 1))


def test_ei_gradient_dense_8x8():
    """grad_x1 ||x2 - x3||^2 with x2 = T x1, x3 = M x2, M = (pi/2m) A^T H2 A, from dense
    matrices: 2 T^T (I - M)^T (I - M) T x1 (scipy rotation, formula A, closed-form H2)."""
    N, n_det, n_full, g = 8, 12, 8, 37
    idx = np.array([1, 2, 5, 7])
    m = len(idx)
    T = _dense_T(N, g)
    A = _dense_A(N, n_det, n_full, idx)
    lag = np.arange(n_det)[:, None] - np.arange(n_det)[None, :]
    H = np.where(lag == 0, 0.5, np.where(lag % 2 == 0, 0.0,
                                         -2 / (np.pi ** 2 * np.maximum(np.abs(lag), 1) ** 2)))
    M = (np.pi / (2 * m)) * A.T @ np.kron(np.eye(m), H) @ A
    x1 = np.random.default_rng(9).standard_normal(N * N)
    I = np.eye(N * N)
    ref = 2 * T.T @ (I - M).T @ (I - M) @ T @ x1
    got = oracle.ei_grad(x1.reshape(N, N), g, idx, n_full, n_det).ravel()
    assert np.max(np.abs(got - ref)) < 1e-12 * max(1.0, np.max(np.abs(ref)))
    assert np.max(np.abs(M - M.T)) < 1e-14  # the sketched FBP-of-projection is symmetric


def test_ei_gradient_finite_difference():
    """d/dx1 ei with ei from oracle_pass (identity network); ei is quadratic in x1, so
    central differences are exact up to rounding."""
    N, n_full, n_det, g = 12, 16, 17, 73
    idx = np.array([0, 3, 5, 8, 13])
    rng = np.random.default_rng(8)
    x = rng.standard_normal((N, N))
    y = rng.standard_normal((n_full, n_det))
    grad = oracle.ei_grad(x, g, idx, n_full, n_det)

    def ei(z):
        return oracle.sketched_pass(z, y, g, idx, n_full)["ei"]

    eps = 1e-3
    for (r, c) in ((0, 0), (5, 7), (11, 3), (6, 6), (2, 9)):
        e = np.zeros((N, N))
        e[r, c] = eps
        fd = (ei(x + e) - ei(x - e)) / (2 * eps)
        assert abs(fd - grad[r, c]) <= 1e-8 * max(1.0, abs(fd))


# --------------------------------------------------------- REI variant
def test_rei_noise_standard_normal_and_independent():
    """The simulated noise is N(0, 1) (Kolmogorov-Smirnov, 2e5 samples) and differs between
    images and iterations (near-zero correlation)."""
    e = oracle.rei_noise(0, 1, 7, 200, 1000).ravel()
    assert st.kstest(e, "norm").pvalue > 0.01
    f = oracle.rei_noise(0, 1, 8, 200, 1000).ravel()
    h = oracle.rei_noise(0, 2, 7, 200, 1000).ravel()
    assert abs(np.corrcoef(e, f)[0, 1]) < 0.01 and abs(np.corrcoef(e, h)[0, 1]) < 0.01


def test_rei_sigma_zero_is_the_plain_pass():
    cfg = synth.CONFIGS["cfg1"]
    x1, y = synth.make_workload(cfg, seed=0)
    g, idx = oracle.draw(0, 0, SH, cfg.n_full, cfg.m)
    a = oracle.sketched_pass(x1[0], y[0], g, idx, cfg.n_full)
    b = oracle.sketched_pass_rei(x1[0], y[0], g, idx, cfg.n_full, 0.0, 0, 0, 0)
    for k in ("x2", "p1", "p2", "q", "xfbp", "r", "grad"):
        assert np.array_equal(a[k], b[k]), k
    assert a["mc"] == b["mc"] and a["ei"] == b["ei"]


def test_rei_dense_8x8():
    """x3_rei = x3 + (pi/2m) A^T H2 (sigma eps) from dense matrices (formula A, closed-form
    H2) with eps = rei_noise (pinned above)."""
    N, n_det, n_full, g, sigma = 8, 12, 8, 37, 0.3
    idx = np.array([1, 2, 5, 7])
    m = len(idx)
    A = _dense_A(N, n_det, n_full, idx)
    lag = np.arange(n_det)[:, None] - np.arange(n_det)[None, :]
    H = np.where(lag == 0, 0.5, np.where(lag % 2 == 0, 0.0,
                                         -2 / (np.pi ** 2 * np.maximum(np.abs(lag), 1) ** 2)))
    Ap = (np.pi / (2 * m)) * A.T @ np.kron(np.eye(m), H)
    rng = np.random.default_rng(4)
    x1 = rng.standard_normal((N, N))
    y = rng.standard_normal((n_full, n_det))
    plain = oracle.sketched_pass(x1, y, g, idx, n_full)
    rei = oracle.sketched_pass_rei(x1, y, g, idx, n_full, sigma, 3, 4, 5)
    eps = oracle.rei_noise(3, 4, 5, m, n_det).ravel()
    ref = plain["xfbp"].ravel() + Ap @ (sigma * eps)
    assert np.max(np.abs(rei["xfbp"].ravel() - ref)) < 1e-12
    assert np.array_equal(rei["p2"], plain["p2"])  # p2 is reported noise-free


def test_rei_monte_carlo_noise_inflation():
    """E ||x3_rei - x3||^2 = sigma^2 ||A_S^+||_F^2 (dense A_S^+ on 8x8); the
    Monte-Carlo mean over 400 noise draws lies within 4 standard errors."""
    N, n_det, n_full, g, sigma = 8, 12, 8, 37, 0.5
    idx = np.array([0, 3, 4, 6])
    m = len(idx)
    A = _dense_A(N, n_det, n_full, idx)
    lag = np.arange(n_det)[:, None] - np.arange(n_det)[None, :]
    H = np.where(lag == 0, 0.5, np.where(lag % 2 == 0, 0.0,
                                         -2 / (np.pi ** 2 * np.maximum(np.abs(lag), 1) ** 2)))
    Ap = (np.pi / (2 * m)) * A.T @ np.kron(np.eye(m), H)
    expect = sigma ** 2 * float(np.sum(Ap ** 2))
    rng = np.random.default_rng(5)
    x1 = rng.standard_normal((N, N))
    y = rng.standard_normal((n_full, n_det))
    plain = oracle.sketched_pass(x1, y, g, idx, n_full)["xfbp"]
    d = np.array([np.sum((oracle.sketched_pass_rei(x1, y, g, idx, n_full, sigma, 0, it, 0)["xfbp"]
                          - plain) ** 2) for it in range(400)])
    assert abs(d.mean() - expect) <= 4 * d.std(ddof=1) / np.sqrt(len(d))


# ------------------------------------------- Theorem-1 deviation
def test_sketch_deviation_equals_dense_spectral_norm():
    """Power iteration of D = (n_full/m) A_S^T A_S - A^T A (oracle) vs numpy's spectral norm
    of the dense D built from the formula matrix (8x8, n_full = 8, m = 4)."""
    N, n_det, n_full = 8, 12, 8
    idx = np.array([1, 2, 5, 7])
    A = _dense_A(N, n_det, n_full, np.arange(n_full))
    AS = _dense_A(N, n_det, n_full, idx)
    D = (n_full / len(idx)) * AS.T @ AS - A.T @ A
    ref = np.linalg.norm(D, 2)
    lam, v = oracle.sketch_deviation(np.random.default_rng(2).standard_normal((N, N)), idx,
                                     n_full, n_det, 3000)
    assert abs(lam - ref) <= 1e-6 * ref
    # the iterate is an eigenvector of D for an eigenvalue of modulus ||D||
    Dv = D @ v.ravel()
    assert abs(np.linalg.norm(Dv) - ref) <= 1e-6 * ref


def test_sketch_deviation_full_sketch_is_zero():
    """m = n_full: S^T S = I, so the deviation vanishes exactly (SURVEY §8(c) sketch reduction)."""
    N, n_det, n_full = 8, 12, 8
    lam, _ = oracle.sketch_deviation(np.ones((N, N)), np.arange(n_full), n_full, n_det, 5)
    assert lam < 1e-10
