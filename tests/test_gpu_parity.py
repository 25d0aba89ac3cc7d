"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle, element by element.

Bar (BASELINE.json north_star): max|gpu - ref| <= 1e-4 * max|ref| for every output tensor
(sinograms, filtered sinograms, images, residuals, gradients), scalars within 1e-4
relative, integer draws bit-identical.  Inputs are seeded synthetic workloads (synth/).
"""
import math

import numpy as np
import pytest
import torch

import oracle
import paper_2411_05771_b200 as sk
import synth

pytestmark = pytest.mark.gpu
TOL = 1e-4
SH = sk.SHARED_IMAGE


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)


def close(gpu, ref, name, tol=TOL):
    g = gpu.detach().double().cpu().numpy() if torch.is_tensor(gpu) else np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64)
    assert g.shape == ref.shape, (name, g.shape, ref.shape)
    scale = float(np.abs(ref).max())
    err = float(np.abs(g - ref).max())
    assert err <= tol * scale + 1e-30, f"{name}: max|err| {err:.3e} > {tol:g} * max|ref| {scale:.3e}"
    return err / max(scale, 1e-300)


def dev(a, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dtype)


def idx_t(idx):
    return dev(np.asarray(idx, np.int32), torch.int32)


# ------------------------------------------------------------------------------ draws
@pytest.mark.parametrize("name", list(synth.CONFIGS))
@pytest.mark.parametrize("mode", [sk.MODE_UNIFORM, sk.MODE_INTERLEAVED])
def test_device_draws_bit_identical(name, mode):
    cfg = synth.CONFIGS[name]
    for it in (0, 1, 17):
        g, idx = sk.draw_device(0, it, 0, 1, True, cfg.n_full, cfg.m, mode)
        og, oidx = oracle.draw(0, it, SH, cfg.n_full, cfg.m, mode)
        assert int(g[0]) == og and np.array_equal(idx[0].cpu().numpy(), oidx)
        g, idx = sk.draw_device(0, it, 0, cfg.B, False, cfg.n_full, cfg.m, mode)
        for b in range(cfg.B):
            og, oidx = oracle.draw(0, it, b, cfg.n_full, cfg.m, mode)
            assert int(g[b]) == og and np.array_equal(idx[b].cpu().numpy(), oidx)


# --------------------------------------------------------------------- stage parity
GEOMS = [  # (N, n_det, n_full, fft_len, B, m)
    (64, 91, 32, 256, 2, 8),       # cfg1
    (256, 363, 128, 1024, 8, 32),  # cfg2
    (50, 71, 20, 0, 3, 5),         # ragged tile, odd batch (BB = 1)
    (40, 57, 12, 0, 4, 12),        # m = n_full (full EI), BB = 4
    (33, 47, 9, 0, 2, 1),          # odd N, single angle
    (64, 40, 16, 0, 6, 4),         # truncated even detector (corner pixels' taps dropped, R18), BB = 2
    (48, 200, 24, 0, 4, 6),        # detector far wider than the image (idle chunks)
    (16, 1, 8, 0, 1, 3),           # a single detector bin
]


def _plan(N, n_det, n_full, P):
    return sk.Plan.get(N, n_det, n_full, P)


@pytest.mark.parametrize("geom", GEOMS)
def test_rotate_parity(geom):
    N, n_det, n_full, P, B, m = geom
    plan = _plan(N, n_det, n_full, P)
    x = synth.rand_images(B, N, 1)
    for g in (1, 37, 90, 123, 180, 270, 301, 360):
        out = sk.rotate(plan, dev(x), idx_t([g]))
        ref = oracle.rotate(x, g)
        if g % 90 == 0:
            assert np.array_equal(out.cpu().numpy(), np.rot90(x, g // 90, axes=(1, 2)))
        close(out, ref, f"rotate g={g}")
    gs = [(17 * b + 5) % 360 + 1 for b in range(B)]  # per-image g
    out = sk.rotate(plan, dev(x), idx_t(gs))
    for b in range(B):
        close(out[b], oracle.rotate(x[b], gs[b]), f"rotate per-image b={b}")


def _draw_list(n_full, m, seed=3):
    return oracle.draw(seed, 0, SH, n_full, m)[1]


@pytest.mark.parametrize("geom", GEOMS)
def test_radon_fwd_parity(geom):
    N, n_det, n_full, P, B, m = geom
    plan = _plan(N, n_det, n_full, P)
    x = synth.rand_images(B, N, 2)
    idx = _draw_list(n_full, m)
    p = sk.radon_fwd(plan, dev(x), idx_t(idx))
    close(p, oracle.fwd(x, idx, n_full, n_det), "fwd")
    # per-image sketches
    idxs = np.stack([oracle.draw(5, 0, b, n_full, m)[1] for b in range(B)])
    p = sk.radon_fwd(plan, dev(x), idx_t(idxs))
    for b in range(B):
        close(p[b], oracle.fwd(x[b], idxs[b], n_full, n_det), f"fwd per-image b={b}")


def test_radon_fwd_small_problem_units_both_sides_of_the_rule():
    """The forward runs small launches (fewer than 8 line blocks per CTA) with at most 3
    angles per unit and larger ones with the largest K (radon_fwd.cu, launch_bb).  Same
    geometry (cfg2's: 256 px, 363 bins, 32 of 128 angles) on both sides of the rule: a batch
    of 4 (3-angle units) and a batch of 64 whose first 4 images are the same (10-angle
    units).  Both against the oracle; against each other the projections agree to fp32
    rounding (a split unit's pieces are cut elsewhere, and the flexible class band moves
    other near-diagonal angles between the row and the column class when K changes)."""
    N, n_det, n_full, P, m = 256, 363, 128, 1024, 32
    plan = _plan(N, n_det, n_full, P)
    xs = synth.rand_images(4, N, 11)
    idx = _draw_list(n_full, m, seed=9)
    ref = oracle.fwd(xs, idx, n_full, n_det)
    p_small = sk.radon_fwd(plan, dev(xs), idx_t(idx))
    close(p_small, ref, "fwd small launch")
    xl = np.concatenate([xs] * 16, axis=0)
    p_large = sk.radon_fwd(plan, dev(xl), idx_t(idx))
    close(p_large[:4], ref, "fwd large launch, images 0..3")
    close(p_large[60:], ref, "fwd large launch, images 60..63")
    close(p_large[:4], p_small.double().cpu().numpy(), "large vs small launch", tol=2e-5)


@pytest.mark.parametrize("geom", GEOMS)
def test_radon_adj_parity(geom):
    N, n_det, n_full, P, B, m = geom
    plan = _plan(N, n_det, n_full, P)
    y = synth.rand_sinograms(B, m, n_det, 3)
    idx = _draw_list(n_full, m)
    x = sk.radon_adj(plan, dev(y), idx_t(idx), 2.0)
    close(x, oracle.adj(y, idx, n_full, N, 2.0), "adj")
    idxs = np.stack([oracle.draw(6, 0, b, n_full, m)[1] for b in range(B)])
    x = sk.radon_adj(plan, dev(y), idx_t(idxs), 1.0)
    for b in range(B):
        close(x[b], oracle.adj(y[b], idxs[b], n_full, N), f"adj per-image b={b}")


@pytest.mark.parametrize("n_det,P", [(91, 256), (363, 1024), (363, 2048), (725, 2048), (1449, 4096), (7, 16)])
def test_ramp_parity(n_det, P):
    plan = sk.Plan.get(max(2, n_det // 2), n_det, 8, P)
    rows = 7  # odd row count: the last packed pair has one row
    p = synth.rand_sinograms(1, rows, n_det, 4)[0]
    q = sk.ramp_filter(plan, dev(p))
    close(q, oracle.ramp(p), f"ramp n_det={n_det} P={P}")


def test_ramp_fft_length_independent():
    """Same result for P = 1024 and P = 2048 at n_det = 363 (App. A.1 exactness)."""
    p = dev(synth.rand_sinograms(1, 6, 363, 5)[0])
    a = sk.ramp_filter(sk.Plan.get(256, 363, 128, 1024), p)
    b = sk.ramp_filter(sk.Plan.get(256, 363, 128, 2048), p)
    close(a, b.double().cpu().numpy(), "P independence", tol=2e-6)


@pytest.mark.parametrize("geom", GEOMS[:3])
def test_fbp_parity(geom):
    N, n_det, n_full, P, B, m = geom
    plan = _plan(N, n_det, n_full, P)
    y = synth.rand_sinograms(B, m, n_det, 7)
    idx = _draw_list(n_full, m)
    x = sk.fbp(plan, dev(y), idx_t(idx))
    close(x, oracle.fbp(y, idx, n_full, N), "fbp")
    x = sk.fbp(plan, dev(y), idx_t(idx), m_total=4 * m)  # angle-shard scaling pi/(2 m_total)
    close(x, oracle.fbp(y, idx, n_full, N, m_total=4 * m), "fbp m_total")


@pytest.mark.parametrize("geom", GEOMS[:3])
def test_residual_parity(geom):
    N, n_det, n_full, P, B, m = geom
    plan = _plan(N, n_det, n_full, P)
    rng = np.random.default_rng(9)
    p1 = rng.standard_normal((B, m, n_det)).astype(np.float32)
    y = rng.standard_normal((B, n_full, n_det)).astype(np.float32)
    x2 = rng.standard_normal((B, N, N)).astype(np.float32)
    x3 = rng.standard_normal((B, N, N)).astype(np.float32)
    idx = _draw_list(n_full, m)
    mc, ei, r = sk.ei_residual(plan, dev(p1), dev(y), idx_t(idx), dev(x2), dev(x3))
    for b in range(B):
        omc, oei, orr = oracle.residual(p1[b], y[b], idx, x2[b], x3[b])
        close(r[b], orr, "r")
        assert abs(float(mc[b]) - omc) <= TOL * omc
        assert abs(float(ei[b]) - oei) <= TOL * oei
    mc2, ei2, _ = sk.ei_residual(plan, dev(p1), dev(y), idx_t(idx), dev(x2), dev(x2), want_r=False)
    assert torch.all(ei2 == 0)
    assert torch.equal(mc, mc2)


# ---------------------------------------------------------------------- whole pass
def _check_pass(cfg, images, mode=sk.MODE_UNIFORM, it=0, seed=0):
    plan = sk.Plan.get(cfg.N, cfg.n_det, cfg.n_full, cfg.fft_len)
    x1, y = synth.make_workload(cfg, seed)
    shared = not cfg.per_image_draws
    g, idx = sk.draw_device(seed, it, 0, 1 if shared else cfg.B, shared, cfg.n_full, cfg.m, mode)
    out = sk.sketched_pass(plan, dev(x1), dev(y), g if not shared else g[:1], idx)
    torch.cuda.synchronize()
    worst = {}
    for b in images:
        og, oidx = oracle.draw(seed, it, SH if shared else b, cfg.n_full, cfg.m, mode)
        gi = int(g[0 if shared else b])
        assert gi == og and np.array_equal(idx[0 if shared else b].cpu().numpy(), oidx)
        ref = oracle.sketched_pass(x1[b], y[b], og, oidx, cfg.n_full)
        for k in ("x2", "p1", "p2", "q", "xfbp", "r", "grad"):
            worst[k] = max(worst.get(k, 0), close(out[k][b], ref[k], f"{cfg.name} {k} b={b}"))
        for k in ("mc", "ei"):
            rel = abs(float(out[k][b]) - ref[k]) / abs(ref[k])
            assert rel <= TOL, f"{cfg.name} {k} b={b}: rel err {rel:.2e}"
            worst[k] = max(worst.get(k, 0), rel)
    return out, worst


@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
@pytest.mark.parametrize("mode", [sk.MODE_UNIFORM, sk.MODE_INTERLEAVED])
def test_pass_parity_small_configs(name, mode):
    cfg = synth.CONFIGS[name]
    _check_pass(cfg, range(cfg.B), mode)


@pytest.mark.slow
@pytest.mark.parametrize("name", ["cfg3", "cfg4", "cfg5"])
@pytest.mark.parametrize("mode", [sk.MODE_UNIFORM, sk.MODE_INTERLEAVED])
def test_pass_parity_full_size(name, mode):
    """BASELINE.json's full sizes in the bench's launch configuration (whole batch on the
    GPU), in both sketch modes (north_star's uniform subset and the paper's interleaved
    minibatches); the oracle recomputes, in full, the first, second, a middle and the
    last image of the batch (each of its own image group of the projector)."""
    cfg = synth.CONFIGS[name]
    _check_pass(cfg, sorted({0, 1, cfg.B // 2, cfg.B - 1} & set(range(cfg.B))), mode)


def _boundary_sketch(n_full, m, seed=0):
    """A uniform draw of m angles forced to contain the class-boundary angles 0, 45, 90 and
    135 degrees (indices 0, n_full/4, n_full/2, 3 n_full/4): the projector's row / column
    class test is exact there (|cos| = |sin| at 45 and 135 degrees, zero sin / cos at 0 and
    90), and the bin-pair windows reach their widest (|beta| = 1/sqrt 2)."""
    _, idx = oracle.draw(seed, 5, SH, n_full, m)
    must = [0, n_full // 4, n_full // 2, 3 * n_full // 4]
    rest = [i for i in idx if i not in must][: m - len(must)]
    return np.array(sorted(must + rest), np.int32)


@pytest.mark.slow
@pytest.mark.parametrize("g", [45, 90, 137])
def test_pass_parity_full_size_class_boundary_angles(g):
    """cfg3 (N = 512) with a sketch holding 0/45/90/135 degrees; images 0, 5, 10 and 15
    (one of each image group of the projector) against the oracle."""
    cfg = synth.CONFIGS["cfg3"]
    plan = sk.Plan.get(cfg.N, cfg.n_det, cfg.n_full, cfg.fft_len)
    x1, y = synth.make_workload(cfg, 0)
    idx = _boundary_sketch(cfg.n_full, cfg.m)
    out = sk.sketched_pass(plan, dev(x1), dev(y), idx_t([g]), idx_t(idx[None]))
    torch.cuda.synchronize()
    for b in (0, 5, 10, 15):
        ref = oracle.sketched_pass(x1[b], y[b], g, idx, cfg.n_full)
        for k in ("x2", "p1", "p2", "q", "xfbp", "r", "grad"):
            close(out[k][b], ref[k], f"boundary g={g} {k} b={b}")
        for k in ("mc", "ei"):
            assert abs(float(out[k][b]) - ref[k]) <= TOL * abs(ref[k]), (k, b)


def _band_sketch(n_full, n_row, seed):
    """m = 90 angles of n_full = 360 with n_row of them strictly in the row class (|cos| >=
    |sin|), including band angles (within 2.1 degrees of 45 / 135 degrees) on both sides."""
    rng = np.random.default_rng(seed)
    strict_row = lambda i: 4 * i <= n_full or 4 * i >= 3 * n_full  # noqa: E731
    rows = [i for i in range(n_full) if strict_row(i)]
    cols = [i for i in range(n_full) if not strict_row(i)]
    must_r, must_c = [88, 89, 90, 270, 271], [91, 92, 268, 269]
    r = must_r + list(rng.choice([i for i in rows if i not in must_r], n_row - len(must_r), replace=False))
    c = must_c + list(rng.choice([i for i in cols if i not in must_c], 90 - n_row - len(must_c), replace=False))
    return np.array(sorted(r + c), np.int32)


@pytest.mark.parametrize("n_row", [46, 44, 43, 47])
def test_radon_fwd_flexible_class_band(n_row):
    """cfg3 geometry (K = 5 angles per unit) with n_row strict row-class angles: the forward
    moves the band angles nearest a diagonal to the other class so the class sizes become
    multiples of K (46 -> 45, 44 -> 45, 43 -> 45, 47 -> 45): those angles are projected with
    |beta| in [0.68, 1/sqrt 2) — still exact for the bin-pair line loop — against the
    oracle, for one group of 4 images (one packed copy, tensor-map columns) and singly."""
    cfg = synth.CONFIGS["cfg3"]
    plan = sk.Plan.get(cfg.N, cfg.n_det, cfg.n_full, cfg.fft_len)
    idx = _band_sketch(cfg.n_full, n_row, n_row)
    x = synth.rand_images(4, cfg.N, 21)
    p = sk.radon_fwd(plan, dev(x), idx_t(idx[None]))
    for b in range(4):
        close(p[b], oracle.fwd(x[b], idx, cfg.n_full, cfg.n_det), f"band fwd n_row={n_row} b={b}")
    p1 = sk.radon_fwd(plan, dev(x[:1]), idx_t(idx[None]))
    close(p1[0], oracle.fwd(x[0], idx, cfg.n_full, cfg.n_det), f"band fwd single n_row={n_row}")


def test_quad_backprojector_ragged_tiles_all_patterns():
    """The quad backprojector (32 x 32 tiles, four pixels per thread; chosen when its grid
    fills a wave) at N = 500 — ragged last tiles in both directions — with a sketch of every
    other angle of 60 (0, 6, ..., 174 degrees), so every per-angle window pattern (|cos| in
    [0, 1/3], (1/3, 1/2], (1/2, 2/3], (2/3, 1]) occurs with both signs of cos: the standalone
    adjoint and FBP (plain staging) for all 8 images, and the pass (bulk staging, fused EI)
    for two images, against the oracle."""
    N, n_det, n_full, B = 500, 708, 60, 8
    plan = sk.Plan.get(N, n_det, n_full, 0)
    idx = np.arange(0, n_full, 2, dtype=np.int32)
    m = len(idx)
    y = synth.rand_sinograms(B, m, n_det, 11)
    x = sk.radon_adj(plan, dev(y), idx_t(idx), 2.0)
    xf = sk.fbp(plan, dev(y), idx_t(idx))
    for b in range(B):
        close(x[b], oracle.adj(y[b], idx, n_full, N, 2.0), f"quad adj b={b}")
        close(xf[b], oracle.fbp(y[b], idx, n_full, N), f"quad fbp b={b}")
    x1 = synth.rand_images(B, N, 12)
    yf = synth.rand_sinograms(B, n_full, n_det, 13)
    out = sk.sketched_pass(plan, dev(x1), dev(yf), idx_t([73]), idx_t(idx[None]))
    torch.cuda.synchronize()
    for b in (0, B - 1):
        ref = oracle.sketched_pass(x1[b], yf[b], 73, idx, n_full)
        for k in ("x2", "p1", "p2", "q", "xfbp", "r", "grad"):
            close(out[k][b], ref[k], f"quad pass {k} b={b}")
        for k in ("mc", "ei"):
            assert abs(float(out[k][b]) - ref[k]) <= TOL * abs(ref[k]), (k, b)


@pytest.mark.parametrize("N,n_det,n_full,P,B,m", [
    (1536, 2173, 32, 8192, 1, 4),   # the largest image the ABI accepts (n <= 1536), P = 8192
    (256, 3072, 16, 8192, 4, 4),    # the widest detector (n_det <= 3072): one angle per unit
])
def test_pass_parity_max_geometry(N, n_det, n_full, P, B, m):
    """The ABI's size limits (include/skei.h): every output of the pass against the oracle."""
    plan = sk.Plan.get(N, n_det, n_full, P)
    rng = np.random.default_rng(N)
    x1 = synth.rand_images(B, N, 21)
    y = rng.standard_normal((B, n_full, n_det)).astype(np.float32)
    g, idx = sk.draw(5, 1, SH, n_full, m)
    out = sk.sketched_pass(plan, dev(x1), dev(y), idx_t([g]), idx_t(idx))
    for b in range(B):
        ref = oracle.sketched_pass(x1[b], y[b], g, idx, n_full)
        for k in ("x2", "p1", "p2", "q", "xfbp", "r", "grad"):
            close(out[k][b], ref[k], f"max geom {k} b={b}")
        for k in ("mc", "ei"):
            assert abs(float(out[k][b]) - ref[k]) <= TOL * abs(ref[k]), k


def test_pass_deterministic_bitwise():
    cfg = synth.CONFIGS["cfg2"]
    plan = sk.Plan.get(cfg.N, cfg.n_det, cfg.n_full, cfg.fft_len)
    x1, y = synth.make_workload(cfg)
    g, idx = sk.draw_device(0, 0, 0, 1, True, cfg.n_full, cfg.m)
    a = sk.sketched_pass(plan, dev(x1), dev(y), g, idx)
    b = sk.sketched_pass(plan, dev(x1), dev(y), g, idx)
    for k in a:
        assert torch.equal(a[k], b[k]), k


@pytest.mark.parametrize("name", ["cfg2", "cfg3"])
def test_pass_backprojections_match_standalone_calls(name):
    """With image groups of 4 the pass stages the backprojector's detector windows by bulk
    copies from interleaved padded copies of q and r (written by the ramp launch); the
    standalone calls stage them from the plain sinograms.  Same arithmetic: bit-identical."""
    cfg = synth.CONFIGS[name]
    plan = sk.Plan.get(cfg.N, cfg.n_det, cfg.n_full, cfg.fft_len)
    x1, y = synth.make_workload(cfg)
    g, idx = sk.draw_device(0, 3, 0, 1, True, cfg.n_full, cfg.m)
    out = sk.sketched_pass(plan, dev(x1), dev(y), g, idx)
    assert torch.equal(sk.ramp_filter(plan, out["p2"]), out["q"])
    assert torch.equal(sk.fbp(plan, out["p2"], idx), out["xfbp"])
    assert torch.equal(sk.radon_adj(plan, out["r"], idx, 2.0), out["grad"])


@pytest.mark.parametrize("name,shared,mode", [("cfg2", True, sk.MODE_UNIFORM),
                                              ("cfg2", True, sk.MODE_INTERLEAVED),
                                              ("cfg3", True, sk.MODE_UNIFORM),
                                              ("cfg2", False, sk.MODE_UNIFORM)])
def test_pass_draw_matches_draw_then_pass(name, shared, mode):
    """skei_pass_draw (draw kernel + programmatically serialised rotate/pack) gives exactly
    the draws of skei_draw_device and the outputs of skei_pass on them, also when captured
    into a CUDA graph and replayed (the bench's timed form)."""
    cfg = synth.CONFIGS[name]
    plan = sk.Plan.get(cfg.N, cfg.n_det, cfg.n_full, cfg.fft_len)
    x1, y = (dev(a) for a in synth.make_workload(cfg))
    nd = 1 if shared else cfg.B
    g, idx = sk.draw_device(7, 11, 3, nd, shared, cfg.n_full, cfg.m, mode)
    ref = sk.sketched_pass(plan, x1, y, g, idx)
    out, g2, idx2 = sk.sketched_pass_draw(plan, x1, y, 7, 11, cfg.m, mode, shared, 3)
    assert torch.equal(g, g2) and torch.equal(idx, idx2)
    for k in ref:
        assert torch.equal(out[k], ref[k]), k
    # graph capture and replay, outputs cleared in between
    for v in out.values():
        v.zero_()
    g2.zero_()
    idx2.zero_()
    ws = plan.workspace(cfg.B, cfg.m)
    torch.cuda.synchronize()
    cap = torch.cuda.Stream()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=cap):
        sk.sketched_pass_draw(plan, x1, y, 7, 11, cfg.m, mode, shared, 3, g=g2, idx=idx2,
                              out=out, ws=ws)
    for v in out.values():
        v.zero_()
    for _ in range(2):
        gr.replay()
    torch.cuda.synchronize()
    assert torch.equal(g, g2) and torch.equal(idx, idx2)
    for k in ref:
        assert torch.equal(out[k], ref[k]), f"graph {k}"


def test_gpu_adjoint_identity():
    cfg = synth.CONFIGS["cfg2"]
    plan = sk.Plan.get(cfg.N, cfg.n_det, cfg.n_full, cfg.fft_len)
    x = synth.rand_images(2, cfg.N, 10)
    yv = synth.rand_sinograms(2, cfg.m, cfg.n_det, 11)
    idx = idx_t(_draw_list(cfg.n_full, cfg.m))
    Ax = sk.radon_fwd(plan, dev(x), idx).double().cpu().numpy()
    ATy = sk.radon_adj(plan, dev(yv), idx).double().cpu().numpy()
    lhs, rhs = float((Ax * yv).sum()), float((x * ATy).sum())
    assert abs(lhs - rhs) / (np.linalg.norm(Ax) * np.linalg.norm(yv)) <= 1e-6


@pytest.mark.parametrize("stage", [False, True])
@pytest.mark.parametrize("name,shared,mode", [("cfg1", True, sk.MODE_UNIFORM),
                                              ("cfg2", True, sk.MODE_UNIFORM),
                                              ("cfg2", True, sk.MODE_INTERLEAVED),
                                              ("cfg2", False, sk.MODE_UNIFORM),
                                              ("cfg2", False, sk.MODE_INTERLEAVED),
                                              ("cfg4", False, sk.MODE_UNIFORM)])
def test_pass_host_matches_device_pass(name, shared, mode, stage):
    """skei_pass_host (only y's sketched rows cross the link: gathered per image into the
    staging buffer — each image's own rows for per-image sketches, several host threads at
    cfg4 — or, for a shared sketch without one, strided copies of runs of consecutive
    angles) gives exactly skei_pass's results on device copies."""
    cfg = synth.CONFIGS[name]
    plan = sk.Plan.get(cfg.N, cfg.n_det, cfg.n_full, cfg.fft_len)
    x1, y = synth.make_workload(cfg)
    draws = [sk.draw(0, 0, SH if shared else b, cfg.n_full, cfg.m, mode)
             for b in range(1 if shared else cfg.B)]
    g = [d[0] for d in draws]
    idx = np.stack([d[1] for d in draws])
    ref = sk.sketched_pass(plan, dev(x1), dev(y), idx_t(g), idx_t(idx))
    h = {k: torch.from_numpy(v).pin_memory() for k, v in (("x1", x1), ("y", y))}
    hg = torch.tensor(g, dtype=torch.int32).pin_memory()
    hidx = torch.tensor(idx, dtype=torch.int32).pin_memory()
    d = sk.alloc_pass_outputs(plan, cfg.B, cfg.m, "cuda")
    d.update(x1=torch.empty_like(dev(x1)), y=torch.full_like(dev(y), float("nan")),
             g=torch.empty(len(g), dtype=torch.int32, device="cuda"),
             idx=torch.empty(idx.shape, dtype=torch.int32, device="cuda"))
    hmc = torch.empty(cfg.B).pin_memory()
    hei = torch.empty(cfg.B).pin_memory()
    ws = plan.workspace(cfg.B, cfg.m)
    ys = torch.full((cfg.B, cfg.m, cfg.n_det), float("nan")).pin_memory() if stage else None
    sk.sketched_pass_host(plan, h["x1"], h["y"], hg, hidx, d, hmc, hei, ws, d["x2"], h_ystage=ys)
    torch.cuda.synchronize()
    assert torch.equal(hmc, ref["mc"].cpu()) and torch.equal(hei, ref["ei"].cpu())
    for k in ("r", "grad", "xfbp", "p1"):
        assert torch.equal(d[k], ref[k]), k


def test_invalid_shapes_raise():
    plan = sk.Plan.get(64, 91, 32, 256)
    x = torch.zeros(0, 64, 64, device="cuda")
    with pytest.raises(sk.SkeiError):
        sk.radon_fwd(plan, x, idx_t([0, 1]))
    with pytest.raises(sk.SkeiError):
        sk.radon_fwd(plan, torch.zeros(1, 64, 64, device="cuda"), idx_t(list(range(33))))
    with pytest.raises(sk.SkeiError):
        sk.rotate(plan, torch.zeros(1, 64, 64, device="cuda", dtype=torch.float64), idx_t([3]))
