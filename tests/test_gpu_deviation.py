"""GPU parity of the next row SURVEY §8(f) #4: the Theorem-1 sketching deviation
||A^T (S^T S - I) A||_2 by power iteration on the pass's
kernels, against the fp64 oracle's power iteration from the same start image."""
import numpy as np
import pytest
import torch

import oracle
import paper_2411_05771_b200 as sk
import synth

from test_gpu_parity import dev, idx_t

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3"])
def test_sketch_deviation_one_application_matches_oracle(name):
    """One application of D = (n_full/m) A_S^T A_S - A^T A to the same unit
    start image on both sides: the GPU's iterate times lambda is D v elementwise, within the
    north_star bar 1e-4 max|ref|, and lambda = ||D v|| within 1e-4 relative.  (A run of
    several iterations compares two different iterates; this isolates the kernels.)"""
    cfg = synth.CONFIGS[name]
    plan = sk.Plan.get(cfg.N, cfg.n_det, cfg.n_full, cfg.fft_len)
    _, idx = sk.draw(0, 1, sk.SHARED_IMAGE, cfg.n_full, cfg.m)
    v0 = np.random.default_rng(3).standard_normal((2, cfg.N, cfg.N)).astype(np.float32)
    v = dev(v0)
    lam = sk.sketch_deviation(plan, idx_t(idx), v, 1)
    dv = (v.double() * lam.double()[:, None, None]).cpu().numpy()
    for b in range(2):
        ref_lam, ref_v = oracle.sketch_deviation(v0[b], idx, cfg.n_full, cfg.n_det, 1)
        ref = ref_v * ref_lam
        err = np.abs(dv[b] - ref).max()
        assert err <= 1e-4 * np.abs(ref).max(), (b, err, np.abs(ref).max())
        assert abs(float(lam[b]) - ref_lam) <= 1e-4 * ref_lam, (b, float(lam[b]), ref_lam)


@pytest.mark.parametrize("name,per_image", [("cfg1", True), ("cfg2", True), ("cfg2", False)])
def test_sketch_deviation_batch_of_four(name, per_image):
    """B = 4 start images: the full-angle forward runs on groups of 4 (one packed copy, the
    column class through the tensor map); with per-image sketches (idx_stride = m) the
    sketched forward groups images singly, so v is packed again in that layout.  One
    application of D against the oracle with each image's own sketch."""
    cfg = synth.CONFIGS[name]
    plan = sk.Plan.get(cfg.N, cfg.n_det, cfg.n_full, cfg.fft_len)
    idxs = [np.asarray(sk.draw(0, 1, b if per_image else sk.SHARED_IMAGE, cfg.n_full, cfg.m)[1])
            for b in range(4)]
    idx = np.stack(idxs) if per_image else idxs[0][None]
    v0 = np.random.default_rng(5).standard_normal((4, cfg.N, cfg.N)).astype(np.float32)
    v = dev(v0)
    lam = sk.sketch_deviation(plan, idx_t(idx), v, 1)
    dv = (v.double() * lam.double()[:, None, None]).cpu().numpy()
    for b in range(4):
        ref_lam, ref_v = oracle.sketch_deviation(v0[b], idxs[b], cfg.n_full, cfg.n_det, 1)
        ref = ref_v * ref_lam
        err = np.abs(dv[b] - ref).max()
        assert err <= 1e-4 * np.abs(ref).max(), (b, err, np.abs(ref).max())
        assert abs(float(lam[b]) - ref_lam) <= 1e-4 * ref_lam, (b, float(lam[b]), ref_lam)


@pytest.mark.parametrize("name,iters", [("cfg1", 80), ("cfg2", 30)])
def test_sketch_deviation_power_iteration_tracks_oracle(name, iters):
    """The converged estimate: both power iterations from the same start image approach
    ||D||_2; after `iters` steps they agree within 1e-3 relative (fp32 vs fp64 iterates;
    the single application above is the kernels' parity check)."""
    cfg = synth.CONFIGS[name]
    plan = sk.Plan.get(cfg.N, cfg.n_det, cfg.n_full, cfg.fft_len)
    _, idx = sk.draw(0, 1, sk.SHARED_IMAGE, cfg.n_full, cfg.m)
    v0 = np.random.default_rng(3).standard_normal((2, cfg.N, cfg.N)).astype(np.float32)
    lam = sk.sketch_deviation(plan, idx_t(idx), dev(v0), iters)
    for b in range(2):
        ref, _ = oracle.sketch_deviation(v0[b], idx, cfg.n_full, cfg.n_det, iters)
        assert abs(float(lam[b]) - ref) <= 1e-3 * ref, (b, float(lam[b]), ref)


def test_sketch_deviation_shrinks_with_sketch_size_and_vanishes_at_full():
    """delta decreases as m grows (Theorem 1: O(1/sqrt m)) and is 0 at m = n_full."""
    cfg = synth.CONFIGS["cfg1"]
    plan = sk.Plan.get(cfg.N, cfg.n_det, cfg.n_full, cfg.fft_len)
    v0 = dev(np.random.default_rng(4).standard_normal((1, cfg.N, cfg.N)).astype(np.float32))
    lams = []
    for m in (4, 8, 16):
        _, idx = sk.draw(0, 2, sk.SHARED_IMAGE, cfg.n_full, m, sk.MODE_INTERLEAVED)
        lams.append(float(sk.sketch_deviation(plan, idx_t(idx), v0.clone(), 60)[0]))
    assert lams[0] > lams[1] > lams[2] > 0
    full = sk.sketch_deviation(plan, idx_t(np.arange(cfg.n_full)), v0.clone(), 3)
    assert float(full[0]) == 0.0
