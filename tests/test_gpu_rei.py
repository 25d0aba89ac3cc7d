"""GPU parity of the next row SURVEY §8(f) #3: the REI pass, whose EI
branch reconstructs from A_S x2 + sigma eps with the counter-based simulated noise
(R23).  Against the oracle's independent generator and REI pass at the
north_star tolerance; sigma = 0 is skei_pass bit for bit."""
import numpy as np
import pytest
import torch

import oracle
import paper_2411_05771_b200 as sk
import synth

from test_gpu_parity import close, dev

pytestmark = pytest.mark.gpu
TOL = 1e-4


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)


def _run(name, sigma_rel, images, image0=0, it=3):
    cfg = synth.CONFIGS[name]
    plan = sk.Plan.get(cfg.N, cfg.n_det, cfg.n_full, cfg.fft_len)
    x1, y = synth.make_workload(cfg, seed=0)
    g, idx = sk.draw_device(0, it, 0, 1, True, cfg.n_full, cfg.m)
    sigma = sigma_rel * float(np.abs(y).max())
    out = sk.sketched_pass_rei(plan, dev(x1), dev(y), g, idx, sigma, 11, it, image0)
    og, oidx = int(g[0]), idx[0].cpu().numpy()
    for b in images:
        ref = oracle.sketched_pass_rei(x1[b], y[b], og, oidx, cfg.n_full, float(np.float32(sigma)),
                                       11, it, image0 + b)
        for k in ("x2", "p1", "p2", "q", "xfbp", "r", "grad"):
            close(out[k][b], ref[k], f"{name} REI {k} b={b}")
        for k in ("mc", "ei"):
            assert abs(float(out[k][b]) - ref[k]) <= TOL * abs(ref[k]), f"{name} REI {k} b={b}"
    return out


@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_rei_pass_parity(name):
    cfg = synth.CONFIGS[name]
    _run(name, 0.01, range(cfg.B))


def test_rei_pass_parity_full_size_and_image_offset():
    _run("cfg3", 0.005, (0, 15), image0=32)


def test_rei_sigma_zero_is_the_pass_bitwise():
    cfg = synth.CONFIGS["cfg2"]
    plan = sk.Plan.get(cfg.N, cfg.n_det, cfg.n_full, cfg.fft_len)
    x1, y = synth.make_workload(cfg, seed=0)
    g, idx = sk.draw_device(0, 1, 0, 1, True, cfg.n_full, cfg.m)
    a = sk.sketched_pass(plan, dev(x1), dev(y), g, idx)
    b = sk.sketched_pass_rei(plan, dev(x1), dev(y), g, idx, 0.0, 5, 1)
    for k in a:
        assert torch.equal(a[k], b[k]), k


def test_rei_noise_through_the_ramp_matches_oracle_generator():
    """x1 = 0: q = ramp(sigma eps) isolates the device generator (cfg2, all images)."""
    cfg = synth.CONFIGS["cfg2"]
    plan = sk.Plan.get(cfg.N, cfg.n_det, cfg.n_full, cfg.fft_len)
    x1 = np.zeros((cfg.B, cfg.N, cfg.N), np.float32)
    y = np.zeros((cfg.B, cfg.n_full, cfg.n_det), np.float32)
    g, idx = sk.draw_device(0, 2, 0, 1, True, cfg.n_full, cfg.m)
    out = sk.sketched_pass_rei(plan, dev(x1), dev(y), g, idx, 1.0, 99, 7, 100)
    for b in range(cfg.B):
        close(out["q"][b], oracle.ramp(oracle.rei_noise(99, 7, 100 + b, cfg.m, cfg.n_det)), f"q b={b}")
