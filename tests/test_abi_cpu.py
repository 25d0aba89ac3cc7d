"""CPU-side checks of the C-ABI library (no GPU needed):
- libskei.so loads and exports every function include/skei.h declares;
- host-side validation returns the documented status codes without launching anything;
- the library's host draw (skei_draw) is bit-identical to the independent oracle draw
  (north_star: "rotation angles and sketch subsets must be bit-identical to the oracle's").
"""
import ctypes
import os
import re

import pytest
import torch

import oracle
import paper_2411_05771_b200 as sk
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "skei.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(skei_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    names = _declared_functions()
    assert len(names) == 30
    L = ctypes.CDLL(sk.lib_path)
    for name in names:
        assert hasattr(L, name), name
    assert sk.version().endswith("sm_100a")


def test_status_strings():
    for s in range(6):
        assert sk.lib().skei_status_string(s)


def test_host_validation_without_device():
    L = sk.lib()
    # NULL plan / NULL pointers -> SKEI_ERR_ARG, nothing launched
    assert L.skei_radon_fwd(None, None, None, 1, None, 1, 0, None, 0, None) == 3
    assert L.skei_ramp_filter(None, None, None, 1, None) == 3
    assert L.skei_rotate_adjoint(None, None, None, 1, None, 0, None) == 3
    assert L.skei_backproject_scatter(None, 1, None, None, None, 1, 0, 1, None, 2, 0, None) == 3
    assert L.skei_band_reduce(None, 1, None, 2, 0, None, None, None, None, None, 0, None) == 3
    assert L.skei_rs_recv_floats(None, 1, 2) == 0
    assert L.skei_plan_create(None, 0, None) == 3
    g = sk._Geom(64, 91, 32, 100)  # fft_len not a power of two -> config error
    h = ctypes.c_void_p()
    assert L.skei_plan_create(ctypes.byref(g), 0, ctypes.byref(h)) == 2
    g = sk._Geom(64, 91, 32, 128)  # 128 < 2*91-1 -> config error
    assert L.skei_plan_create(ctypes.byref(g), 0, ctypes.byref(h)) == 2
    g = sk._Geom(1537, 2174, 32, 0)  # n > 1536: a line block would not fit shared memory
    assert L.skei_plan_create(ctypes.byref(g), 0, ctypes.byref(h)) == 2
    if not torch.cuda.is_available():
        g = sk._Geom(64, 91, 32, 0)
        assert L.skei_plan_create(ctypes.byref(g), 0, ctypes.byref(h)) == 5  # no device


def test_draw_errors():
    with pytest.raises(sk.SkeiError):
        sk.draw(0, 0, sk.SHARED_IMAGE, 10, 11)
    with pytest.raises(sk.SkeiError):
        sk.draw(0, 0, sk.SHARED_IMAGE, 10, 3, sk.MODE_INTERLEAVED)
    with pytest.raises(sk.SkeiError):
        sk.draw(0, 0, sk.SHARED_IMAGE, 10, 0)


@pytest.mark.parametrize("name", list(synth.CONFIGS))
@pytest.mark.parametrize("mode", [sk.MODE_UNIFORM, sk.MODE_INTERLEAVED])
def test_host_draw_bit_identical_to_oracle(name, mode):
    cfg = synth.CONFIGS[name]
    images = [sk.SHARED_IMAGE, 0, 1, cfg.B - 1, 12345]
    for it in range(40):
        for im in images:
            assert sk.draw(0, it, im, cfg.n_full, cfg.m, mode) == \
                tuple_list(oracle.draw(0, it, im, cfg.n_full, cfg.m, mode))
    # other seeds / sizes, including m = n_full and m = 1
    for seed in (1, 2 ** 63 + 5):
        for (n_full, m) in ((7, 1), (7, 7), (1024, 256), (16384, 3)):
            if mode == sk.MODE_INTERLEAVED and n_full % m:
                continue
            assert sk.draw(seed, 3, 9, n_full, m, mode) == tuple_list(oracle.draw(seed, 3, 9, n_full, m, mode))


def tuple_list(gi):
    return gi[0], [int(v) for v in gi[1]]
