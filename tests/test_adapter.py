"""Drop-in check at the reference's plugin boundary.

The reference's own ``fde::gmres`` (proj/src/krylov.cpp:12-166) and step loop
(driver.cpp:34-52) run with ``B200Op : fde::LinOp`` and ``B200Mgm :
fde::Precond`` -- adapters over the C ABI built from the reference's own
operator and V-cycle hierarchy (oracle/adapter.cpp).  Mixing
reference and B200 objects in one solve must not change the iteration counts
and may move the solution only by rounding.
"""
import ctypes

import numpy as np
import pytest

from oracles import ADAPTER_SO, adapter, dims_of, spec

pytestmark = pytest.mark.skipif(not ADAPTER_SO.exists(),
                                reason="oracle/_ref/libfde_adapter.so not built")


def test_adapter_exports():
    lib = ctypes.CDLL(str(ADAPTER_SO))
    for name in ("adapter_gmres", "adapter_march", "adapter_last_error"):
        assert hasattr(lib, name), name


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


CASES = [
    dict(cfg=1),
    dict(cfg=2),
    dict(cfg=3, n1=255, n2=255, steps=4),                  # (1,-1) blocks, semicoarsened plan
    dict(cfg=3, n1=127, n2=127, steps=4, coarse=0),        # dense-LU coarsest
    dict(cfg=4, n1=511, n2=511),
]


@pytest.mark.gpu
@pytest.mark.parametrize("kw", CASES, ids=lambda kw: "-".join(f"{k}{v}" for k, v in kw.items()))
def test_reference_gmres_drives_b200(kw, ref):
    ad = adapter()
    kw = dict(kw)
    s = spec(kw.pop("cfg"), **kw)
    b = _rhs(s)
    x0, it0, c0, h0 = ad.gmres(s, b, gpu_op=False, gpu_pc=False)  # all reference
    for gop, gpc in ((True, False), (False, True), (True, True)):
        x, it, conv, h = ad.gmres(s, b, gpu_op=gop, gpu_pc=gpc)
        assert conv == c0 and it == it0, (gop, gpc, it, it0)
        assert rel(x, x0) <= 1e-10, (gop, gpc, rel(x, x0))
        np.testing.assert_allclose(h, h0, rtol=1e-6, atol=1e-13)


def _rhs(s):
    n1, n2 = dims_of(s)
    return np.random.default_rng(11).standard_normal(n1 * n2)


@pytest.mark.gpu
def test_reference_step_loop_drives_b200(ref):
    s = spec(1, steps=16)
    got = adapter().march(s)
    want = ref.march(s)
    np.testing.assert_array_equal(got["its"], want["its"])
    assert rel(got["u"], want["u"]) <= 1e-10
