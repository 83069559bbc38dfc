"""GPU parity of the P1 support kernels against the oracle, and the paper's
Table 3 (2D majorant) reproduced by the CUDA path
(SURVEY §8(f) f3)."""
import json
import math
import os
import sys

import numpy as np
import pytest
import torch

from oracle import oracle as ora

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "examples"))


@pytest.fixture(scope="module")
def api():
    from paper_1409_4618_b200 import api as a

    assert torch.cuda.is_available()
    return a


@pytest.mark.parametrize("dim,n", [(2, 9), (3, 4)])
def test_p1_parity(api, dim, n):
    c, e = api.build_mesh(dim, n, 0.15, 21, device="cuda:0")
    hc, he = c.cpu().numpy(), e.cpu().numpy()
    p1 = api.P1Assembler(c, e)
    A = p1.assemble()
    rp, ci, vm, vk = ora.p1_assemble(dim, hc, he)
    assert np.array_equal(A.row_ptr.cpu().numpy(), rp) and np.array_equal(A.col_idx.cpu().numpy(), ci)
    np.testing.assert_allclose(A.vals_K.cpu().numpy(), vk, rtol=0, atol=1e-12 * np.abs(vk).max())
    np.testing.assert_allclose(A.vals_M.cpu().numpy(), vm, rtol=0, atol=1e-12 * np.abs(vm).max())
    rng = np.random.default_rng(dim)
    fq = rng.normal(size=(he.shape[0], api.quad_size(dim)))
    b = p1.load(torch.from_numpy(fq).cuda()).cpu().numpy()
    rb = ora.p1_load(dim, hc, he, fq)
    np.testing.assert_allclose(b, rb, rtol=0, atol=1e-13 * np.abs(rb).max())
    v = rng.normal(size=hc.shape[0])
    g = api.p1_gradient(c, e, torch.from_numpy(v).cuda()).cpu().numpy()
    rg = ora.p1_grad(dim, hc, he, v)
    np.testing.assert_allclose(g, np.repeat(rg[:, None, :], g.shape[1], axis=1), rtol=0, atol=1e-11)


def test_dirichlet_elimination(api):
    c, e = api.build_mesh(2, 6, 0.1, 2, device="cuda:0")
    p1 = api.P1Assembler(c, e)
    A = p1.assemble()
    mask = torch.zeros(c.shape[0], dtype=torch.bool, device="cuda")
    mask[::3] = True
    b = torch.ones(c.shape[0], dtype=torch.float64, device="cuda")
    api.dirichlet(A, mask, b)
    rp, ci, vk = A.row_ptr.cpu().numpy(), A.col_idx.cpu().numpy(), A.vals_K.cpu().numpy()
    m = mask.cpu().numpy()
    rows = np.repeat(np.arange(len(rp) - 1), np.diff(rp))
    hit = m[rows] | m[ci]
    assert np.all(vk[hit & (rows == ci)] == 1.0) and np.all(vk[hit & (rows != ci)] == 0.0)
    assert np.all(b.cpu().numpy()[m] == 0.0)


def _trunc(x, digits):
    f = 10.0 ** digits
    return math.floor(x * f + 1e-9) / f


@pytest.mark.parametrize("col", [0, 1, 2], ids=["T512", "T131072", "T2097152"])
def test_majorant_table3_gpu(api, col):
    import majorant

    t = json.load(open(os.path.join(ROOT, "tests", "golden", "paper_table3_4_majorant.json")))["table3_2d"]
    hist, _, _ = majorant.run(2, t["n"][col])
    rows = t["rows"][col]
    assert len(hist) == len(rows)
    for (beta, sm, ieff), (_, pb, pm, pi) in zip(hist, rows):
        assert _trunc(beta, 3) == pytest.approx(pb, abs=1e-9)
        assert abs(sm - pm) <= 0.51e-6
        assert _trunc(ieff, 2) == pytest.approx(pi, abs=1e-9)


def test_majorant_3d_guaranteed_and_monotone_gpu(api):
    import majorant

    hist, err2, _ = majorant.run(3, 12)
    ms = [h[1] ** 2 for h in hist]
    assert all(m >= err2 for m in ms)
    assert all(b <= a * (1 + 1e-12) for a, b in zip(ms, ms[1:]))
