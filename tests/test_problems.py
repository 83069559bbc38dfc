"""Pins of the eddy-current problem data (problems.py) against finite
differences and the properties PAPER.md:883-905 states for it."""
import numpy as np

import problems as P


def _pts(n=400, seed=0, side=1):
    rng = np.random.default_rng(seed)
    x = rng.uniform(0.02, 0.98, size=(n, 2))
    keep = (x[:, 0] - x[:, 1]) * side > 0.02  # stay off the diagonal for the stencils
    return x[keep, 0], x[keep, 1]


def _fd(f, x1, x2, h=1e-5):
    d1 = (f(x1 + h, x2) - f(x1 - h, x2)) / (2 * h)
    d2 = (f(x1, x2 + h) - f(x1, x2 - h)) / (2 * h)
    return d1, d2


def test_curl_matches_finite_differences():
    x1, x2 = _pts()
    e1 = lambda a, b: P.eddy_E(a, b)[0]  # noqa: E731
    e2 = lambda a, b: P.eddy_E(a, b)[1]  # noqa: E731
    d1e2 = _fd(e2, x1, x2)[0]
    d2e1 = _fd(e1, x1, x2)[1]
    np.testing.assert_allclose(P.eddy_curlE(x1, x2), d1e2 - d2e1, rtol=1e-6, atol=1e-7)


def test_F_is_curl_curl_plus_E():
    x1, x2 = _pts(seed=1)
    c1, c2 = _fd(P.eddy_curlE, x1, x2)
    E1, E2 = P.eddy_E(x1, x2)
    F1, F2 = P.eddy_F(x1, x2)
    np.testing.assert_allclose(F1, c2 + E1, rtol=1e-6, atol=1e-6)
    np.testing.assert_allclose(F2, -c1 + E2, rtol=1e-6, atol=1e-6)


def test_zero_on_omega2():
    x1, x2 = _pts(seed=2, side=-1)
    for f in (P.eddy_E(x1, x2)[0], P.eddy_E(x1, x2)[1], P.eddy_curlE(x1, x2), P.eddy_F(x1, x2)[0]):
        assert np.all(f == 0.0)


def test_paper_stated_properties():
    """Tangential E continuous across x1 = x2 (E|Omega_1 . (1,1) = 0 there),
    curl E = 0 on the diagonal and on the whole boundary."""
    s = np.linspace(0.0, 1.0, 101)
    # on the diagonal, evaluate the Omega_1 formula (x1 slightly above x2 picks it)
    e1, e2 = P.eddy_E(s + 1e-300, s)
    np.testing.assert_allclose(e1 + e2, 0.0, atol=1e-12)
    np.testing.assert_allclose(P.eddy_curlE(s + 1e-300, s), 0.0, atol=1e-12)
    one, zero = np.ones_like(s), np.zeros_like(s)
    for x1, x2 in ((one, s), (s, zero)):  # the boundary pieces inside Omega_1's closure
        np.testing.assert_allclose(P.eddy_curlE(x1 + 0 * s, x2), 0.0, atol=1e-12)


def test_table5_sizes_match_the_structured_mesh():
    """#T = 2 n^2 and #E = 3 n^2 + 2 n for the unit-square meshes of Table 5."""
    for r in table5():
        n = r["n"]
        assert r["T"] == 2 * n * n and r["E"] == 3 * n * n + 2 * n


def table5():
    import json
    import os

    return json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_table5_eddy.json")))["rows"]
