"""Problem data of the paper's experiments (inputs, not the method).

The 2D eddy-current example of PAPER.md:863-920 (Sec. 4.2, Example "equality"):
unit square, kappa = mu = 1, Gamma_D empty, the exact solution E is
discontinuous across the diagonal x1 = x2:

    E|Omega_1 = ( sin(2 pi x1) + 2 pi cos(2 pi x1) (x1 - x2),
                  sin((x1 - x2)^2 (x1 - 1)^2 x2) - sin(2 pi x1) ),   Omega_1 = {x1 > x2}
    E|Omega_2 = 0,

curl E = 2 x2 (x1 - x2)(x1 - 1)(2 x1 - x2 - 1) cos(x2 (x1 - x2)^2 (x1 - 1)^2)
(PAPER.md:896-900), and the right-hand side of the weak form
 is F = curl_vec(mu^-1 curl E) + kappa E with
curl_vec c = (d2 c, -d1 c).  The derivatives below are worked out by hand
(product rule) and pinned against finite differences in
tests/test_problems.py.

Shared by the GPU examples / tests and the oracle tests as the seeded mesh
generator is: problem data only, no assembly arithmetic.  Every function
takes an array namespace `xp` (numpy or torch) so the same formulas run on
host arrays and device tensors.

The paper's printed results for this problem (Table 5) are a test fixture:
tests/golden/paper_table5_eddy.json.
"""
from __future__ import annotations

import math

import numpy as np

TWO_PI = 2.0 * math.pi


def _parts(x1, x2, xp):
    A = x1 - x2
    B = x1 - 1.0
    C = 2.0 * x1 - x2 - 1.0
    g = A * A * B * B * x2                      # argument of sin / cos
    g1 = 2.0 * x2 * A * B * C                   # d g / d x1
    g2 = B * B * A * (x1 - 3.0 * x2)            # d g / d x2
    return A, B, C, g, g1, g2


def eddy_E(x1, x2, xp=np):
    """Exact solution (both components), zero on Omega_2 = {x1 <= x2}."""
    A, B, C, g, g1, g2 = _parts(x1, x2, xp)
    e1 = xp.sin(TWO_PI * x1) + TWO_PI * xp.cos(TWO_PI * x1) * A
    e2 = xp.sin(g) - xp.sin(TWO_PI * x1)
    in1 = x1 > x2
    z = xp.zeros_like(x1)
    return xp.where(in1, e1, z), xp.where(in1, e2, z)


def eddy_curlE(x1, x2, xp=np):
    """curl E = d1 E2 - d2 E1 = cos(g) d1 g on Omega_1, 0 on Omega_2."""
    A, B, C, g, g1, g2 = _parts(x1, x2, xp)
    c = xp.cos(g) * g1
    return xp.where(x1 > x2, c, xp.zeros_like(x1))


def eddy_F(x1, x2, xp=np):
    """F = curl_vec(curl E) + E with curl_vec c = (d2 c, -d1 c)."""
    A, B, C, g, g1, g2 = _parts(x1, x2, xp)
    # h = g1 = 2 x2 A B C;  dh/dx1 = 2 x2 (B C + A C + 2 A B);  dh/dx2 = 2 A B C - 2 x2 (B C + A B)
    h1 = 2.0 * x2 * (B * C + A * C + 2.0 * A * B)
    h2 = 2.0 * A * B * C - 2.0 * x2 * (B * C + A * B)
    sg, cg = xp.sin(g), xp.cos(g)
    c1 = -sg * g1 * g1 + cg * h1                # d curlE / d x1
    c2 = -sg * g2 * g1 + cg * h2                # d curlE / d x2
    e1 = xp.sin(TWO_PI * x1) + TWO_PI * xp.cos(TWO_PI * x1) * A
    e2 = sg - xp.sin(TWO_PI * x1)
    in1 = x1 > x2
    z = xp.zeros_like(x1)
    return xp.where(in1, c2 + e1, z), xp.where(in1, -c1 + e2, z)


# --------------------------------------------------------------------------- majorant example
# Poisson -lap u = f, u = 0 on the boundary of (0,1)^d, exact solution the
# bubble u(x) = prod_i x_i (x_i - 1); the Friedrichs constant of the unit
# square / cube (reading F1 in DESIGN.md): C_F = 1 / (pi sqrt(d)).

def bubble_u(x, xp=np):
    """x: (..., d)."""
    return xp.prod(x * (x - 1.0), -1) if xp is np else (x * (x - 1.0)).prod(-1)


def _others(x, i):
    d = x.shape[-1]
    out = None
    for j in range(d):
        if j != i:
            t = x[..., j] * (x[..., j] - 1.0)
            out = t if out is None else out * t
    return out


def bubble_grad(x, xp=np):
    d = x.shape[-1]
    comps = [_others(x, i) * (2.0 * x[..., i] - 1.0) for i in range(d)]
    return xp.stack(comps, -1) if xp is np else xp.stack(comps, dim=-1)


def bubble_f(x, xp=np):
    """f = -lap u = -sum_i 2 prod_{j != i} x_j (x_j - 1)."""
    d = x.shape[-1]
    out = None
    for i in range(d):
        t = -2.0 * _others(x, i)
        out = t if out is None else out + t
    return out


def friedrichs_unit(dim):
    return 1.0 / (math.pi * math.sqrt(dim))
