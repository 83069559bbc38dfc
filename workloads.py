"""Seeded synthetic workloads shared by tests, bench.py and smoke().

Holds only the input recipe (mesh kind, size, jitter, seed) of BASELINE.json's
five configs -- none of the method's arithmetic.  The GPU mesh generator
(efem_build_mesh) and the oracle's generator (ora_build_mesh) each implement
the same counter-hash recipe independently; see DESIGN.md "Inputs".
"""

RT0, NED0 = 0, 1
ELEMENT_NAMES = {RT0: "RT0", NED0: "NE0"}

# BASELINE.json "configs", in order.  alpha = jitter as a fraction of h = 1/n.
CONFIGS = {
    1: dict(dim=2, element=RT0, n=16, alpha=0.10, seed=0, name="cfg1_rt0_2d_16x16"),
    2: dict(dim=2, element=NED0, n=1024, alpha=0.20, seed=1, name="cfg2_ne0_2d_1024x1024"),
    3: dict(dim=3, element=RT0, n=64, alpha=0.15, seed=2, name="cfg3_rt0_3d_64cube"),
    4: dict(dim=3, element=NED0, n=128, alpha=0.15, seed=3, name="cfg4_ne0_3d_128cube"),
    5: dict(dim=2, element=RT0, n=4096, alpha=0.20, seed=4, name="cfg5_rt0_2d_4096x4096"),
}


def counts(dim: int, element: int, n: int):
    """Closed-form sizes of the structured meshes (fitted exactly):
    returns (N, T, R, nnz)."""
    if dim == 2:
        return (n + 1) ** 2, 2 * n * n, 3 * n * n + 2 * n, 15 * n * n + 2 * n
    N, T = (n + 1) ** 3, 6 * n ** 3
    if element == RT0:
        return N, T, 12 * n ** 3 + 6 * n ** 2, 84 * n ** 3 + 6 * n ** 2
    return N, T, 7 * n ** 3 + 9 * n ** 2 + 3 * n, 115 * n ** 3 + 45 * n ** 2 + 3 * n
