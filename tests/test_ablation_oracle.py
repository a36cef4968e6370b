"""Pin the oracle's ablation_volume against the SPEC examples,
closed forms of the clipping, and the stated invariants (monotone, continuous)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2009_10400_b200 import meshgen

# unit-volume tetrahedron (|det| / 6 = 1)
TET = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 6]], float)
TET_EL = np.array([[0, 1, 2, 3]])


def test_spec_single_tet_fraction():  # ((70-60)/(70-50))^3 = 0.125, < 1e-12
    v, n = O.ablation_volume("T4", TET, TET_EL, [70, 50, 50, 50], 60.0)
    assert abs(v - 0.125) <= 1e-12 * 0.125 and n == 1


@pytest.mark.parametrize("kind", ["T4", "H8"])
def test_spec_uniform_fields(kind):
    nodes, el = meshgen.structured_h8(3, 0.3) if kind == "H8" else meshgen.kuhn_t4(3, 0.3)
    v70, n70 = O.ablation_volume(kind, nodes, el, np.full(len(nodes), 70.0), 60.0)
    v37, n37 = O.ablation_volume(kind, nodes, el, np.full(len(nodes), 37.0), 60.0)
    assert abs(v70 - 0.027) <= 1e-12 * 0.027 and n70 == len(el)
    assert v37 == 0.0 and n37 == 0


@pytest.mark.parametrize("vals,frac", [
    ([70, 70, 50, 50], 0.5),                 # 2-2 split at mid-edges: half by symmetry
    ([70, 70, 70, 50], 1 - 0.125),           # 3-1: complement of the corner tetrahedron
    ([60, 50, 50, 50], 0.0),                 # touching the threshold at one node
    ([60, 60, 60, 60], 1.0),                 # >= threshold counts as inside
    ([80, 40, 40, 40], (20 / 40) ** 3),
])
def test_clipping_cases(vals, frac):
    v, _ = O.ablation_volume("T4", TET, TET_EL, vals, 60.0)
    assert abs(v - frac) <= 1e-12


def test_two_two_split_matches_integration():
    """2-2 wedge formula against a Monte-Carlo-free exact check: the above-region volume
    of a linear field on the tet equals the integral of the indicator, computed by
    refining the tet 64x (Kuhn) and clipping each child (children are exact for a
    linear field, so the sums must agree to rounding)."""
    rng = np.random.default_rng(3)
    for _ in range(20):
        vals = np.array([rng.uniform(60, 90), rng.uniform(60, 90), rng.uniform(30, 60), rng.uniform(30, 60)])
        v1, _ = O.ablation_volume("T4", TET, TET_EL, vals, 60.0)
        # same field on 8 children by midpoint subdivision (Freudenthal): linear field -> exact
        P = TET
        mids = {}
        pts = [P[i] for i in range(4)]
        T = list(vals)

        def mid(i, j):
            k = (min(i, j), max(i, j))
            if k not in mids:
                mids[k] = len(pts)
                pts.append(0.5 * (pts[i] + pts[j]))
                T.append(0.5 * (T[i] + T[j]))
            return mids[k]
        m01, m02, m03, m12, m13, m23 = mid(0, 1), mid(0, 2), mid(0, 3), mid(1, 2), mid(1, 3), mid(2, 3)
        children = [[0, m01, m02, m03], [m01, 1, m12, m13], [m02, m12, 2, m23], [m03, m13, m23, 3],
                    [m01, m02, m03, m13], [m01, m02, m12, m13], [m02, m03, m13, m23], [m02, m12, m13, m23]]
        v8, _ = O.ablation_volume("T4", np.array(pts), np.array(children), np.array(T), 60.0)
        assert abs(v1 - v8) <= 1e-12, (vals, v1, v8)


def test_h8_linear_field_is_exact():
    """A field linear in x is linear on every one of the 6 tetrahedra: the clipped volume
    of the unit cube is exactly the slab x >= x*."""
    nodes, el = meshgen.structured_h8(4, 1.0)
    T = 50.0 + 20.0 * nodes[:, 0]
    for thr, expect in [(60.0, 0.5), (55.0, 0.75), (66.0, 0.2)]:
        v, _ = O.ablation_volume("H8", nodes, el, T, thr)
        assert abs(v - expect) <= 1e-12


def test_deformed_configuration():  # SPEC.md:439 (X + u)
    nodes, el = meshgen.kuhn_t4(3, 0.3)
    T = np.full(len(nodes), 70.0)
    u = 0.1 * nodes  # uniform stretch 1.1
    v, _ = O.ablation_volume("T4", nodes, el, T, 60.0, disp=u)
    assert abs(v - 0.027 * 1.1 ** 3) <= 1e-12 * 0.027


def test_monotone_and_continuous_in_threshold():
    nodes, el = meshgen.structured_h8(5, 0.05)
    c = nodes - 0.025
    T = 37.0 + 50.0 * np.exp(-np.sum(c * c, axis=1) / (2 * 0.01 ** 2))
    thr = np.linspace(40, 85, 46)
    vols = [O.ablation_volume("H8", nodes, el, T, t)[0] for t in thr]
    assert all(a >= b for a, b in zip(vols, vols[1:]))
    for t in (47.3, 61.1, 72.9):  # away from nodal values: no jump under 1e-9 perturbation
        a = O.ablation_volume("H8", nodes, el, T, t - 1e-9)[0]
        b = O.ablation_volume("H8", nodes, el, T, t + 1e-9)[0]
        assert abs(a - b) <= 1e-6 * max(a, 1e-30)
