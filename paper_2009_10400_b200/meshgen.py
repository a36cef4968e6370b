"""Synthetic mesh generators.

The reference's ``run_bench`` generates structured cube meshes
(engine.hpp:155-159); the CT-derived liver mesh of the paper is
unavailable, so a liver-shaped two-ellipsoid T4 mesh stands in for it.  All
generators are deterministic (fixed seeds) and vectorised so a 16M-element mesh
builds in seconds.
"""
from __future__ import annotations

import numpy as np

# Kuhn / Freudenthal subdivision: 6 tets per cube sharing the main diagonal.
# Each permutation (p0, p1, p2) of the axes gives the path v0 -> +e_p0 -> +e_p1 -> +e_p2 = v7.
_PERMS = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]


def _corner(offs):
    return offs[0] + 2 * offs[1] + 4 * offs[2]  # bit-coded cube corner


def _kuhn_local():
    """(6, 4) cube-corner codes (x + 2y + 4z), each tet positively oriented."""
    tets = []
    for p in _PERMS:
        c = [0, 0, 0]
        verts = [tuple(c)]
        for ax in p:
            c[ax] = 1
            verts.append(tuple(c))
        X = np.array(verts, float)
        J = np.stack([X[1] - X[0], X[2] - X[0], X[3] - X[0]], axis=1)
        if np.linalg.det(J) < 0:
            verts[1], verts[2] = verts[2], verts[1]
        tets.append([_corner(v) for v in verts])
    return np.array(tets, np.int64)


def structured_h8(n: int, length: float = 1.0, nx=None, ny=None, nz=None):
    """n^3 (or nx*ny*nz) H8 cells on [0,length]^3 (cubic cells).  Node (i,j,k) id =
    i + (nx+1)(j + (ny+1)k); standard brick ordering."""
    nx = nx or n
    ny = ny or n
    nz = nz or n
    h = length / n
    i, j, k = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1), np.arange(nz + 1), indexing="ij")
    nodes = np.stack([i.ravel(order="F"), j.ravel(order="F"), k.ravel(order="F")], axis=1).astype(np.float64) * h
    ci, cj, ck = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    ci, cj, ck = ci.ravel(order="F"), cj.ravel(order="F"), ck.ravel(order="F")

    def nid(a, b, c):
        return a + (nx + 1) * (b + (ny + 1) * c)

    el = np.stack([nid(ci, cj, ck), nid(ci + 1, cj, ck), nid(ci + 1, cj + 1, ck), nid(ci, cj + 1, ck),
                   nid(ci, cj, ck + 1), nid(ci + 1, cj, ck + 1), nid(ci + 1, cj + 1, ck + 1),
                   nid(ci, cj + 1, ck + 1)], axis=1).astype(np.int32)
    return nodes, el


def kuhn_t4(n: int, length: float = 1.0):
    """n^3 cubes x 6 Kuhn tets on [0,length]^3; nodes numbered like structured_h8."""
    nodes, _ = structured_h8(n, length)
    ci, cj, ck = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    ci, cj, ck = ci.ravel(order="F"), cj.ravel(order="F"), ck.ravel(order="F")
    loc = _kuhn_local()
    dx, dy, dz = loc & 1, (loc >> 1) & 1, (loc >> 2) & 1
    el = ((ci[:, None, None] + dx[None]) + (n + 1) * ((cj[:, None, None] + dy[None]) +
                                                       (n + 1) * (ck[:, None, None] + dz[None])))
    return nodes, el.reshape(-1, 4).astype(np.int32)


def tet_volumes(nodes, el):
    X = nodes[el]
    J = np.stack([X[:, 1] - X[:, 0], X[:, 2] - X[:, 0], X[:, 3] - X[:, 0]], axis=2)
    return np.linalg.det(J) / 6.0


def _in_liver(p):
    e1 = ((p[..., 0] / 0.080) ** 2 + (p[..., 1] / 0.055) ** 2 + (p[..., 2] / 0.045) ** 2) <= 1.0
    q = p - np.array([-0.055, 0.025, 0.005])
    e2 = ((q[..., 0] / 0.045) ** 2 + (q[..., 1] / 0.040) ** 2 + (q[..., 2] / 0.035) ** 2) <= 1.0
    return e1 | e2


def _liver_cells(h):
    lo = np.array([-0.100, -0.060, -0.050])
    hi = np.array([0.085, 0.070, 0.050])
    n = np.ceil((hi - lo) / h).astype(int)
    ci, cj, ck = np.meshgrid(np.arange(n[0]), np.arange(n[1]), np.arange(n[2]), indexing="ij")
    cells = np.stack([ci.ravel(), cj.ravel(), ck.ravel()], axis=1)
    cen = lo + (cells + 0.5) * h
    keep = _in_liver(cen)
    return lo, n, cells[keep]


def liver_t4(target_elements: int = 100_000, seed: int = 2009104003, jitter: float = 0.15):
    """Liver-shaped T4 mesh: union of two ellipsoids, Kuhn cells
    whose centroid is inside, h bisected so E = target +-2%, interior nodes jittered."""
    lo_h, hi_h = 1e-3, 2e-2
    for _ in range(60):
        h = 0.5 * (lo_h + hi_h)
        _, _, cells = _liver_cells(h)
        E = 6 * len(cells)
        if abs(E - target_elements) <= 0.02 * target_elements:
            break
        if E > target_elements:
            lo_h = h
        else:
            hi_h = h
    lo, n, cells = _liver_cells(h)
    loc = _kuhn_local()
    dx, dy, dz = loc & 1, (loc >> 1) & 1, (loc >> 2) & 1
    gid = lambda i, j, k: i + (n[0] + 1) * (j + (n[1] + 1) * k)  # noqa: E731
    el = gid(cells[:, 0, None, None] + dx[None], cells[:, 1, None, None] + dy[None],
             cells[:, 2, None, None] + dz[None]).reshape(-1, 4)
    used, inv = np.unique(el.ravel(), return_inverse=True)   # drop orphans, renumber ascending
    el = inv.reshape(-1, 4).astype(np.int32)
    gi = used % (n[0] + 1)
    gj = (used // (n[0] + 1)) % (n[1] + 1)
    gk = used // ((n[0] + 1) * (n[1] + 1))
    nodes = lo + np.stack([gi, gj, gk], axis=1) * h
    # interior nodes: all 8 surrounding cells kept
    cellset = set(map(tuple, cells.tolist()))
    interior = np.ones(len(nodes), bool)
    for ox in (0, 1):
        for oy in (0, 1):
            for oz in (0, 1):
                cc = np.stack([gi - ox, gj - oy, gk - oz], axis=1)
                interior &= np.array([tuple(c) in cellset for c in cc.tolist()])
    rng = np.random.default_rng(seed)
    jit = rng.uniform(-jitter * h, jitter * h, size=(len(nodes), 3))
    jit[~interior] = 0.0
    scale = np.ones(len(nodes))
    for _ in range(30):
        X = nodes + jit * scale[:, None]
        bad = tet_volumes(X, el) <= 0
        if not bad.any():
            break
        scale[np.unique(el[bad].ravel())] *= 0.5
    nodes = nodes + jit * scale[:, None]
    assert (tet_volumes(nodes, el) > 0).all()
    return nodes, el, h


def centroids(nodes, el):
    return nodes[el].mean(axis=1)


def elements_in_sphere(nodes, el, center, diameter):
    c = centroids(nodes, el)
    return np.nonzero(np.linalg.norm(c - np.asarray(center), axis=1) <= 0.5 * diameter)[0].astype(np.int32)
