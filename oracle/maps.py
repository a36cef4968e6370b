"""Independent numpy restatement of the integer maps of the device layout.

TEST INFRASTRUCTURE ONLY.  The reference defines only the canonical node ->
(element, local) adjacency (ascending element, then local; mesh.hpp:58-61).
The Morton element order, first-touch node order, RCB partition and halo lists
are this build's own design; they are restated here from their
written definition so tests can demand bit-exact agreement with the C++
planner (paper_2009_10400_b200/csrc/plan.cpp).
"""
from __future__ import annotations

import numpy as np


def centroids(nodes, el):
    nn = el.shape[1]
    s = np.zeros((el.shape[0], 3))
    for a in range(nn):  # sequential sum, then divide (matches the C++ loop order)
        s = s + nodes[el[:, a]]
    return s / nn


def _spread21(v):
    v = v.astype(np.uint64) & np.uint64(0x1FFFFF)
    v = (v | (v << np.uint64(32))) & np.uint64(0x1F00000000FFFF)
    v = (v | (v << np.uint64(16))) & np.uint64(0x1F0000FF0000FF)
    v = (v | (v << np.uint64(8))) & np.uint64(0x100F00F00F00F00F)
    v = (v | (v << np.uint64(4))) & np.uint64(0x10C30C30C30C30C3)
    v = (v | (v << np.uint64(2))) & np.uint64(0x1249249249249249)
    return v


_T4E = [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]
_H8E = [(0, 1), (1, 2), (2, 3), (3, 0), (4, 5), (5, 6), (6, 7), (7, 4), (0, 4), (1, 5), (2, 6), (3, 7)]


def min_edge(nodes, el):
    edges = _T4E if el.shape[1] == 4 else _H8E
    L = np.inf
    for a, b in edges:
        d = nodes[el[:, a]] - nodes[el[:, b]]
        d2 = d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1] + d[:, 2] * d[:, 2]  # same summation order as C++
        L = min(L, float(np.sqrt(d2).min()))
    return L


def morton_scale(c, lo, hi, lmin):
    ext = float((hi - lo).max())
    s = 1.0 / lmin if lmin > 0 else 0.0
    if ext > 0 and ext * s > 2097151.0:
        s = 2097151.0 / ext
    return s


def morton_keys(c, lo, scale):
    """round((c - lo) * scale) per axis on the element lattice, 21 bits each, bit-interleaved."""
    q = []
    for k in range(3):
        v = np.floor((c[:, k] - lo[k]) * scale + 0.5)
        v = np.clip(v, 0.0, 2097151.0)
        q.append(v.astype(np.uint64))
    return _spread21(q[0]) | (_spread21(q[1]) << np.uint64(1)) | (_spread21(q[2]) << np.uint64(2))


def rcb(c, nranks):
    owner = np.zeros(c.shape[0], np.int32)

    def rec(ids, parts, first):
        if parts == 1:
            owner[ids] = first
            return
        sub = c[ids]
        ext = sub.max(axis=0) - sub.min(axis=0)
        ax = int(np.argmax(ext))  # first axis on ties
        left = parts // 2
        nl = (len(ids) * left) // parts
        order = np.lexsort((ids, sub[:, ax]))
        rec(np.sort(ids[order[:nl]]), left, first)
        rec(np.sort(ids[order[nl:]]), parts - left, first + left)

    rec(np.arange(c.shape[0]), nranks, 0)
    return owner


def adjacency(el, N):
    """Canonical CSR (mesh.hpp:58-61): per node, (element, local) ascending."""
    E, nn = el.shape
    flat = el.reshape(-1)
    order = np.argsort(flat, kind="stable")  # flat index e*nn + a is already (e, a)-ascending
    off = np.zeros(N + 1, np.int64)
    np.add.at(off, flat + 1, 1)
    off = np.cumsum(off)
    return off, order // nn, order % nn


def rank_plan(nodes, el, nranks=1, rank=0, reorder=True):
    E, nn = el.shape
    N = nodes.shape[0]
    c = centroids(nodes, el)
    lo, hi = c.min(axis=0), c.max(axis=0)
    owner = rcb(c, nranks) if nranks > 1 else np.zeros(E, np.int32)
    touch = np.zeros(N, np.uint64)
    for a in range(nn):
        np.bitwise_or.at(touch, el[:, a], (np.uint64(1) << owner.astype(np.uint64)))
    me = np.uint64(1) << np.uint64(rank)
    mine = np.nonzero(owner == rank)[0]
    shared_other = (touch[el[mine]] & ~me) != 0
    bnd = mine[shared_other.any(axis=1)]
    inr = mine[~shared_other.any(axis=1)]
    if reorder:
        # lattice origin: the partition's own lowest centroid (plan.cpp build_rank_plan)
        klo = c[mine].min(axis=0) if nranks > 1 and len(mine) else lo
        keys = morton_keys(c, klo, morton_scale(c, lo, hi, min_edge(nodes, el)))
        bnd = bnd[np.lexsort((bnd, keys[bnd]))]
        inr = inr[np.lexsort((inr, keys[inr]))]
        if len(bnd) % 2 == 1 and len(inr):  # even chunk starts (plan.cpp: aligned element rows)
            bnd, inr = np.append(bnd, inr[0]), inr[1:]
        elem_orig = np.concatenate([bnd, inr]).astype(np.int32)
        seen = np.full(N, -1, np.int64)
        node_orig = []
        for i in el[elem_orig].reshape(-1):
            if seen[i] < 0:
                seen[i] = len(node_orig)
                node_orig.append(i)
        node_orig = np.array(node_orig, np.int32)
    else:
        elem_orig = np.arange(E, dtype=np.int32)
        node_orig = np.arange(N, dtype=np.int32)
    local = np.full(N, -1, np.int64)
    local[node_orig] = np.arange(len(node_orig))
    elem_local = np.full(E, -1, np.int64)
    elem_local[elem_orig] = np.arange(len(elem_orig))
    conn = local[el[elem_orig]].astype(np.int32)
    off, ae, al = adjacency(el, N)
    # halo: contributions (e, a) of elements owned by r to nodes shared with s, canonical order
    neighbors, send, recv = [], [], []
    for s in range(nranks):
        if s == rank:
            continue
        sbit = np.uint64(1) << np.uint64(s)
        both = (touch & me != 0) & (touch & sbit != 0)
        mask_nodes = both[el]  # (E, nn)
        send_s = [(e, a) for e, a in zip(*np.nonzero(mask_nodes & (owner == rank)[:, None]))]
        recv_s = [(e, a) for e, a in zip(*np.nonzero(mask_nodes & (owner == s)[:, None]))]
        if send_s or recv_s:
            neighbors.append(s)
            send.append(sorted(send_s))
            recv.append(sorted(recv_s))
    send_slots = [elem_local[e] * nn + a for lst in send for e, a in lst]
    send_off = np.cumsum([0] + [len(x) for x in send])
    recv_off = np.cumsum([0] + [len(x) for x in recv])
    recv_index = {}
    for j, lst in enumerate(recv):
        for k, key in enumerate(lst):
            recv_index[key] = recv_off[j] + k
    base = len(elem_orig) * nn
    csr_off = [0]
    csr = []
    for i in node_orig:
        for k in range(off[i], off[i + 1]):
            e, a = ae[k], al[k]
            csr.append(elem_local[e] * nn + a if owner[e] == rank else base + recv_index[(e, a)])
        csr_off.append(len(csr))
    return dict(element_orig=elem_orig, node_orig=node_orig, conn=conn, csr_offsets=np.array(csr_off, np.int32),
                csr_slots=np.array(csr, np.int32), num_boundary_elements=len(bnd), element_owner=owner,
                neighbors=np.array(neighbors, np.int32), send_offsets=np.array(send_off, np.int32),
                send_slots=np.array(send_slots, np.int32), recv_offsets=np.array(recv_off, np.int32))
