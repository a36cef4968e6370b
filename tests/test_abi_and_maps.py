"""CPU tests of the product library: it loads, exports every symbol the C header
declares, rejects what the reference rejects, and its integer maps (Morton /
first-touch order, canonical gather CSR, RCB partition, halo lists) agree
bit-exactly with an independent restatement (oracle/maps.py) and with the
oracle's own adjacency (mesh.hpp:58-61).  No GPU compute is called here."""
import os
import re

import numpy as np
import pytest

import paper_2009_10400_b200 as tg
from oracle import maps
from oracle import oracle as O
from paper_2009_10400_b200 import configs, meshgen
from paper_2009_10400_b200.problem import H8, T4

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "tvegpu.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tvegpu_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = tg.lib()
    syms = declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(tg.engine.EXPORTS), set(syms) ^ set(tg.engine.EXPORTS)
    assert L.tvegpu_abi_version() == 1
    assert L.tvegpu_status_string(3) == b"InstabilityError"


def test_engine_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(tg.CudaError):
        tg.Engine(configs.small_problem(kind=H8, n=2))


@pytest.mark.parametrize("kind", [T4, H8])
def test_critical_timestep_matches_oracle(kind):
    p = configs.small_problem(kind=kind, n=3)
    p.nodes = p.nodes + np.random.default_rng(0).uniform(-0.002, 0.002, p.nodes.shape)
    a = tg.critical_timestep(p)
    b = O.critical_timestep(p)
    assert a[1] == b[1]  # same formula, same min-edge
    assert a[0] == pytest.approx(b[0], rel=1e-13)  # eigenvalue solvers differ


def test_validation_errors_match_reference_cases():
    p = configs.small_problem(kind=T4, n=2)
    p.elements = p.elements.copy()
    p.elements[3, [1, 2]] = p.elements[3, [2, 1]]
    with pytest.raises(tg.ValidationError, match="element 4"):
        tg.plan(p)
    p = configs.small_problem(kind=T4, n=2)
    p.elements = p.elements.copy()
    p.elements[0, 0] = 10_000
    with pytest.raises(tg.ValidationError, match="element 1"):
        tg.plan(p)
    p = configs.small_problem(kind=H8, n=2)
    p.prony_phi, p.prony_tau = [0.7, 0.4], [1.0, 2.0]
    with pytest.raises(tg.ValidationError, match="Prony"):
        tg.plan(p)


def _check_plan(p, nranks, rank, reorder=True):
    a = tg.plan(p, nranks, rank, reorder)
    b = maps.rank_plan(p.nodes, p.elements.astype(np.int64), nranks, rank, reorder)
    for k in ("element_orig", "node_orig", "conn", "csr_offsets", "csr_slots", "element_owner", "neighbors",
              "send_offsets", "send_slots", "recv_offsets"):
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)
    assert a["num_boundary_elements"] == b["num_boundary_elements"]
    return a


@pytest.mark.parametrize("kind,n", [(T4, 3), (H8, 4)])
def test_single_rank_maps_bit_exact(kind, n):
    p = configs.small_problem(kind=kind, n=n)
    a = _check_plan(p, 1, 0)
    # gather list == the oracle's adjacency, mapped through the permutations
    pre = O.precompute(p)
    nn = p.nn
    for li, i in enumerate(a["node_orig"]):
        slots = a["csr_slots"][a["csr_offsets"][li]:a["csr_offsets"][li + 1]]
        got = [(a["element_orig"][s // nn], s % nn) for s in slots]
        off = pre["adj_offsets"]
        want = list(zip(pre["adj_elem"][off[i]:off[i + 1]], pre["adj_local"][off[i]:off[i + 1]]))
        assert got == want
    _check_plan(p, 1, 0, reorder=False)


def test_liver_maps_bit_exact():
    nodes, el, _ = meshgen.liver_t4(6000)
    p = configs.small_problem(kind=T4, n=2)
    p.nodes, p.elements = nodes, el
    _check_plan(p, 1, 0)


@pytest.mark.parametrize("nranks", [2, 3, 4, 8])
def test_partition_maps_bit_exact(nranks):
    p = configs.small_problem(kind=H8, n=6)
    plans = [_check_plan(p, nranks, r) for r in range(nranks)]
    owner = plans[0]["element_owner"]
    assert all((pl["element_owner"] == owner).all() for pl in plans)
    assert sorted(np.concatenate([pl["element_orig"] for pl in plans]).tolist()) == list(range(p.num_elements))
    counts = np.bincount(owner, minlength=nranks)
    assert counts.max() - counts.min() <= nranks  # RCB balance
    # every send list matches the peer's receive area, element by element
    nn = p.nn
    for r, pl in enumerate(plans):
        for j, s in enumerate(pl["neighbors"]):
            sent = pl["send_slots"][pl["send_offsets"][j]:pl["send_offsets"][j + 1]]
            sent_keys = [(pl["element_orig"][x // nn], x % nn) for x in sent]
            q = plans[s]
            jj = list(q["neighbors"]).index(r)
            assert q["recv_offsets"][jj + 1] - q["recv_offsets"][jj] == len(sent_keys)


def test_gather_sums_bit_identical_across_partitions():
    """Emulate the multi-GPU gather on the CPU: every rank sums its local slots and
    the slots received from its neighbours in its CSR order; node sums must equal
    the single-rank sums bit for bit."""
    p = configs.small_problem(kind=H8, n=5)
    nn, E = p.nn, p.num_elements
    rng = np.random.default_rng(3)
    contrib = rng.normal(size=(E, nn))  # per (original element, local) contributions
    one = tg.plan(p, 1, 0)
    ref = {}
    for li, i in enumerate(one["node_orig"]):
        s = 0.0
        for sl in one["csr_slots"][one["csr_offsets"][li]:one["csr_offsets"][li + 1]]:
            s += contrib[one["element_orig"][sl // nn], sl % nn]
        ref[i] = s
    for nranks in (2, 4):
        plans = [tg.plan(p, nranks, r) for r in range(nranks)]
        for r, pl in enumerate(plans):
            El = pl["num_elements"]
            local = contrib[pl["element_orig"]].reshape(-1)
            recv = np.zeros(int(pl["recv_offsets"][-1]))
            for j, s in enumerate(pl["neighbors"]):
                q = plans[s]
                jj = list(q["neighbors"]).index(r)
                sent = q["send_slots"][q["send_offsets"][jj]:q["send_offsets"][jj + 1]]
                recv[pl["recv_offsets"][j]:pl["recv_offsets"][j + 1]] = contrib[q["element_orig"][sent // nn],
                                                                                sent % nn]
            slots = np.concatenate([local, recv])
            assert slots.size == El * nn + recv.size
            for li, i in enumerate(pl["node_orig"]):
                s = 0.0
                for sl in pl["csr_slots"][pl["csr_offsets"][li]:pl["csr_offsets"][li + 1]]:
                    s += slots[sl]
                assert s == ref[i]
