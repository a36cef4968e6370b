"""The multi-GPU step code on one GPU: RCB partitions stepped by
enqueue_partitioned_step, CUDA-graph capture of all partitions' streams, agreement on
the first failure and the device state gather of checkpoints, with both halo paths:

- HALO_PEER (default): the boundary chunks run as SEND launches of the element kernels,
  which store each interface contribution straight into the neighbours' receive areas
  and raise per-phase flags there; the node kernels wait for the flags on the device
  (kernels.cuh peer_send / peer_signal / peer_wait) — the same kernels and tables a
  partition per GPU runs over NVLink peer memory, here with the other partitions'
  buffers as the "peer" memory (plus events ordering each node kernel after its
  neighbours' SEND launches, so no waiting kernel can starve a sender of SMs);
- HALO_NCCL: halo pack + ev_pack, the exchange on each partition's comm stream ending in
  ev_comm, the node kernels after ev_comm — with a device copy of each neighbour's
  packed segment instead of ncclSend/ncclRecv (engine.cu LoopbackTransport vs
  NcclTransport).

Partition invariance is bit-exact by construction (canonical gather order over
replicated nodes, node constants built once on the global mesh; engine.hpp:80-82
determinism claim), so every comparison here is array_equal.
"""
import numpy as np
import pytest

import paper_2009_10400_b200 as tg
from paper_2009_10400_b200 import configs
from paper_2009_10400_b200.engine import PartitionGroup
from paper_2009_10400_b200.problem import COUPLED, H8, MECHANICAL_ONLY, T4, THERMAL_ONLY

pytestmark = pytest.mark.gpu
FIELDS = ("T", "u", "u_prev", "viscous")


def assert_same(a, b, keys=FIELDS):
    for k in keys:
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)
    assert a["time"] == b["time"] and a["step"] == b["step"]


HALOS = [pytest.param(tg.HALO_PEER, id="peer"), pytest.param(tg.HALO_NCCL, id="nccl")]


@pytest.mark.parametrize("kind,n", [(H8, 6), (T4, 5)])
@pytest.mark.parametrize("nparts", [2, 3, 4, 8])
@pytest.mark.parametrize("spg", [7, 64])
@pytest.mark.parametrize("halo", HALOS)
def test_partitioned_step_bit_identical(kind, n, nparts, spg, halo):
    """P partitions (graph chunks of 7 or 64 steps, so several replays plus direct
    remainders) reproduce the single-partition state bit for bit."""
    steps = 150
    p = configs.small_problem(kind=kind, n=n, steps=steps)
    one = tg.Engine(p)
    one.step(steps)
    grp = PartitionGroup(p, nparts, steps_per_graph=spg, halo_transport=halo)
    grp.step(3)  # plain steps first, then graph replays
    grp.step(steps - 3)
    assert_same(one.state(), grp.state())


@pytest.mark.parametrize("mode", [THERMAL_ONLY, MECHANICAL_ONLY])
@pytest.mark.parametrize("halo", HALOS)
def test_partitioned_modes(mode, halo):
    p = configs.small_problem(kind=H8, n=5, steps=80)
    p.mode = mode
    one = tg.Engine(p)
    one.step(80)
    grp = PartitionGroup(p, 4, steps_per_graph=16, halo_transport=halo)
    grp.step(80)
    assert_same(one.state(), grp.state())


def test_partitioned_source_windows():
    """Source windows switching mid-run split the graph chunks on every partition alike."""
    p = configs.small_problem(kind=T4, n=5, steps=100)
    p.sources[0].t_start, p.sources[0].t_end = 9.5 * p.dt, 61.5 * p.dt
    one = tg.Engine(p)
    one.step(100)
    grp = PartitionGroup(p, 3, steps_per_graph=16)
    grp.step(100)
    assert_same(one.state(), grp.state())


@pytest.mark.parametrize("kind", [T4, H8])
@pytest.mark.parametrize("mode", [COUPLED, THERMAL_ONLY])
def test_partitioned_step_io(kind, mode):
    """tvegpu_group_step_io == the single engine's tvegpu_step_io, bit for bit, for a
    changing source schedule (the partitioned form a NCCL rank runs)."""
    p = configs.small_problem(kind=kind, n=4, steps=60)
    p.mode = mode
    a = tg.Engine(p)
    g = PartitionGroup(p, 4, steps_per_graph=8)
    rng = np.random.default_rng(3)
    Ta, ua = np.empty(p.num_nodes), np.empty(3 * p.num_nodes)
    Tg, ug = np.empty(p.num_nodes), np.empty(3 * p.num_nodes)
    for n in (1, 2, 17):
        q = rng.uniform(0, 2e-3, p.num_nodes)
        a.step_io(q, n, Ta, ua)
        g.step_io(q, n, Tg, ug)
        np.testing.assert_array_equal(Ta, Tg)
        np.testing.assert_array_equal(ua, ug)
    assert_same(a.state(), g.state())


def test_partitioned_checkpoint_round_trip():
    """SPEC.md:386/395 across partition counts: save from 4 partitions (device gather +
    all-reduce through the transport), load into 2 partitions and into one engine, run
    on; all bit-identical to the uninterrupted single-partition run.  The image itself
    equals the one a single-partition engine writes, byte for byte."""
    p = configs.small_problem(kind=H8, n=6, steps=60)
    ref = tg.Engine(p)
    ref.step(25)
    g4 = PartitionGroup(p, 4, steps_per_graph=8)
    g4.step(25)
    q = np.random.default_rng(4).uniform(0, 1e-3, p.num_nodes)  # with a source override in the image
    ref.set_nodal_sources(q)
    g4.set_nodal_sources(q)
    img = g4.save_checkpoint()
    assert img == ref.save_checkpoint()
    ref.step(35)
    g2 = PartitionGroup(p, 2, steps_per_graph=8)
    g2.load_checkpoint(img)
    g2.step(35)
    e1 = tg.Engine(p)
    e1.load_checkpoint(img)
    e1.step(35)
    assert_same(ref.state(), g2.state())
    assert_same(ref.state(), e1.state())
    # and back: the single engine's image loads into 4 partitions
    g4b = PartitionGroup(p, 4)
    g4b.load_checkpoint(e1.save_checkpoint())
    assert_same(e1.state(), g4b.state())


@pytest.mark.parametrize("kind", [T4, H8])
@pytest.mark.parametrize("halo", HALOS)
def test_partitioned_failure_is_collective(kind, halo):
    """A NaN injected into one node (held by one or several partitions): every partition
    reports the same InstabilityError (step, node) as the single engine, the group's
    state is then refused until set_state, and after a reset the group runs on bit-
    identically to the single engine (ADVICE: the halt must not leave partitions at
    different steps silently)."""
    p = configs.small_problem(kind=kind, n=5, steps=40)
    p.expansion_enabled = False  # the NaN would reach F_ther and be reported as an element error instead
    one = tg.Engine(p)
    grp = PartitionGroup(p, 4, steps_per_graph=4, halo_transport=halo)
    one.step(5)
    grp.step(5)
    s = one.state()
    T = s["T"].copy()
    T[p.num_nodes // 2] = np.nan
    for e in (one, grp):
        e.set_state(T, s["u"], s["u_prev"], s["viscous"], s["time"], s["step"])
    with pytest.raises(tg.InstabilityError) as e1:
        one.step(10)
    with pytest.raises(tg.InstabilityError) as eg:
        grp.step(10)
    assert (eg.value.step, eg.value.node) == (e1.value.step, e1.value.node)
    assert grp.step_count() == one.step_count() and grp.time() == one.time()
    with pytest.raises(tg.InstabilityError, match="invalid"):
        grp.state()
    with pytest.raises(tg.InstabilityError):  # halted until reset
        grp.step(1)
    s = one.state()
    s["T"][np.isnan(s["T"])] = 37.0
    for e in (one, grp):
        e.set_state(s["T"], s["u"], s["u_prev"], s["viscous"], s["time"], s["step"])
        e.step(7)
    assert_same(one.state(), grp.state())


@pytest.mark.slow
@pytest.mark.parametrize("nparts", [2, 8])
@pytest.mark.parametrize("halo", HALOS)
def test_cfg4_partitions_bit_identical(nparts, halo):
    """cfg4 (1M-element H8, the benchmark workload) at 200 steps: 2 and 8 partitions
    (multi-chunk boundary ordering, 128-element chunks on both sides of each cut)
    bit-identical to one partition."""
    p = configs.cfg4(steps=200)
    one = tg.Engine(p)
    one.step(200)
    a = one.state()
    one.close()
    grp = PartitionGroup(p, nparts, halo_transport=halo)
    grp.step(200)
    assert_same(a, grp.state())


def test_peer_halo_timeout_is_reported_not_hung():
    """Fault injection: partition 1 of 3 never raises its halo flags (TVEGPU_HALO_DROP_RANK).
    Its neighbours' node kernels give up after TVEGPU_HALO_TIMEOUT_MS instead of spinning
    forever, and every partition reports the same halo error; the state is then invalid
    until reset.  (On one device the waiting kernels are launched after the silent sender
    finished, so nothing ever waits on a kernel that is not running.)"""
    import os
    p = configs.small_problem(kind=H8, n=6, steps=10)
    os.environ["TVEGPU_HALO_DROP_RANK"] = "1"
    os.environ["TVEGPU_HALO_TIMEOUT_MS"] = "50"
    try:
        grp = PartitionGroup(p, 3, steps_per_graph=4)
    finally:
        del os.environ["TVEGPU_HALO_DROP_RANK"], os.environ["TVEGPU_HALO_TIMEOUT_MS"]
    with pytest.raises(tg.NcclError, match="halo exchange"):
        grp.step(2)
    with pytest.raises(tg.TveError):
        grp.state()


def test_peer_api_errors_and_solo_partition():
    """tvegpu_peer_export refuses a single-GPU engine; tvegpu_peer_attach needs one
    descriptor per rank; a partition created without an NCCL id can be stepped alone with
    tvegpu_peer_attach_solo (the per-rank timing hook) and then reports the peer path."""
    p = configs.small_problem(kind=H8, n=6, steps=10)
    one = tg.Engine(p)
    with pytest.raises(tg.TveError, match="not a partitioned engine"):
        one.peer_export()
    solo = tg.Engine(p, nranks=4, rank=1)
    blob = solo.peer_export()
    assert len(blob) > 0 and not solo.halo_peer
    with pytest.raises(tg.TveError, match="one descriptor per rank"):
        solo.peer_attach([blob])
    with pytest.raises(tg.TveError):  # stepping a partition without NCCL needs an attached halo
        solo.step(1)
    solo2 = tg.Engine(p, nranks=4, rank=2)
    solo2.peer_attach_solo()
    assert solo2.halo_peer and solo2.kernels_per_step() == 4
    solo2.step(5)  # its halo values are scratch: only that it runs is checked
    solo2.peer_detach()
    assert not solo2.halo_peer


@pytest.mark.parametrize("kind", [T4, H8])
@pytest.mark.parametrize("mode", [THERMAL_ONLY, MECHANICAL_ONLY])
def test_fp32_slots_partitioned_modes(kind, mode):
    """Mixed-precision mode x single-physics steps (the end-of-step acks of the peer path)
    x both element kinds: partitions stay bit-identical to one engine."""
    p = configs.small_problem(kind=kind, n=5, steps=60)
    p.mode = mode
    one = tg.Engine(p, slot_fp32=True)
    one.step(60)
    grp = PartitionGroup(p, 3, steps_per_graph=8, slot_fp32=True)
    grp.step(60)
    assert_same(one.state(), grp.state())


def test_long_tables_and_prony_partitioned():
    """Property tables longer than the launch-parameter copies and Prony terms beyond the
    staged history rows (read from device memory) under partitioning: bit-identical."""
    import math
    p = configs.small_problem(kind=H8, n=6, steps=60)
    p.prony_phi = [0.2, 0.15, 0.1, 0.08, 0.06, 0.05]
    p.prony_tau = [0.58, 0.058, 0.0058, 5.8, 0.0012, 0.021]
    Tc = np.linspace(36.99, 37.13, 20)
    p.c_table = [(float(t), 3600.0 + 700.0 * math.sin(9.0 * i)) for i, t in enumerate(Tc)]
    one = tg.Engine(p)
    one.step(60)
    for halo in (tg.HALO_PEER, tg.HALO_NCCL):
        grp = PartitionGroup(p, 4, steps_per_graph=16, halo_transport=halo)
        grp.step(60)
        assert_same(one.state(), grp.state())
