"""Multi-process (world_size 2 and 4, gloo on CPU) run of the multi-GPU halo protocol.

Each process plays one rank exactly as the NCCL path does: it builds its own RCB
partition plan through the product library (host-only, no GPU), fills its local
slot buffer with the element contributions of the elements it owns (here: the
oracle's real thermal loads and internal forces of the global problem), packs its
send lists, exchanges them with its neighbours (dist.isend/irecv; NCCL
ncclSend/ncclRecv on the GPU), and assembles every local node through its gather
list (local slots + receive area) in canonical order.  The per-node sums must be
bit-identical to the single-rank assembly: the precondition for results at P GPUs
to equal 1 GPU.

transport "peer" plays the peer-memory halo instead (engine.cu peer_attach, kernels.cuh
peer_send): the ranks all-gather their descriptors (neighbour list, receive segment
offsets — what tvegpu_peer_export publishes besides the IPC handles), each rank derives
for every send-list entry the destination index in the neighbour's receive area by the
same rule as peer_attach (recv_off'[j'] + position in the segment), and "stores" its
contributions there (here: (index, value) pairs over gloo, scattered by the receiver).
Every receive slot must be written exactly once and the node sums must again be
bit-identical to one rank.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _peer_destinations(pl, descs, rank):
    """engine.cu peer_attach: per neighbour j, the receive-area index of each send entry."""
    out = []
    for j, r in enumerate(pl["neighbors"]):
        d = descs[int(r)]
        jj = list(d["neighbors"]).index(rank)
        a, b = int(pl["send_offsets"][j]), int(pl["send_offsets"][j + 1])
        assert d["recv_offsets"][jj + 1] - d["recv_offsets"][jj] == b - a, "halo size"
        out.append(np.arange(b - a, dtype=np.int64) + int(d["recv_offsets"][jj]))
    return out


def _worker(rank, world, port, result_q, transport="sendrecv"):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch

    import paper_2009_10400_b200 as tg
    from oracle import oracle as O
    from paper_2009_10400_b200 import configs
    from paper_2009_10400_b200.problem import H8

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        p = configs.small_problem(kind=H8, n=6, steps=5)
        o = O.OracleEngine(p, workers=1)
        o.step(3)
        d = o.diagnostics()
        nn = p.nn
        th = d["thermal_loads"].reshape(-1, nn)          # (E, nn) per original element
        fm = d["forces"].reshape(-1, nn, 3)               # (E, nn, 3)
        pl = tg.plan(p, world, rank)
        El = pl["num_elements"]
        if transport == "peer":
            mine = {"neighbors": np.asarray(pl["neighbors"]), "recv_offsets": np.asarray(pl["recv_offsets"])}
            descs = [None] * world
            dist.all_gather_object(descs, mine)
            dests = _peer_destinations(pl, descs, rank)
        for width, contrib in ((1, th[..., None]), (3, fm)):
            local = contrib[pl["element_orig"]].reshape(El * nn, width)
            sendbuf = local[pl["send_slots"]]
            nrecv = int(pl["recv_offsets"][-1])
            recv = np.zeros((nrecv, width))
            if transport == "peer":
                # each sender "stores" at the indices it derived; the receiver only scatters
                reqs, bufs = [], []
                for j, s in enumerate(pl["neighbors"]):
                    a, b = pl["send_offsets"][j], pl["send_offsets"][j + 1]
                    reqs.append(dist.isend(torch.from_numpy(dests[j]), int(s)))
                    reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(sendbuf[a:b])), int(s)))
                    n = int(pl["recv_offsets"][j + 1] - pl["recv_offsets"][j])
                    ri, rv = torch.zeros(n, dtype=torch.int64), torch.zeros((n, width), dtype=torch.float64)
                    bufs.append((ri, rv))
                    reqs.append(dist.irecv(ri, int(s)))
                    reqs.append(dist.irecv(rv, int(s)))
                for q in reqs:
                    q.wait()
                hits = np.zeros(nrecv, np.int64)
                for ri, rv in bufs:
                    recv[ri.numpy()] = rv.numpy()
                    np.add.at(hits, ri.numpy(), 1)
                if not np.all(hits == 1):
                    raise AssertionError(f"rank {rank}: receive slots written {hits.min()}..{hits.max()} times")
            else:
                reqs, bufs = [], []
                for j, s in enumerate(pl["neighbors"]):
                    a, b = pl["send_offsets"][j], pl["send_offsets"][j + 1]
                    t = torch.from_numpy(np.ascontiguousarray(sendbuf[a:b]))
                    reqs.append(dist.isend(t, int(s)))
                    ra, rb = pl["recv_offsets"][j], pl["recv_offsets"][j + 1]
                    r = torch.zeros((int(rb - ra), width), dtype=torch.float64)
                    bufs.append((ra, rb, r))
                    reqs.append(dist.irecv(r, int(s)))
                for q in reqs:
                    q.wait()
                for ra, rb, r in bufs:
                    recv[ra:rb] = r.numpy()
            slots = np.concatenate([local, recv])
            off, idx = pl["csr_offsets"], pl["csr_slots"]
            sums = np.zeros((pl["num_nodes"], width))
            for li in range(pl["num_nodes"]):
                acc = np.zeros(width)
                for k in range(off[li], off[li + 1]):
                    acc = acc + slots[idx[k]]
                sums[li] = acc
            # single-rank reference: canonical assembly over the whole mesh
            one = tg.plan(p, 1, 0)
            loc1 = contrib[one["element_orig"]].reshape(-1, width)
            ref = {}
            for li, i in enumerate(one["node_orig"]):
                acc = np.zeros(width)
                for k in range(one["csr_offsets"][li], one["csr_offsets"][li + 1]):
                    acc = acc + loc1[one["csr_slots"][k]]
                ref[int(i)] = acc
            for li, i in enumerate(pl["node_orig"]):
                if not np.array_equal(sums[li], ref[int(i)]):
                    raise AssertionError(f"rank {rank}: node {i} width {width} differs")
        result_q.put((rank, "ok", int(pl["num_nodes"]), len(pl["neighbors"])))
    except Exception as e:  # report to the parent instead of hanging it
        result_q.put((rank, f"error: {e!r}", 0, 0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("transport", ["sendrecv", "peer"])
@pytest.mark.parametrize("world", [2, 4])
def test_halo_protocol_gloo(world, transport):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, transport)) for r in range(world)]
    for pr in procs:
        pr.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    assert all(r[1] == "ok" for r in results), results
    assert all(r[3] >= 1 for r in results)  # every rank has at least one neighbour
