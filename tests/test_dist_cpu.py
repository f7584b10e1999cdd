"""Multi-rank host logic on CPU: world_size-2 (and 3) torch.distributed over gloo, 127.0.0.1.

Covers what the N>1 path does on the host: the process-group helpers used to bootstrap the
communicator and to reduce benchmark timings (paper_2406_08646_b200.dist), the per-rank input
recipe (every rank generates exactly its slab; the union is the global problem), and the halo
protocol of the distributed MatMult -- pack by the owner's root offsets, point-to-point
exchange, unpack into the ghost vector, y = A_d x + A_o lvec -- driven from the oracle's plan
over real process boundaries and compared with the single-process product.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(rank, world, port, fn, q):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn(rank, world)
        q.put((rank, "ok"))
    except Exception as e:  # noqa: BLE001
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def spawn(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    bad = {r: m for r, m in res.items() if m != "ok"}
    assert not bad, bad


# ------------------------------------------------------------------ workers
def w_helpers(rank, world):
    from paper_2406_08646_b200 import dist as sd
    assert sd.world() == (world, rank)
    offs = sd.layout(10 + rank)
    assert offs == [0] + list(np.cumsum([10 + r for r in range(world)]))
    assert sd.max_over_ranks(float(rank) * 1.5) == (world - 1) * 1.5
    assert sd.sum_over_ranks(rank + 1) == world * (world + 1) // 2
    uid = sd.share_unique_id(lambda: bytes(range(128)))
    assert uid == bytes(range(128))
    sd.barrier()


def w_partition(rank, world):
    import synth
    # stencil slab: each rank generates its own rows; union == global triplets
    shape = (6, 5, 4 * world)
    sizes = synth.slab_sizes(shape, world)
    off = synth.offsets_from_sizes(sizes)
    i, j, v = synth.stencil_coo(shape, 7, rows=(off[rank], off[rank + 1]), values="real")
    assert torch.all((i >= off[rank]) & (i < off[rank + 1]))
    trip = torch.stack([i.double(), j.double(), v], 1)
    n = torch.tensor([trip.shape[0]])
    ns = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(ns, n)
    mx = int(max(t.item() for t in ns))
    pad = torch.zeros(mx, 3, dtype=torch.float64)
    pad[:trip.shape[0]] = trip
    allt = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(allt, pad)
    got = torch.cat([t[:int(c.item())] for t, c in zip(allt, ns)])
    gi, gj, gv = synth.stencil_coo(shape, 7, values="real")
    want = torch.stack([gi.double(), gj.double(), gv], 1)
    assert torch.equal(got, want)
    # q1 element slabs cover every element exactly once
    n1 = 4 * world
    lo, hi = synth.q1_slab_elems(n1, world, rank)
    cnt = torch.tensor([hi - lo])
    dist.all_reduce(cnt)
    assert int(cnt.item()) == (n1 - 1) ** 3


def w_halo_protocol(rank, world):
    """Distributed MatMult driven by the oracle's plan across real processes (gloo p2p)."""
    import oracle
    import synth
    for kind in ("7pt", "q1", "random"):
        if kind == "7pt":
            shape = (7, 6, 3 * world)
            M = int(np.prod(shape))
            sizes = synth.slab_sizes(shape, world)
            off = synth.offsets_from_sizes(sizes)
            coo = [synth.stencil_coo(shape, 7, rows=(off[q], off[q + 1]), values="real") for q in range(world)]
            N, csz = M, sizes
        elif kind == "q1":
            n = 3 * world
            M = n ** 3
            sizes = synth.slab_sizes((n, n, n), world)
            coo = [synth.q1_coo(n, elems=synth.q1_slab_elems(n, world, q), values="real") for q in range(world)]
            N, csz = M, sizes
        else:
            M, N = 53, 61
            sizes = synth.split_sizes(M, world)
            csz = synth.split_sizes(N, world)
            coo = [synth.random_coo(M, N, 300, seed=7 + q, values="real") for q in range(world)]
        O = oracle.OracleMat(M, N, sizes, csz, [c[0] for c in coo], [c[1] for c in coo])
        O.set_values([c[2] for c in coo])
        x = synth.x_vector(0, N, "real").numpy()
        coff = synth.offsets_from_sizes(csz)
        xl = x[coff[rank]:coff[rank + 1]]
        # --- owner side: pack x by root offsets for every requester, send
        rc, ro = O.export(rank, "root_count"), O.export(rank, "root_offsets")
        reqs = []
        pos = 0
        for p in range(world):
            if rc[p] and p != rank:
                buf = torch.from_numpy(np.ascontiguousarray(xl[ro[pos:pos + rc[p]]]))
                reqs.append(dist.isend(buf, dst=p))
            pos += rc[p]
        # --- leaf side: receive per owner, unpack into lvec (REPLACE)
        lo_, lof = O.export(rank, "leaf_owner"), O.export(rank, "leaf_offset")
        lvec = np.zeros(lo_.size)
        for q in range(world):
            sel = np.nonzero(lo_ == q)[0]
            if sel.size and q != rank:
                buf = torch.zeros(sel.size, dtype=torch.float64)
                dist.recv(buf, src=q)
                lvec[sel] = buf.numpy()
        for r in reqs:
            r.wait()
        # --- local product in the oracle's order: y = S_d (+ S_o)
        rpd, cd, vd = O.export(rank, "rowptr_d"), O.export(rank, "col_d"), O.export(rank, "val_d")
        rpo, co, vo = O.export(rank, "rowptr_o"), O.export(rank, "col_o"), O.export(rank, "val_o")
        y = np.zeros(sizes[rank])
        for q in range(sizes[rank]):
            sd = 0.0
            for t in range(rpd[q], rpd[q + 1]):
                sd = sd + vd[t] * xl[cd[t]]
            if rpo[q + 1] > rpo[q]:
                so = 0.0
                for t in range(rpo[q], rpo[q + 1]):
                    so = so + vo[t] * lvec[co[t]]
                sd = sd + so
            y[q] = sd
        roff = synth.offsets_from_sizes(sizes)
        want = O.mult(x)[roff[rank]:roff[rank + 1]]
        assert np.array_equal(y, want), kind
        dist.barrier()


@pytest.mark.parametrize("world", [2, 3])
def test_dist_helpers(world):
    spawn(w_helpers, world)


def test_partition_union():
    spawn(w_partition, 2)


@pytest.mark.parametrize("world", [2, 3])
def test_halo_protocol_gloo(world):
    spawn(w_halo_protocol, world)
