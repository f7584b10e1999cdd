"""Multi-rank GPU parity (one process per GPU, NCCL).  Launched by tests/test_gpu_multirank.py:

    torchrun --nproc-per-node P --master-addr 127.0.0.1 tests/mp_gpu_parity.py

Every rank builds the oracle's in-process P-rank simulation of the same global problem and
checks ITS OWN part of the GPU result against it: CSR structure, colmap, contribution plan
(jmap, source ranks, source positions), COO send/receive plans, halo SF plan -- all
bit-exact -- assembled values bit-exact, and y (integer inputs bit-exact, real inputs within
1e-12 relative max-norm, and equal to the P=1 global product).
"""
import os
import sys
import traceback

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_2406_08646_b200 as sp  # noqa: E402
import synth  # noqa: E402

TOL = 1e-12


def canon(a):
    a = np.asarray(a, dtype=np.float64).copy()
    a[a == 0] = 0.0
    return a


def rel_err(y, ref):
    ref = np.asarray(ref)
    if ref.size == 0:
        return 0.0
    s = np.max(np.abs(ref))
    d = np.max(np.abs(np.asarray(y) - ref))
    return d / s if s > 0 else d


class Ctx:
    def __init__(self):
        self.P = dist.get_world_size()
        self.r = dist.get_rank()
        self.comm = sp.Comm()

    def log(self, *a):
        print(f"[rank {self.r}]", *a, flush=True)


def oracle_positions(O, r):
    """Oracle contribution list of rank r as (src, position-in-message-from-src or k)."""
    csrc, ck = O.export(r, "csrc"), O.export(r, "ck")
    pos = ck.copy()
    P = O.P
    for src in range(P):
        if src == r:
            continue
        sc = O.export(src, "send_count")
        sk = O.export(src, "send_k")
        start = int(np.sum(sc[:r]))
        seg = sk[start:start + sc[r]]
        where = {int(k): p for p, k in enumerate(seg)}
        m = csrc == src
        pos[m] = [where[int(k)] for k in ck[m]]
    return csrc, pos


def check_matrix(c, name, M, N, row_sizes, col_sizes, coo, values, x_global, exact_y, bs=1):
    """coo: list over ranks of (i, j, v) CPU tensors (every rank has all of them)."""
    P, r = c.P, c.r
    O = oracle.OracleMat(M, N, row_sizes, col_sizes, [t[0] for t in coo], [t[1] for t in coo])
    O.set_values([t[2] for t in coo])
    i, j, v = coo[r]
    A = sp.Mat(c.comm, row_sizes[r], col_sizes[r], M, N, i.cuda(), j.cuda())
    A.set_values(v.cuda())
    if bs > 1:
        A.set_block_size(bs)
    c.halo_mode = A.halo_mode()
    info = A.info()
    if bs == 3 and info["n_offdiag_rows"] > 0 and os.environ.get("SPMAT_BSR_OFFDIAG", "1") != "0":
        assert info["offdiag_3x3"] == 1, f"{name}: off-diagonal block not kept in 3x3 blocks"
    assert info["rstart"] == O.info(r, "rstart") and info["cstart"] == O.info(r, "cstart")
    for key in ("rowptr_d", "col_d", "rowptr_o", "col_o", "colmap", "jmap", "send_count",
                "recv_count", "send_k"):
        g, o = A.export(key), O.export(r, key)
        assert np.array_equal(g, o), f"{name}: {key} differs on rank {r}"
    osrc, opos = oracle_positions(O, r)
    assert np.array_equal(A.export("csrc"), osrc), f"{name}: contribution sources differ"
    assert np.array_equal(A.export("cpos"), opos), f"{name}: contribution positions differ"
    for key in ("val_d", "val_o"):
        assert np.array_equal(canon(A.export(key)), canon(O.export(r, key))), f"{name}: {key} differ"
    # halo SF plan; its own NVLink transport is built on first use when the MatMult halo has
    # its own NVLink path (halo_mode 2), right at create otherwise
    i_pre = A.info()
    if i_pre["halo_mode"] == 2:
        assert i_pre["halo_sf_transport"] == 0, f"{name}: halo SF transport built eagerly"
    hs = A.halo_sf()
    if P > 1:
        assert A.info()["halo_sf_transport"] in (1, 2), f"{name}: halo SF transport missing"
    lo, lof = O.export(r, "leaf_owner"), O.export(r, "leaf_offset")
    nbrs = [q for q in range(P) if np.any(lo == q)]
    assert list(sp.sf_export(hs, "recv_ranks")) == nbrs
    assert list(sp.sf_export(hs, "recv_counts")) == [int(np.sum(lo == q)) for q in nbrs]
    assert np.array_equal(sp.sf_export(hs, "leaf_idx"), np.concatenate(
        [np.nonzero(lo == q)[0] for q in nbrs]) if nbrs else np.zeros(0, np.int64))
    rc, ro = O.export(r, "root_count"), O.export(r, "root_offsets")
    req = [p for p in range(P) if rc[p] > 0]
    assert list(sp.sf_export(hs, "send_ranks")) == req
    assert list(sp.sf_export(hs, "send_counts")) == [int(rc[p]) for p in req]
    assert np.array_equal(sp.sf_export(hs, "root_idx"), ro)
    # MatMult
    off = np.concatenate([[0], np.cumsum(col_sizes)])
    roff = np.concatenate([[0], np.cumsum(row_sizes)])
    xl = torch.from_numpy(np.ascontiguousarray(x_global[off[r]:off[r + 1]])).cuda()
    y = torch.empty(row_sizes[r], dtype=torch.float64, device="cuda")
    A.mult(xl, y)
    torch.cuda.synchronize()
    yo = O.mult(x_global)[roff[r]:roff[r + 1]]
    yg = y.cpu().numpy()
    if exact_y:
        assert np.array_equal(canon(yg), canon(yo)), f"{name}: y not bit-exact on rank {r}"
    else:
        assert rel_err(yg, yo) <= TOL, f"{name}: y rel err {rel_err(yg, yo)}"
    # repeated MatMult and ADD re-assembly through the same plan
    A.set_values(v.cuda(), sp.ADD)
    A.mult(xl, y)
    O.set_values([t[2] for t in coo], oracle.ADD)
    yo2 = O.mult(x_global)[roff[r]:roff[r + 1]]
    assert rel_err(y.cpu().numpy(), yo2) <= TOL
    assert A.info()["plan_builds"] == 1
    # many back-to-back MatMults (exercises the halo epoch protocol), then check y again
    i0 = A.info()
    for _ in range(20):
        A.mult(xl, y)
    A.check()
    i1 = A.info()  # byte counters: 20 MatMults' halo (16 B lines over NVLink, 8 B over NCCL)
    assert i1["n_mult"] - i0["n_mult"] == 20
    nsend = sp.sf_get_info(A.halo_sf())["n_send"]
    if i1["halo_mode"] == 2:
        assert i1["nvlink_bytes_put"] - i0["nvlink_bytes_put"] == 20 * 16 * nsend, f"{name}: NVLink counter"
    elif i1["halo_mode"] == 1:
        assert i1["nccl_bytes_sent"] - i0["nccl_bytes_sent"] == 20 * 8 * nsend, f"{name}: NCCL counter"
    assert rel_err(y.cpu().numpy(), yo2) <= TOL
    A.close()
    return info, yg


def case_stencil(c, values):
    P = c.P
    shape = (12, 10, 4 * P)
    M = int(np.prod(shape))
    sizes = synth.slab_sizes(shape, P)
    off = synth.offsets_from_sizes(sizes)
    coo = [synth.stencil_coo(shape, 7, rows=(off[q], off[q + 1]), values=values) for q in range(P)]
    x = synth.x_vector(0, M, values).numpy()
    info, y = check_matrix(c, f"7pt-{values}", M, M, sizes, sizes, coo, values, x, exact_y=True)
    nb = (c.r > 0) + (c.r < P - 1)
    assert info["n_ghost"] == nb * 12 * 10
    # global vs partitioned (P7): the single-rank product of the same global matrix
    i1, j1, v1 = synth.stencil_coo(shape, 7, values=values)
    O1 = oracle.OracleMat(M, M, [M], [M], [i1], [j1])
    O1.set_values([v1])
    y1 = O1.mult(x)[off[c.r]:off[c.r + 1]]
    if values == "int":
        assert np.array_equal(canon(y), canon(y1))
    else:
        assert rel_err(y, y1) <= 1e-14


def case_q1(c, values):
    P = c.P
    n = 4 * P
    M = n ** 3
    sizes = synth.slab_sizes((n, n, n), P)
    coo = [synth.q1_coo(n, elems=synth.q1_slab_elems(n, P, q), variant="mass", values=values)
           for q in range(P)]
    x = synth.x_vector(0, M, values).numpy()
    info, _ = check_matrix(c, f"q1-{values}", M, M, sizes, sizes, coo, values, x,
                        exact_y=(values == "int"))
    if c.r < P - 1:
        assert info["n_send"] > 0
    if c.r > 0:
        assert info["n_mixed"] > 0


def case_box(c, npts, values):
    """Box (cube) decomposition with per-rank renumbering: strided owner
    faces (gathered by the halo puts / SF pack kernel), up to 26 neighbours."""
    P = c.P
    procs = synth.box_procs(P)
    shape = (8 * procs[0] + 1, 6 * procs[1], 5 * procs[2])
    sizes = synth.box_sizes(shape, procs)
    M = sum(sizes)
    coo = [synth.stencil_coo_box(shape, npts, procs, q, values=values) for q in range(P)]
    x = synth.x_vector(0, M, values).numpy()
    info, _ = check_matrix(c, f"box{npts}-{values}", M, M, sizes, sizes, coo, values, x,
                           exact_y=(values == "int"))
    assert info["n_ghost"] > 0


def case_elasticity(c):
    P = c.P
    n = 2 * P
    M = 3 * n ** 3
    sizes = synth.slab_sizes((n, n, n), P, dof=3)
    nodes = sizes[0] // 3
    coo = [synth.elasticity_coo(n, nodes=(q * nodes, (q + 1) * nodes), values="real") for q in range(P)]
    x = synth.x_vector(0, M, "real").numpy()
    check_matrix(c, "elasticity", M, M, sizes, sizes, coo, "real", x, exact_y=False)
    check_matrix(c, "elasticity-bsr", M, M, sizes, sizes, coo, "real", x, exact_y=False, bs=3)
    # larger slabs, integer values: the 3x3 off-diagonal kernel must be bit-exact
    n = 4 * P
    M = 3 * n ** 3
    sizes = synth.slab_sizes((n, n, n), P, dof=3)
    nodes = sizes[0] // 3
    coo = [synth.elasticity_coo(n, nodes=(q * nodes, (q + 1) * nodes), values="int") for q in range(P)]
    x = synth.x_vector(0, M, "int").numpy()
    check_matrix(c, "elasticity-bsr-int", M, M, sizes, sizes, coo, "int", x, exact_y=True, bs=3)


def case_random(c, seed):
    P = c.P
    rng = np.random.default_rng(seed)
    M, N = int(rng.integers(P, 200)), int(rng.integers(P, 200))
    cuts = np.sort(rng.integers(0, M + 1, P - 1))
    rs = list(np.diff(np.concatenate([[0], cuts, [M]])).astype(int))
    if seed % 2 == 0:
        rs = synth.split_sizes(M, P)
    cs = synth.split_sizes(N, P)
    coo = [synth.random_coo(M, N, int(rng.integers(0, 800)), dup_frac=0.5, neg_frac=0.2,
                            seed=seed * 31 + q) for q in range(P)]
    x = synth.x_vector(0, N, "int", seed=seed).numpy()
    check_matrix(c, f"random{seed}", M, N, rs, cs, coo, "int", x, exact_y=True)


def case_sf(c, seed):
    """Standalone SF: random graph with holes and fan-in, REPLACE and SUM vs graph walk."""
    P, r = c.P, c.r
    rng = np.random.default_rng(seed)
    nroots = [int(rng.integers(0, 20)) for _ in range(P)]
    owners = [q for q in range(P) if nroots[q] > 0]
    leaves, rootdata, leafdata = [], [], []
    for p in range(P):
        nl = int(rng.integers(0, 30)) if owners else 0
        space = nl + int(rng.integers(0, 5))
        il = rng.permutation(space)[:nl].astype(np.int64)
        rr = rng.choice(owners, nl).astype(np.int64) if nl else np.zeros(0, np.int64)
        ro = np.array([rng.integers(0, nroots[q]) for q in rr], dtype=np.int64)
        leaves.append((il, rr, ro))
        rootdata.append(rng.integers(-50, 50, nroots[p]).astype(float))
        leafdata.append(rng.integers(-50, 50, space).astype(float))
    il, rr, ro = leaves[r]
    sf = sp.StarForest(c.comm, nroots[r], il, rr, ro)
    want_t = 1 if os.environ.get("SPMAT_HALO") == "nccl" else 2
    assert P == 1 or sf.transport() == want_t, f"sf transport {sf.transport()}"
    # several rounds: the NVLink transport cycles its two staging buffers and waits on the
    # consumers' release flags from the third operation on
    for rnd in range(3):
        rd = [a + 100 * rnd for a in rootdata]
        ld = [a - 7 * rnd for a in leafdata]
        for op in (sp.REPLACE, sp.SUM):
            want = oracle.sf_bcast(nroots, leaves, rd, ld, op)[r]
            root = torch.from_numpy(rd[r]).cuda()
            leaf = torch.from_numpy(ld[r]).cuda()
            sf.bcast_begin(root, leaf, op)
            sf.bcast_end(root, leaf, op)
            assert np.array_equal(leaf.cpu().numpy(), want), f"sf seed {seed} round {rnd} op {op} rank {r}"
            # reduce leaf -> root, (source rank, leaf index) order (oracle.sf_reduce)
            want = oracle.sf_reduce(nroots, leaves, ld, rd, op)[r]
            root = torch.from_numpy(rd[r]).cuda()
            leaf = torch.from_numpy(ld[r]).cuda()
            sf.reduce_begin(leaf, root, op)
            sf.reduce_end(leaf, root, op)
            assert np.array_equal(root.cpu().numpy(), want), f"sf reduce seed {seed} round {rnd} op {op} rank {r}"
    sf.check()
    sf.close()


def case_cg(c):
    """CGAsync analogue across ranks: iterate vs the oracle's P-rank CG; the residual history
    (device scalars from the scalar board) is bit-identical on every rank."""
    P, r = c.P, c.r
    shape = (10, 9, 4 * P)
    M = int(np.prod(shape))
    sizes = synth.slab_sizes(shape, P)
    off = synth.offsets_from_sizes(sizes)
    coo = [synth.stencil_coo(shape, 7, rows=(off[q], off[q + 1]), values="int") for q in range(P)]
    O = oracle.OracleMat(M, M, sizes, sizes, [t[0] for t in coo], [t[1] for t in coo])
    O.set_values([t[2] for t in coo])
    i, j, v = coo[r]
    A = sp.Mat(c.comm, sizes[r], sizes[r], M, M, i.cuda(), j.cuda())
    A.set_values(v.cuda())
    rhs = synth.x_vector(0, M, "real", seed=9).numpy()
    b = torch.from_numpy(np.ascontiguousarray(rhs[off[r]:off[r + 1]])).cuda()
    iters = 25
    x = torch.zeros(sizes[r], dtype=torch.float64, device="cuda")
    hist = torch.zeros(iters + 1, dtype=torch.float64, device="cuda")
    A.cg(b, x, iters, hist)
    xo, ho = O.cg(rhs, np.zeros(M), iters)
    assert rel_err(x.cpu().numpy(), xo[off[r]:off[r + 1]]) <= 1e-10
    h = hist.cpu()
    allh = [torch.zeros_like(h) for _ in range(P)]
    dist.all_gather_object(allh, h)
    for q in range(P):
        assert torch.equal(allh[q], h), "residual history differs between ranks"
    assert np.max(np.abs(h.numpy() - ho) / ho[0]) <= 1e-10
    # dot product of integer vectors: exact
    a = synth.x_vector(off[r], off[r + 1], "int", seed=4).cuda()
    bb = synth.x_vector(off[r], off[r + 1], "int", seed=5).cuda()
    res = torch.zeros(1, dtype=torch.float64, device="cuda")
    A.dot(a, bb, res)
    ga = synth.x_vector(0, M, "int", seed=4).numpy()
    gb = synth.x_vector(0, M, "int", seed=5).numpy()
    assert res.item() == float(np.dot(ga, gb))
    # the CUDA-graph CG (device-side epochs) equals the eagerly launched one bit for bit
    outs = []
    for g in ("1", "0"):
        os.environ["SPMAT_GRAPH"] = g
        xg = torch.zeros(sizes[r], dtype=torch.float64, device="cuda")
        A.cg(b, xg, iters)
        A.cg(b, xg, 3)  # a second call replays the cached graph
        outs.append(xg.cpu())
    os.environ.pop("SPMAT_GRAPH")
    assert torch.equal(outs[0], outs[1])
    A.check()
    A.close()


def case_host_pipeline(c, kind):
    """Host x/y with >= 2^20 rows per rank take the chunked H2D / SpMV / D2H pipeline with the
    standalone NVLink put and per-chunk off-diagonal adds; bit-identical to device pointers."""
    P, r = c.P, c.r
    if kind == "slab":
        shape = (128, 128, 64 * P)
        sizes = synth.slab_sizes(shape, P)
        off = synth.offsets_from_sizes(sizes)
        i, j, v = synth.stencil_coo(shape, 7, rows=(off[r], off[r + 1]), values="real", device="cuda")
    else:
        procs = synth.box_procs(P)
        shape = (112 * procs[0], 96 * procs[1], 100 * procs[2])
        sizes = synth.box_sizes(shape, procs)
        off = synth.offsets_from_sizes(sizes)
        i, j, v = synth.stencil_coo_box(shape, 7, procs, r, values="real", device="cuda")
    M = off[-1]
    A = sp.Mat(c.comm, sizes[r], sizes[r], M, M, i, j)
    A.set_values(v)
    x = synth.x_vector(off[r], off[r + 1], "real", device="cuda")
    yd = torch.empty(sizes[r], dtype=torch.float64, device="cuda")
    A.mult(x, yd)
    xh = x.cpu().pin_memory()
    yh = torch.full((sizes[r],), float("nan"), dtype=torch.float64).pin_memory()
    for _ in range(3):  # epochs stay in step with the device-pointer MatMults
        A.mult(xh, yh)
        assert torch.equal(yh, yd.cpu()), f"host pipeline {kind} rank {r}"
        A.mult(x, yd)
    # asynchronous calls through the two staging slots (epochs chained by events), one sync
    xs = [synth.x_vector(off[r], off[r + 1], "real", seed=30 + k, device="cuda") for k in range(4)]
    want = []
    for xk in xs:
        A.mult(xk, yd)
        want.append(yd.cpu())
    xhs = [xk.cpu().pin_memory() for xk in xs]
    yhs = [torch.full((sizes[r],), float("nan"), dtype=torch.float64).pin_memory() for _ in xs]
    s = torch.cuda.current_stream()
    for xk, yk in zip(xhs, yhs):
        A.mult_async(xk, yk, s)
    s.synchronize()
    for k, (yk, w) in enumerate(zip(yhs, want)):
        assert torch.equal(yk, w), f"async host pipeline {kind} rank {r} call {k}"
    for yk in yhs:  # pipelined calls: downloads waited for at the next call / flush
        yk.fill_(float("nan"))
    for xk, yk in zip(xhs, yhs):
        A.mult_pipelined(xk, yk, s)
    A.flush(s)
    s.synchronize()
    for k, (yk, w) in enumerate(zip(yhs, want)):
        assert torch.equal(yk, w), f"pipelined host calls {kind} rank {r} call {k}"
    A.check()
    A.close()


def case_transpose(c, seed):
    """MatMultTranspose across ranks (halo SF reduce) vs the oracle, bit-exact with real values."""
    P, r = c.P, c.r
    rng = np.random.default_rng(800 + seed)
    M, N = int(rng.integers(P, 150)), int(rng.integers(P, 150))
    rs = synth.split_sizes(M, P)
    cs = synth.split_sizes(N, P)
    coo = [synth.random_coo(M, N, int(rng.integers(0, 600)), dup_frac=0.4, neg_frac=0.1, values="real",
                            seed=seed * 17 + q) for q in range(P)]
    O = oracle.OracleMat(M, N, rs, cs, [t[0] for t in coo], [t[1] for t in coo])
    O.set_values([t[2] for t in coo])
    i, j, v = coo[r]
    A = sp.Mat(c.comm, rs[r], cs[r], M, N, i.cuda(), j.cuda())
    A.set_values(v.cuda())
    roff, coff = synth.offsets_from_sizes(rs), synth.offsets_from_sizes(cs)
    xg = synth.x_vector(0, M, "real", seed=seed).numpy()
    x = torch.from_numpy(xg[roff[r]:roff[r + 1]].copy()).cuda()
    y = torch.full((cs[r],), float("nan"), dtype=torch.float64, device="cuda")
    for _ in range(2):
        A.mult_transpose(x, y)
        want = O.mult_transpose(xg)[coff[r]:coff[r + 1]]
        assert np.array_equal(canon(y.cpu().numpy()), canon(want)), f"transpose seed {seed} rank {r}"
    A.check()
    A.close()


def case_full_c4(c):
    """The bench's default workload at full size (C4: 256^3 rows per rank, z-slabs, the fused
    NVLink MatMult): sampled rows of every rank vs the oracle from the COO definition."""
    P, r = c.P, c.r
    i, j, v, sizes = synth.config_rank_coo("c4", P, r, values="real", device="cuda")
    off = synth.offsets_from_sizes(sizes)
    M = off[-1]
    A = sp.Mat(c.comm, sizes[r], sizes[r], M, M, i, j)
    del i, j
    y = torch.empty(sizes[r], dtype=torch.float64, device="cuda")
    # integer values: A.1 over EVERY row of every rank = out-of-grid neighbour count (P3)
    _, _, vi, _ = synth.config_rank_coo("c4", P, r, values="int", device="cuda")
    A.set_values(vi)
    del vi
    A.mult(torch.ones(sizes[r], dtype=torch.float64, device="cuda"), y)
    shape = synth.config_shape("c4", P)
    g = torch.arange(off[r], off[r + 1], device="cuda")
    want = torch.zeros_like(y)
    for n in shape:
        cc = g % n
        want += (cc == 0).double() + (cc == n - 1).double()
        g = g // n
    assert torch.equal(y, want), f"full-size C4 A.1 rank {r}: {int((y != want).sum())} rows differ"
    A.set_values(v)
    del v
    x = synth.x_vector(off[r], off[r + 1], "real", device="cuda")
    for _ in range(3):  # several epochs of the NVLink halo
        A.mult(x, y)
    A.check()
    g = torch.Generator().manual_seed(100 + r)
    rows = torch.unique(torch.cat([torch.randint(off[r], off[r + 1], (800,), generator=g),
                                   torch.tensor([off[r], off[r] + 1, off[r + 1] - 2, off[r + 1] - 1])]))
    ih, jh, vh = synth.stencil_coo(synth.config_shape("c4", P), 7, rows=rows, values="real")
    xg = synth.x_vector(0, M, "real").numpy()
    ys = oracle.sample_rows(ih, jh, vh, rows.numpy(), xg)
    got = y[(rows - off[r]).cuda()].cpu().numpy()
    assert rel_err(got, ys) <= TOL, f"full-size C4 rank {r}"
    A.close()
    torch.cuda.empty_cache()


def case_full_c4b(c):
    """C4b at full size (256^3 rows per rank, box decomposition with per-rank renumbering): the
    split off-diagonal tail, whose sums the consumer warps fold into most boundary rows as they
    write them (the rest by the add pass after the sweep).  A.1 over EVERY row against the
    out-of-grid neighbour count (P3, integer values, exact), then real values on sampled rows
    vs the oracle from the COO definition, over several halo epochs."""
    P, r = c.P, c.r
    shape, procs = synth.config_shape("c4b", P), synth.box_procs(P)
    sizes = synth.box_sizes(shape, procs)
    off = synth.offsets_from_sizes(sizes)
    M = off[-1]
    i, j, vi, _ = synth.config_rank_coo("c4b", P, r, values="int", device="cuda")
    A = sp.Mat(c.comm, sizes[r], sizes[r], M, M, i, j)
    A.set_values(vi)
    del vi
    y = torch.empty(sizes[r], dtype=torch.float64, device="cuda")
    ones = torch.ones(sizes[r], dtype=torch.float64, device="cuda")
    px, py, pz = procs
    bx, by, bz = r % px, (r // px) % py, r // (px * py)
    lo = [(b * n) // p for b, n, p in zip((bx, by, bz), shape, procs)]
    ext = [((b + 1) * n) // p - (b * n) // p for b, n, p in zip((bx, by, bz), shape, procs)]
    loc = torch.arange(sizes[r], device="cuda")
    coords = [lo[0] + loc % ext[0], lo[1] + (loc // ext[0]) % ext[1], lo[2] + loc // (ext[0] * ext[1])]
    want = torch.zeros_like(y)
    for cc, n in zip(coords, shape):
        want += (cc == 0).double() + (cc == n - 1).double()
    for it in range(4):  # several epochs: the fold and the add pass both see every flag parity
        A.mult(ones, y)
        assert torch.equal(y, want), f"full-size C4b A.1 rank {r} epoch {it}: {int((y != want).sum())} rows differ"
    _, _, v, _ = synth.config_rank_coo("c4b", P, r, values="real", device="cuda")
    A.set_values(v)
    xg = synth.x_vector(0, M, "real", device="cuda")
    x = xg[off[r]:off[r + 1]].contiguous()
    for _ in range(3):
        A.mult(x, y)
    A.check()
    g = torch.Generator().manual_seed(200 + r)
    rows = torch.unique(torch.cat([torch.randint(off[r], off[r + 1], (600,), generator=g),
                                   torch.tensor([off[r], off[r + 1] - 1]),
                                   off[r] + torch.arange(0, sizes[r], ext[0])[:200]]))  # x-face rows
    sel = torch.isin(i, rows.cuda())
    ih, jh, vh = i[sel].cpu(), j[sel].cpu(), v[sel].cpu()
    del i, j, v
    ys = oracle.sample_rows(ih, jh, vh, rows.numpy(), xg.cpu().numpy())
    got = y[(rows - off[r]).cuda()].cpu().numpy()
    assert rel_err(got, ys) <= TOL, f"full-size C4b rank {r}"
    A.close()
    torch.cuda.empty_cache()


def case_full_c5(c):
    """C5 at full size (24 M rows, 1.92 G nonzeros, z-slabs of 200/P planes) with 3x3 blocks
    (diagonal and off-diagonal) and with CSR: A.1 over EVERY row of every rank against the
    Kronecker closed form 6 * prod_d (4 + n_d) (integer values, exact), then real values on
    node windows at the slab boundaries vs the oracle from the COO definition."""
    P, r = c.P, c.r
    n = 200
    i, j, vi, sizes = synth.config_rank_coo("c5", P, r, values="int", device="cuda")
    off = synth.offsets_from_sizes(sizes)
    M = off[-1]
    A = sp.Mat(c.comm, sizes[r], sizes[r], M, M, i, j)
    del i, j
    A.set_values(vi)
    del vi
    torch.cuda.empty_cache()
    node = torch.arange(off[r], off[r + 1], device="cuda") // 3
    want = torch.full((sizes[r],), 6.0, dtype=torch.float64, device="cuda")
    for _ in range(3):
        cc = node % n
        want *= 4 + (cc > 0).double() + (cc < n - 1).double()
        node = node // n
    y = torch.empty(sizes[r], dtype=torch.float64, device="cuda")
    ones = torch.ones(sizes[r], dtype=torch.float64, device="cuda")
    for bs in (3, 1):
        A.set_block_size(bs)
        for _ in range(3):
            A.mult(ones, y)
        A.check()
        assert torch.equal(y, want), f"C5 bs={bs} A.1 rank {r}: {int((y != want).sum())} rows differ"
    del want, ones
    _, _, v, _ = synth.config_rank_coo("c5", P, r, values="real", device="cuda")
    A.set_values(v)
    del v
    torch.cuda.empty_cache()
    x = synth.x_vector(off[r], off[r + 1], "real", device="cuda")
    xg = synth.x_vector(0, M, "real").numpy()
    n0, n1 = off[r] // 3, off[r + 1] // 3
    pi, pj, pv, rws = [], [], [], []
    for a0 in sorted({n0, max(n0, n1 - 64 * n - 5), (n0 + n1) // 2, n1 - 64}):
        ih, jh, vh = synth.elasticity_coo(n, nodes=(a0, a0 + 64), values="real")
        pi.append(ih); pj.append(jh); pv.append(vh)
        rws.append(torch.arange(3 * a0, 3 * (a0 + 64)))
    rows = torch.unique(torch.cat(rws))
    ys = oracle.sample_rows(torch.cat(pi), torch.cat(pj), torch.cat(pv), rows.numpy(), xg)
    for bs in (3, 1):
        A.set_block_size(bs)
        A.mult(x, y)
        A.check()
        got = y[(rows - off[r]).cuda()].cpu().numpy()
        assert rel_err(got, ys) <= TOL, f"full-size C5 bs={bs} rank {r}: {rel_err(got, ys)}"
    A.close()
    torch.cuda.empty_cache()


def case_errors(c):
    P, r = c.P, c.r
    # an error only one rank can see (its m_local >= 2^31): every rank returns an error, none
    # blocks in the next collective (Comm::agree)
    big = 1 << 31
    mloc = big if r == P - 1 else 2
    Mg = 2 * (P - 1) + big
    try:
        sp.Mat(c.comm, mloc, mloc, Mg, Mg, torch.zeros(0, dtype=torch.int64, device="cuda"),
               torch.zeros(0, dtype=torch.int64, device="cuda"))
        raise AssertionError("rank-local error not raised")
    except sp.SpmatError as e:
        assert e.status == sp.SPMAT_ERR_ARG, e
    # only the last rank has an out-of-range index: every rank must report it
    i = torch.tensor([0, 1] if r < P - 1 else [0, 99], device="cuda") + c.r * 2
    j = torch.tensor([0, 1], device="cuda")
    try:
        sp.Mat(c.comm, 2, 2, 2 * P, 2 * P, i, j)
        raise AssertionError("range error not raised")
    except sp.SpmatError as e:
        assert e.status == sp.SPMAT_ERR_RANGE, e
        assert f"rank {P - 1}" in e.message
    try:
        sp.Mat(c.comm, 2 if r else 3, 2, 2 * P, 2 * P, i[:0], j[:0])
        raise AssertionError("mismatch not raised")
    except sp.SpmatError as e:
        assert e.status == sp.SPMAT_ERR_MISMATCH, e


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    c = Ctx()
    failures = 0
    cases = [("stencil-int", lambda: case_stencil(c, "int")),
             ("stencil-real", lambda: case_stencil(c, "real")),
             ("q1-int", lambda: case_q1(c, "int")), ("q1-real", lambda: case_q1(c, "real")),
             ("elasticity", lambda: case_elasticity(c))]
    cases += [(f"random{s}", (lambda s=s: case_random(c, s))) for s in range(16)]
    cases += [(f"sf{s}", (lambda s=s: case_sf(c, s))) for s in range(24)]
    cases += [("box7-int", lambda: case_box(c, 7, "int")), ("box7-real", lambda: case_box(c, 7, "real")),
              ("box27-real", lambda: case_box(c, 27, "real"))]
    cases += [("cg", lambda: case_cg(c))]
    cases += [("host-pipeline-slab", lambda: case_host_pipeline(c, "slab")),
              ("host-pipeline-box", lambda: case_host_pipeline(c, "box"))]
    cases += [(f"transpose{s}", (lambda s=s: case_transpose(c, s))) for s in range(6)]
    cases += [("full-c4", lambda: case_full_c4(c)), ("full-c4b", lambda: case_full_c4b(c)),
              ("full-c5", lambda: case_full_c5(c))]
    cases += [("errors", lambda: case_errors(c))]
    only = [s for s in os.environ.get("MP_CASES", "").split(",") if s]
    if only:
        cases = [(nm, fn) for nm, fn in cases if any(nm.startswith(s) for s in only)]
    for name, fn in cases:
        try:
            fn()
            dist.barrier()
            if c.r == 0:
                c.log(f"PASS {name}")
        except Exception:
            failures += 1
            c.log(f"FAIL {name}\n{traceback.format_exc()}")
            dist.barrier()
    c.comm.close()
    dist.destroy_process_group()
    if c.r == 0:
        print(f"halo_mode={getattr(c, 'halo_mode', -1)}", flush=True)
        print(f"MULTIRANK P={c.P} failures={failures}", flush=True)
    sys.exit(1 if failures else 0)


if __name__ == "__main__":
    main()
