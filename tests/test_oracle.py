"""Pins of the CPU oracle against what the paper and the mathematics fix (no GPU).

Each test pins oracle/ to something other than itself: closed forms (nnz counts, A.1 row
sums, polynomial x), invariants, SPEC.md worked examples stored under tests/golden/, and
numpy brute force (np.add.at dense assembly + numpy matmul) on tiny inputs.
"""
import itertools
import os

import numpy as np
import pytest
import torch

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _np(t):
    return t.numpy() if hasattr(t, "numpy") else np.asarray(t)


def build_stencil(shape, npts, P=1, values="int", seed=8646, sizes=None):
    M = int(np.prod(shape))
    if sizes is None:
        sizes = synth.split_sizes(M, P)
    off = synth.offsets_from_sizes(sizes)
    ii, jj, vv = [], [], []
    for r in range(len(sizes)):
        i, j, v = synth.stencil_coo(shape, npts, rows=(off[r], off[r + 1]), values=values, seed=seed)
        ii.append(i); jj.append(j); vv.append(v)
    A = oracle.OracleMat(M, M, sizes, sizes, ii, jj)
    A.set_values(vv)
    return A, ii, jj, vv


def numpy_dense(M, N, ii, jj, vv):
    """Independent brute force: scatter-add every valid triplet."""
    A = np.zeros((M, N))
    for i, j, v in zip(ii, jj, vv):
        i, j, v = _np(i), _np(j), _np(v)
        ok = (i >= 0) & (j >= 0)
        np.add.at(A, (i[ok], j[ok]), v[ok])
    return A


def struct_pattern(M, N, ii, jj):
    S = np.zeros((M, N), dtype=bool)
    for i, j in zip(ii, jj):
        i, j = _np(i), _np(j)
        ok = (i >= 0) & (j >= 0)
        S[i[ok], j[ok]] = True
    return S


# ---------------------------------------------------------------- P1 nnz closed forms
@pytest.mark.parametrize("n", [3, 5, 8, 64])
def test_nnz_5pt(n):
    A, *_ = build_stencil((n, n), 5)
    assert A.info(0, "nnz_d") == 5 * n * n - 4 * n


@pytest.mark.parametrize("n", [2, 3, 6, 9])
def test_nnz_7pt(n):
    A, *_ = build_stencil((n, n, n), 7)
    assert A.info(0, "nnz_d") == 7 * n ** 3 - 6 * n ** 2


@pytest.mark.parametrize("n", [2, 3, 5, 6])
def test_nnz_q1(n):
    i, j, v = synth.q1_coo(n)
    A = oracle.OracleMat(n ** 3, n ** 3, [n ** 3], [n ** 3], [i], [j])
    assert A.info(0, "nnz_d") == (3 * n - 2) ** 3
    assert A.info(0, "ncontrib") == 64 * (n - 1) ** 3


@pytest.mark.parametrize("n", [2, 3, 4])
def test_nnz_elasticity(n):
    i, j, v = synth.elasticity_coo(n)
    M = 3 * n ** 3
    A = oracle.OracleMat(M, M, [M], [M], [i], [j])
    assert A.info(0, "nnz_d") == 9 * (3 * n - 2) ** 3


# ---------------------------------------------------------------- P8 invariants
@pytest.mark.parametrize("P", [1, 2, 3, 4])
def test_csr_invariants(P):
    shape = (5, 4, 6)
    A, ii, jj, _ = build_stencil(shape, 7, P=P)
    M = int(np.prod(shape))
    total = 0
    for r in range(P):
        rs, re = A.info(r, "rstart"), A.info(r, "rend")
        for blk in ("d", "o"):
            rp = A.export(r, f"rowptr_{blk}")
            col = A.export(r, f"col_{blk}")
            assert rp[0] == 0 and np.all(np.diff(rp) >= 0) and rp[-1] == col.size
            for q in range(re - rs):
                assert np.all(np.diff(col[rp[q]:rp[q + 1]]) > 0)
        cm = A.export(r, "colmap")
        assert np.all(np.diff(cm) > 0)
        assert not np.any((cm >= rs) & (cm < re))
        total += A.info(r, "nnz_d") + A.info(r, "nnz_o")
    assert total == 7 * 5 * 4 * 6 - 2 * (5 * 4 + 4 * 6 + 5 * 6)


# ---------------------------------------------------------------- SPEC worked examples
def _parse_golden(name):
    d = {}
    for line in open(os.path.join(GOLD, name)):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        k, rest = line.split(None, 1)
        d[k] = rest
    return d


def test_spec_coo_example():
    g = _parse_golden("spec_coo_example.txt")
    M, N = int(g["M"]), int(g["N"])
    i = np.array(g["i"].split(), dtype=np.int64)
    j = np.array(g["j"].split(), dtype=np.int64)
    v = np.array(g["v"].split(), dtype=np.float64)
    A = oracle.OracleMat(M, N, [M], [N], [i], [j])
    sp = [tuple(int(t) for t in s.strip("()").split(",")) for s in g["sparsity"].split()]
    rp, cd = A.export(0, "rowptr_d"), A.export(0, "col_d")
    got = [(q, int(c)) for q in range(M) for c in cd[rp[q]:rp[q + 1]]]
    assert got == sp
    A.set_values([v], oracle.INSERT)
    want = np.array([[float(t) for t in row.split()] for row in g["insert"].split(";")])
    assert np.array_equal(A.dense(), want)
    A.set_values([v], oracle.ADD)
    A.set_values([v], oracle.ADD)
    want = np.array([[float(t) for t in row.split()] for row in g["insert_add_add"].split(";")])
    assert np.array_equal(A.dense(), want)


def test_spec_sf_examples():
    g = _parse_golden("spec_sf_examples.txt")
    # pingpong REPLACE / SUM
    for key, op in (("pingpong_replace", oracle.REPLACE), ("pingpong_sum", oracle.SUM)):
        toks = g[key].split()
        init = [float(t) for t in toks[1:4]]
        want = [float(t) for t in toks[5:8]]
        leaves = [(None, [], []), (None, [0, 0, 0], [0, 1, 2])]
        out = oracle.sf_bcast([3, 0], leaves, [[10, 20, 30], []], [[], init], op)
        assert out[1].tolist() == want and out[0].size == 0
    toks = g["fanin_replace"].split()
    out = oracle.sf_bcast([1], [(None, [0, 0], [0, 0])], [[float(toks[1])]], [[0.0, 0.0]],
                          oracle.REPLACE)
    assert out[0].tolist() == [float(t) for t in toks[3:5]]


def test_sf_random_graphs_vs_python_walk():
    """Random SFs with holes and fan-in vs an independent Python edge walk."""
    rng = np.random.default_rng(7)
    for trial in range(40):
        P = int(rng.integers(1, 6))
        nroots = [int(rng.integers(0, 12)) for _ in range(P)]
        owners = [q for q in range(P) if nroots[q] > 0]
        leaves, rootdata, leafdata = [], [], []
        for p in range(P):
            nl = int(rng.integers(0, 10)) if owners else 0
            space = nl + int(rng.integers(0, 4))
            il = rng.permutation(space)[:nl] if nl else np.zeros(0, np.int64)
            rr = rng.choice(owners, nl) if nl else np.zeros(0, np.int64)
            ro = np.array([rng.integers(0, nroots[q]) for q in rr], dtype=np.int64)
            leaves.append((il, rr, ro))
            rootdata.append(rng.integers(-50, 50, nroots[p]).astype(float))
            leafdata.append(rng.integers(-50, 50, space).astype(float))
        for op in (oracle.REPLACE, oracle.SUM):
            out = oracle.sf_bcast(nroots, leaves, rootdata, leafdata, op)
            for p in range(P):
                want = leafdata[p].copy()
                il, rr, ro = leaves[p]
                for l in range(len(rr)):
                    val = rootdata[rr[l]][ro[l]]
                    want[il[l]] = val if op == oracle.REPLACE else want[il[l]] + val
                assert np.array_equal(out[p], want)


def test_sf_offset_out_of_range():
    with pytest.raises(ValueError):
        oracle.sf_bcast([2], [(None, [0], [2])], [[1.0, 2.0]], [[0.0]])


# ---------------------------------------------------------------- P6 brute force
@pytest.mark.parametrize("case", ["5pt8", "7pt6", "q1_5", "el4"])
@pytest.mark.parametrize("values", ["int", "real"])
def test_dense_bruteforce(case, values):
    if case == "5pt8":
        M = 64
        i, j, v = synth.stencil_coo((8, 8), 5, values=values)
    elif case == "7pt6":
        M = 216
        i, j, v = synth.stencil_coo((6, 6, 6), 7, values=values)
    elif case == "q1_5":
        M = 125
        i, j, v = synth.q1_coo(5, values=values)
    else:
        M = 3 * 64
        i, j, v = synth.elasticity_coo(4, values=values)
    A = oracle.OracleMat(M, M, [M], [M], [i], [j])
    A.set_values([v])
    D = numpy_dense(M, M, [i], [j], [v])
    S = struct_pattern(M, M, [i], [j])
    Ad = A.dense()
    if values == "int":
        assert np.array_equal(Ad, D)
    else:
        assert np.allclose(Ad, D, rtol=0, atol=1e-13)
    # structure: stored positions == positions referenced by a valid triplet
    nnz = A.info(0, "nnz_d")
    assert nnz == S.sum()
    x = synth.x_vector(0, M, values).numpy()
    y = A.mult(x)
    ref = (D.astype(np.longdouble) @ x.astype(np.longdouble)).astype(np.float64)
    if values == "int":
        assert np.array_equal(y, ref)
    else:
        assert np.max(np.abs(y - ref)) <= 1e-13 * max(1.0, np.max(np.abs(ref)))


# ---------------------------------------------------------------- P2 contributions per nonzero
def test_q1_contribution_counts():
    n = 5
    i, j, v = synth.q1_coo(n)
    A = oracle.OracleMat(n ** 3, n ** 3, [n ** 3], [n ** 3], [i], [j])
    jm = A.export(0, "jmap")
    rp, cd = A.export(0, "rowptr_d"), A.export(0, "col_d")
    cnt = np.diff(jm)

    def coords(g):
        return g % n, (g // n) % n, g // (n * n)

    for q in range(n ** 3):
        ci = coords(q)
        for t in range(rp[q], rp[q + 1]):
            cj = coords(int(cd[t]))
            want = 1
            for d in range(3):
                interior = 0 < ci[d] < n - 1
                want *= 2 if (ci[d] == cj[d] and interior) else 1
            assert cnt[t] == want
    assert cnt.sum() == 64 * (n - 1) ** 3


# ---------------------------------------------------------------- P3 A.1 closed forms
def test_ones_5pt():
    n = 9
    A, *_ = build_stencil((n, n), 5)
    y = A.mult(np.ones(n * n))
    for g in range(n * n):
        ix, iy = g % n, g // n
        out = (ix == 0) + (ix == n - 1) + (iy == 0) + (iy == n - 1)
        assert y[g] == out


def test_ones_7pt_partitioned():
    n = 6
    for P in (1, 2, 3):
        A, *_ = build_stencil((n, n, n), 7, P=P)
        y = A.mult(np.ones(n ** 3))
        for g in range(n ** 3):
            c = (g % n, (g // n) % n, g // (n * n))
            assert y[g] == sum((ci == 0) + (ci == n - 1) for ci in c)


def test_ones_q1():
    n = 5
    for variant in ("lap", "mass"):
        i, j, v = synth.q1_coo(n, variant=variant)
        A = oracle.OracleMat(n ** 3, n ** 3, [n ** 3], [n ** 3], [i], [j])
        A.set_values([v])
        y = A.mult(np.ones(n ** 3))
        if variant == "lap":
            assert np.all(y == 0.0)
        else:
            for g in range(n ** 3):
                c = (g % n, (g // n) % n, g // (n * n))
                assert y[g] == 27 * np.prod([2 if 0 < ci < n - 1 else 1 for ci in c])


def test_ones_elasticity():
    n = 4
    i, j, v = synth.elasticity_coo(n)
    M = 3 * n ** 3
    A = oracle.OracleMat(M, M, [M], [M], [i], [j])
    A.set_values([v])
    y = A.mult(np.ones(M))
    for row in range(M):
        g = row // 3
        c = (g % n, (g // n) % n, g // (n * n))
        nd = [(ci > 0) + (ci < n - 1) for ci in c]
        assert y[row] == 6 * np.prod([4 + k for k in nd])


# ---------------------------------------------------------------- P4 polynomial x
def test_polynomial_7pt():
    n = 7
    A, *_ = build_stencil((n, n, n), 7)
    g = np.arange(n ** 3)
    ix, iy, iz = g % n, (g // n) % n, g // (n * n)
    interior = (ix > 0) & (ix < n - 1) & (iy > 0) & (iy < n - 1) & (iz > 0) & (iz < n - 1)
    y = A.mult((3 * ix - 2 * iy + iz + 5).astype(float))
    assert np.all(y[interior] == 0)
    y = A.mult((ix ** 2 + iy ** 2 + iz ** 2).astype(float))
    assert np.all(y[interior] == -6)


def test_polynomial_5pt():
    n = 8
    A, *_ = build_stencil((n, n), 5)
    g = np.arange(n * n)
    ix, iy = g % n, g // n
    interior = (ix > 0) & (ix < n - 1) & (iy > 0) & (iy < n - 1)
    y = A.mult((ix ** 2 + iy ** 2).astype(float))
    assert np.all(y[interior] == -4)


# ---------------------------------------------------------------- P7 global vs partitioned
@pytest.mark.parametrize("values", ["int", "real"])
def test_partitioned_equivalence(values):
    shape = (6, 5, 8)
    M = int(np.prod(shape))
    A1, *_ = build_stencil(shape, 7, P=1, values=values)
    x = synth.x_vector(0, M, values).numpy()
    y1 = A1.mult(x)
    for P in (2, 3, 4, 5, 8):  # 3 and 5: uneven slabs (remainder planes to the low ranks)
        sizes = synth.slab_sizes(shape, P)
        assert sum(sizes) == M and all(s % (6 * 5) == 0 for s in sizes)
        AP, *_ = build_stencil(shape, 7, P=P, values=values, sizes=sizes)
        yP = AP.mult(x)
        assert np.array_equal(AP.dense(), A1.dense())  # assembled values: same (src,k) order
        if values == "int":
            assert np.array_equal(yP, y1)
        else:
            assert np.max(np.abs(yP - y1)) <= 1e-14 * np.max(np.abs(y1))


def test_q1_slabs_remote_entries():
    """Element slabs: the top face of each slab is owned by the next rank (remote COO)."""
    n, P = 6, 3
    M = n ** 3
    sizes = synth.slab_sizes((n, n, n), P)
    ii, jj, vv = [], [], []
    for r in range(P):
        i, j, v = synth.q1_coo(n, elems=synth.q1_slab_elems(n, P, r), values="real")
        ii.append(i); jj.append(j); vv.append(v)
    A = oracle.OracleMat(M, M, sizes, sizes, ii, jj)
    A.set_values(vv)
    i1, j1, v1 = synth.q1_coo(n, values="real")
    A1 = oracle.OracleMat(M, M, [M], [M], [i1], [j1])
    A1.set_values([v1])
    assert np.array_equal(A.dense(), A1.dense())  # bit-exact: canonical (src, k) order
    assert sum(A.info(r, "nsend") for r in range(P)) > 0
    # sum of sends == sum of receives, per pair
    for r in range(P):
        for q in range(P):
            assert A.export(r, "send_count")[q] == A.export(q, "recv_count")[r]
    plane = n * n
    for r in range(P - 1):  # rows of the 4 top-face nodes of each top-layer element
        assert A.export(r, "send_count")[r + 1] == 4 * 8 * (n - 1) ** 2  # 4 top nodes x 8 cols


# ---------------------------------------------------------------- P10 halo plan
@pytest.mark.parametrize("P", [2, 4])
def test_halo_closed_forms(P):
    shape = (5, 4, 8)
    sizes = synth.slab_sizes(shape, P)
    A, ii, jj, _ = build_stencil(shape, 7, P=P, sizes=sizes)
    plane = 5 * 4
    off = synth.offsets_from_sizes(sizes)
    for r in range(P):
        nb = (r > 0) + (r < P - 1)
        assert A.info(r, "n_ghost") == nb * plane
        # brute force: referenced columns minus owned ones, sorted
        j = _np(jj[r])
        ref = np.unique(j[(j >= 0) & ((j < off[r]) | (j >= off[r + 1]))])
        assert np.array_equal(A.export(r, "colmap"), ref)
        own = A.export(r, "leaf_owner")
        ofs = A.export(r, "leaf_offset")
        assert np.array_equal(np.asarray(off)[own] + ofs, ref)
    # root side mirrors the leaf side
    for q in range(P):
        rc = A.export(q, "root_count")
        ro = A.export(q, "root_offsets")
        pos = 0
        for p in range(P):
            lo = A.export(p, "leaf_owner")
            lof = A.export(p, "leaf_offset")
            assert rc[p] == np.sum(lo == q)
            assert np.array_equal(ro[pos:pos + rc[p]], lof[lo == q])
            pos += rc[p]


def test_halo_elasticity_ghosts():
    n, P = 4, 2
    M = 3 * n ** 3
    sizes = synth.slab_sizes((n, n, n), P, dof=3)
    ii, jj = [], []
    for r in range(P):
        nodes = sizes[0] // 3
        i, j, v = synth.elasticity_coo(n, nodes=(r * nodes, (r + 1) * nodes))
        ii.append(i); jj.append(j)
    A = oracle.OracleMat(M, M, sizes, sizes, ii, jj)
    for r in range(P):
        assert A.info(r, "n_ghost") == 3 * n * n


# ---------------------------------------------------------------- random COO + errors
@pytest.mark.parametrize("seed", range(12))
def test_random_coo_bruteforce(seed):
    rng = np.random.default_rng(seed)
    P = int(rng.integers(1, 6))
    M, N = int(rng.integers(1, 40)), int(rng.integers(1, 40))
    rs = synth.split_sizes(M, P) if seed % 2 else list(np.diff(np.sort(np.concatenate([[0, M], rng.integers(0, M + 1, P - 1)]))))
    cs = synth.split_sizes(N, P)
    ii, jj, vv = [], [], []
    for r in range(P):
        n = int(rng.integers(0, 60))
        i, j, v = synth.random_coo(M, N, n, dup_frac=0.5, neg_frac=0.2, seed=seed * 100 + r)
        ii.append(i); jj.append(j); vv.append(v)
    A = oracle.OracleMat(M, N, rs, cs, ii, jj)
    A.set_values(vv, oracle.INSERT)
    D = numpy_dense(M, N, ii, jj, vv)
    assert np.array_equal(A.dense(), D)
    S = struct_pattern(M, N, ii, jj)
    assert sum(A.info(r, "nnz_d") + A.info(r, "nnz_o") for r in range(P)) == S.sum()
    x = synth.x_vector(0, N, "int", seed=seed).numpy()
    assert np.array_equal(A.mult(x), D @ x)
    A.set_values(vv, oracle.ADD)
    assert np.array_equal(A.dense(), 2 * D)


def test_range_error_names_k():
    i = np.array([0, -1, 5, 1, 7])
    j = np.array([0, 9, 1, 3, 0])
    with pytest.raises(oracle.OracleRangeError) as e:
        oracle.OracleMat(6, 4, [6], [4], [i], [j])
    assert (e.value.rank, e.value.k) == (0, 4)  # k=1 ignored (i<0 even though j>=N)
    with pytest.raises(oracle.OracleRangeError) as e:
        oracle.OracleMat(6, 4, [3, 3], [2, 2], [i[:2], np.array([2, 0, 4])], [j[:2], np.array([1, 4, 0])])
    assert (e.value.rank, e.value.k) == (1, 1)


def test_sample_rows_matches_full_p1():
    for values in ("int", "real"):
        shape = (9, 7, 6)
        M = int(np.prod(shape))
        A, ii, jj, vv = build_stencil(shape, 7, values=values)
        x = synth.x_vector(0, M, "real").numpy()
        y = A.mult(x)
        rows = np.array([0, 5, 17, 100, M - 1])
        ys = oracle.sample_rows(ii[0], jj[0], vv[0], rows, x)
        assert np.array_equal(ys, y[rows])
    i, j, v = synth.q1_coo(5, values="real")
    A = oracle.OracleMat(125, 125, [125], [125], [i], [j])
    A.set_values([v])
    x = synth.x_vector(0, 125, "real").numpy()
    rows = np.arange(0, 125, 7)
    assert np.array_equal(oracle.sample_rows(i, j, v, rows, x), A.mult(x)[rows])


@pytest.mark.parametrize("shape,npts", [((64, 64), 5), ((9, 7, 6), 7), ((7, 7, 7), 125), ((11, 3, 5), 27),
                                        ((9, 7, 6), 45)])
def test_csr_direct_equals_coo_assembly(shape, npts):
    """orc_csr_direct (the full-size timing path) is the COO definition specialised to
    duplicate-free, row-sorted COO: its CSR equals orc_create_coo + INSERT bit for bit, the
    numpy scatter-add brute force, and the stencil A.1 closed form (out-of-grid counts)."""
    M = int(np.prod(shape))
    for values in ("int", "real"):
        A, ii, jj, vv = build_stencil(shape, npts, values=values)
        C = oracle.OracleCsr(M, M, ii[0], jj[0], vv[0])
        assert C.nnz == A.info(0, "nnz_d")
        if npts == 45:  # box 5 x 3 x 3: per axis 5n-6 or 3n-2 in-grid (node, offset) pairs
            assert C.nnz == (5 * shape[0] - 6) * (3 * shape[1] - 2) * (3 * shape[2] - 2)
        assert np.array_equal(C.rowptr, A.export(0, "rowptr_d"))
        assert np.array_equal(C.col[:C.nnz], A.export(0, "col_d"))
        assert np.array_equal(C.val[:C.nnz].view(np.int64), A.export(0, "val_d").view(np.int64))
        x = synth.x_vector(0, M, values).numpy()
        assert np.array_equal(C.mult(x).view(np.int64), A.mult(x).view(np.int64))
        if M <= 500:
            D = numpy_dense(M, M, ii, jj, vv)
            dense = np.zeros((M, M))
            for q in range(M):
                dense[q, C.col[C.rowptr[q]:C.rowptr[q + 1]]] = C.val[C.rowptr[q]:C.rowptr[q + 1]]
            assert np.array_equal(dense, D)
    # A.1 closed form on the integer stencil: number of out-of-grid neighbours (P3)
    A, ii, jj, vv = build_stencil(shape, npts, values="int")
    C = oracle.OracleCsr(M, M, ii[0], jj[0], vv[0])
    offs = synth.stencil_offsets(len(shape), npts)
    g = np.arange(M)
    coords, rem = [], g
    for n in shape:
        coords.append(rem % n)
        rem = rem // n
    out = np.zeros(M)
    for o in offs:  # offsets are (d_slowest, ..., d_fastest), coords fastest first
        inside = np.ones(M, dtype=bool)
        for d, n in enumerate(shape):
            c = coords[d] + o[len(shape) - 1 - d]
            inside &= (c >= 0) & (c < n)
        out += ~inside
    assert np.array_equal(C.mult(np.ones(M)), out)


def test_csr_direct_refuses_other_coo():
    """Duplicates or unsorted entries are refused (ValueError), never assembled silently;
    negatives are skipped; out-of-range indices raise."""
    i, j, v = synth.q1_coo(4, values="real")  # element COO: duplicate positions
    with pytest.raises(ValueError):
        oracle.OracleCsr(64, 64, i, j, v)
    with pytest.raises(ValueError):
        oracle.OracleCsr(3, 3, np.array([0, 1, 0]), np.array([0, 0, 1]), np.ones(3))
    with pytest.raises(ValueError):
        oracle.OracleCsr(3, 3, np.array([0, 0]), np.array([2, 1]), np.ones(2))
    with pytest.raises(ValueError):
        oracle.OracleCsr(3, 3, np.array([0, 3]), np.array([0, 0]), np.ones(2))
    C = oracle.OracleCsr(4, 4, np.array([-1, 0, 2, 2, 3]), np.array([0, 1, -5, 3, 0]),
                         np.array([9.0, -0.0, 7.0, 2.0, 3.0]))
    assert C.nnz == 3 and list(C.rowptr) == [0, 1, 1, 2, 3]
    assert list(C.col[:3]) == [1, 3, 0]
    assert C.val[0] == 0.0 and not np.signbit(C.val[0])  # INSERT: +0.0 + (-0.0) = +0.0 (Z2)


@pytest.mark.parametrize("nthreads", [1, 2, 3, 8, 64])
def test_csr_mult_threads_bit_identical(nthreads):
    """The all-cores oracle leg (row slices over POSIX threads) gives orc_mult's y bit for bit,
    also with more threads than rows."""
    for shape, npts in (((20, 17, 9), 7), ((5, 3), 5), ((6, 6, 6), 27)):
        M = int(np.prod(shape))
        A, ii, jj, vv = build_stencil(shape, npts, values="real")
        C = oracle.OracleCsr(M, M, ii[0], jj[0], vv[0])
        x = synth.x_vector(0, M, "real").numpy()
        want = A.mult(x)
        assert np.array_equal(C.mult(x, nthreads=nthreads).view(np.int64), want.view(np.int64))
    # element COO (duplicates) through the general assembly, then the threaded row loop
    i, j, v = synth.q1_coo(6, values="real")
    A = oracle.OracleMat(216, 216, [216], [216], [i], [j])
    A.set_values([v])
    C = oracle.OracleCsr.from_oracle(A)
    x = synth.x_vector(0, 216, "real").numpy()
    assert np.array_equal(C.mult(x, nthreads=nthreads).view(np.int64), A.mult(x).view(np.int64))
    with pytest.raises(ValueError):
        C.mult(x, nthreads=0)


def test_spec_sf_reduce_examples():
    g = _parse_golden("spec_sf_examples.txt")
    t = g["reduce_pingpong_sum"].split()
    leaf = [float(v) for v in t[1:4]]
    root0 = [float(v) for v in t[5:8]]
    want = [float(v) for v in t[9:12]]
    leaves = [(None, [], []), (None, [0, 0, 0], [0, 1, 2])]
    out = oracle.sf_reduce([3, 0], leaves, [[], leaf], [root0, []], oracle.SUM)
    assert out[0].tolist() == want
    t = g["reduce_fanin"].split()
    lv = [float(t[1]), float(t[2])]
    for op, key in ((oracle.SUM, "sum"), (oracle.REPLACE, "replace")):
        out = oracle.sf_reduce([1], [(None, [0, 0], [0, 0])], [lv], [[0.0]], op)
        assert out[0].tolist() == [float(t[t.index(key) + 1])]


def test_sf_reduce_random_vs_python_walk():
    rng = np.random.default_rng(11)
    for trial in range(40):
        P = int(rng.integers(1, 5))
        nroots = [int(rng.integers(0, 10)) for _ in range(P)]
        owners = [q for q in range(P) if nroots[q] > 0]
        leaves, leafdata, rootdata = [], [], []
        for p in range(P):
            nl = int(rng.integers(0, 12)) if owners else 0
            space = nl + int(rng.integers(0, 3))
            il = rng.permutation(space)[:nl] if nl else np.zeros(0, np.int64)
            rr = rng.choice(owners, nl) if nl else np.zeros(0, np.int64)
            ro = np.array([rng.integers(0, nroots[q]) for q in rr], dtype=np.int64)
            leaves.append((il, rr, ro))
            leafdata.append(rng.integers(-50, 50, space).astype(float))
            rootdata.append(rng.integers(-50, 50, nroots[p]).astype(float))
        for op in (oracle.REPLACE, oracle.SUM):
            out = oracle.sf_reduce(nroots, leaves, leafdata, rootdata, op)
            want = [r.copy() for r in rootdata]
            # independent walk: contributions in ascending (source rank, leaf index)
            for p in range(P):
                il, rr, ro = leaves[p]
                for l in np.argsort(il, kind="stable"):
                    q, off = rr[l], ro[l]
                    c = leafdata[p][il[l]]
                    want[q][off] = c if op == oracle.REPLACE else want[q][off] + c
            for q in range(P):
                assert np.array_equal(out[q], want[q])


# ---------------------------------------------------------------- CG (NEXT #1) pins
def _spd_system(n=5, values="int", P=1):
    shape = (n, n)
    M = n * n
    A, *_ = build_stencil(shape, 5, P=P, values=values)
    return A, M


def test_cg_solves_spd_system():
    """After enough iterations CG's iterate solves A x = b (numpy.linalg.solve, independent)."""
    A, M = _spd_system(6)
    D = A.dense()
    b = synth.x_vector(0, M, "real", seed=3).numpy()
    x, hist = A.cg(b, np.zeros(M), 60)
    xs = np.linalg.solve(D, b)
    assert np.max(np.abs(x - xs)) <= 1e-10 * np.max(np.abs(xs))
    assert hist[-1] <= 1e-20 * hist[0]


def test_cg_first_step_closed_form():
    """x1 = x0 + (r0.r0 / r0.A r0) r0 with r0 = b - A x0, computed with numpy's dense matrix."""
    A, M = _spd_system(5)
    D = A.dense()
    b = synth.x_vector(0, M, "real", seed=4).numpy()
    x0 = synth.x_vector(0, M, "real", seed=5).numpy()
    r0 = b - D @ x0
    alpha = (r0 @ r0) / (r0 @ (D @ r0))
    x1, hist = A.cg(b, x0, 1)
    assert np.max(np.abs(x1 - (x0 + alpha * r0))) <= 1e-13 * np.max(np.abs(x1))
    assert abs(hist[0] - r0 @ r0) <= 1e-13 * (r0 @ r0)


def test_cg_energy_error_monotone():
    """||x - x_k||_A is non-increasing along CG iterations (textbook property)."""
    A, M = _spd_system(7)
    D = A.dense()
    b = synth.x_vector(0, M, "real", seed=6).numpy()
    xs = np.linalg.solve(D, b)
    prev = None
    for k in range(0, 25, 3):
        x, _ = A.cg(b, np.zeros(M), k)
        e = x - xs
        en = e @ (D @ e)
        if prev is not None:
            assert en <= prev * (1 + 1e-12)
        prev = en


def test_cg_partition_independent():
    """CG on the same global matrix simulated on 1 and 3 ranks: only the diag/off-diagonal
    split of MatMult's row sums differs (O5), so iterates agree to rounding."""
    A1, M = _spd_system(6, P=1)
    A3, _ = _spd_system(6, P=3)
    b = synth.x_vector(0, M, "int", seed=7).numpy()
    x1, h1 = A1.cg(b, np.zeros(M), 12)
    x3, h3 = A3.cg(b, np.zeros(M), 12)
    assert np.max(np.abs(x1 - x3)) <= 1e-12 * np.max(np.abs(x1))
    assert np.max(np.abs(h1 - h3) / h1) <= 1e-10
    assert h1[0] == h3[0]  # r0 = b - A*0 = b exactly


def test_cg_zero_rhs_stops():
    A, M = _spd_system(4)
    x, hist = A.cg(np.zeros(M), np.zeros(M), 5)
    assert np.all(x == 0) and np.all(hist == 0)


# ---------------------------------------------------------------- variants (NEXT #4)
@pytest.mark.parametrize("P,npts", [(2, 7), (4, 7), (8, 27), (3, 7)])
def test_box_decomposition_is_a_renumbering(P, npts):
    """Box (cube) partition with per-rank renumbering: permuting the
    assembled matrix back to natural order gives exactly the natural stencil matrix."""
    shape = (6, 4, 5) if P != 8 else (4, 4, 4)
    procs = synth.box_procs(P)
    sizes = synth.box_sizes(shape, procs)
    M = int(np.prod(shape))
    assert sum(sizes) == M
    ii, jj, vv = [], [], []
    for r in range(P):
        i, j, v = synth.stencil_coo_box(shape, npts, procs, r, values="real")
        ii.append(i); jj.append(j); vv.append(v)
    O = oracle.OracleMat(M, M, sizes, sizes, ii, jj)
    O.set_values(vv)
    g = torch.arange(M)
    nx, ny = shape[0], shape[1]
    perm = synth.box_global_id(g % nx, (g // nx) % ny, g // (nx * ny), shape, procs).numpy()
    assert sorted(perm.tolist()) == list(range(M))
    i1, j1, v1 = synth.stencil_coo(shape, npts, values="real")
    O1 = oracle.OracleMat(M, M, [M], [M], [i1], [j1])
    O1.set_values([v1])
    assert np.array_equal(O.dense()[np.ix_(perm, perm)], O1.dense())


def test_q2_125pt_nnz():
    """125-point (Q2-like) stencil: nnz = (5n - 6)^3 for an n^3 grid (closed form)."""
    for n in (3, 5, 6):
        i, j, v = synth.stencil_coo((n, n, n), 125)
        A = oracle.OracleMat(n ** 3, n ** 3, [n ** 3], [n ** 3], [i], [j])
        assert A.info(0, "nnz_d") == (5 * n - 6) ** 3


# ---------------------------------------------------------------- SPEC acceptance sizes
def _random_sf(rng, pmax, rmax, lmax):
    P = int(rng.integers(1, pmax + 1))
    nroots = [int(rng.integers(0, rmax)) for _ in range(P)]
    owners = [q for q in range(P) if nroots[q] > 0]
    leaves, rootdata, leafdata = [], [], []
    for p in range(P):
        nl = int(rng.integers(0, lmax)) if owners else 0
        space = nl + int(rng.integers(0, 4))
        il = rng.permutation(space)[:nl] if nl else np.zeros(0, np.int64)
        rr = rng.choice(owners, nl) if nl else np.zeros(0, np.int64)
        ro = np.array([rng.integers(0, nroots[q]) for q in rr], dtype=np.int64)
        leaves.append((il, rr, ro))
        rootdata.append(rng.integers(-50, 50, nroots[p]).astype(float))
        leafdata.append(rng.integers(-50, 50, space).astype(float))
    return P, nroots, leaves, rootdata, leafdata


def test_sf_acceptance_1000_random_graphs():
    """1,000 random SFs with up to 8 ranks (holes, fan-in, empty ranks); bcast and
    reduce, REPLACE and SUM, vs independent Python edge walks."""
    rng = np.random.default_rng(705)
    for trial in range(1000):
        P, nroots, leaves, rootdata, leafdata = _random_sf(rng, 8, 9, 9)
        for op in (oracle.REPLACE, oracle.SUM):
            out = oracle.sf_bcast(nroots, leaves, rootdata, leafdata, op)
            for p in range(P):
                want = leafdata[p].copy()
                il, rr, ro = leaves[p]
                for l in range(len(rr)):
                    val = rootdata[rr[l]][ro[l]]
                    want[il[l]] = val if op == oracle.REPLACE else want[il[l]] + val
                assert np.array_equal(out[p], want), (trial, op, p)
            out = oracle.sf_reduce(nroots, leaves, leafdata, rootdata, op)
            want = [r.copy() for r in rootdata]
            for p in range(P):
                il, rr, ro = leaves[p]
                for l in np.argsort(il, kind="stable"):
                    c = leafdata[p][il[l]]
                    want[rr[l]][ro[l]] = c if op == oracle.REPLACE else want[rr[l]][ro[l]] + c
            for q in range(P):
                assert np.array_equal(out[q], want[q]), (trial, op, q)


def test_random_coo_acceptance_500():
    """500 random COO instances (<= 50 % duplicates, <= 20 % negatives, up to 8
    ranks, uneven and empty ranks) vs a dense brute force: assembled matrix, INSERT then ADD,
    and MatMult exact in integers."""
    rng = np.random.default_rng(706)
    for trial in range(500):
        P = int(rng.integers(1, 9))
        M, N = int(rng.integers(1, 30)), int(rng.integers(1, 30))
        cuts = np.sort(rng.integers(0, M + 1, P - 1))
        rs = list(np.diff(np.concatenate([[0], cuts, [M]])).astype(int))
        cs = synth.split_sizes(N, P)
        ii, jj, vv = [], [], []
        for r in range(P):
            n = int(rng.integers(0, 40))
            i, j, v = synth.random_coo(M, N, n, dup_frac=float(rng.uniform(0, 0.5)),
                                       neg_frac=float(rng.uniform(0, 0.2)), seed=trial * 16 + r)
            ii.append(i); jj.append(j); vv.append(v)
        A = oracle.OracleMat(M, N, rs, cs, ii, jj)
        A.set_values(vv, oracle.INSERT)
        D = numpy_dense(M, N, ii, jj, vv)
        assert np.array_equal(A.dense(), D), trial
        x = synth.x_vector(0, N, "int", seed=trial).numpy()
        assert np.array_equal(A.mult(x), D @ x), trial
        A.set_values(vv, oracle.ADD)
        assert np.array_equal(A.dense(), 2 * D), trial


# ---------------------------------------------------------------- MatMultTranspose
@pytest.mark.parametrize("seed", range(20))
def test_mult_transpose_dense_and_partition(seed):
    """orc_mult_transpose = the dense A^T x (integer values: exact in any order), on random
    COO with uneven and empty ranks, for every partition of the same matrix."""
    rng = np.random.default_rng(900 + seed)
    M, N = int(rng.integers(1, 35)), int(rng.integers(1, 35))
    n = int(rng.integers(0, 150))
    i, j, v = synth.random_coo(M, N, n, dup_frac=0.4, neg_frac=0.15, seed=900 + seed)
    D = numpy_dense(M, N, [i], [j], [v])
    x = synth.x_vector(0, M, "int", seed=seed).numpy()
    for P in (1, 2, 3, 5):
        rs = synth.split_sizes(M, P)
        cs = synth.split_sizes(N, P)
        off = synth.offsets_from_sizes(rs)
        ii = [i[(i >= off[r]) & (i < off[r + 1])] for r in range(P)]
        jj = [j[(i >= off[r]) & (i < off[r + 1])] for r in range(P)]
        vv = [v[(i >= off[r]) & (i < off[r + 1])] for r in range(P)]
        A = oracle.OracleMat(M, N, rs, cs, ii, jj)
        A.set_values(vv)
        assert np.array_equal(A.mult_transpose(x), D.T @ x), (seed, P)


def test_mult_transpose_symmetric_stencil():
    """The Dirichlet 7-point Laplacian is symmetric: A^T x == A x bit for bit in integers, and
    <A^T x, z> == <x, A z> for the nonsymmetric Q1-mass-plus-random case."""
    n = 6
    M = n ** 3
    i, j, v = synth.stencil_coo((n, n, n), 7, values="int")
    P = 3
    rs = synth.split_sizes(M, P)
    off = synth.offsets_from_sizes(rs)
    ii = [i[(i >= off[r]) & (i < off[r + 1])] for r in range(P)]
    jj = [j[(i >= off[r]) & (i < off[r + 1])] for r in range(P)]
    vv = [v[(i >= off[r]) & (i < off[r + 1])] for r in range(P)]
    A = oracle.OracleMat(M, M, rs, rs, ii, jj)
    A.set_values(vv)
    x = synth.x_vector(0, M, "int", seed=3).numpy()
    assert np.array_equal(A.mult_transpose(x), A.mult(x))
    # adjoint identity on a nonsymmetric matrix (integers: exact)
    i2, j2, v2 = synth.random_coo(M, M, 3000, dup_frac=0.3, neg_frac=0.1, seed=77)
    B = oracle.OracleMat(M, M, [M], [M], [i2], [j2])
    B.set_values([v2])
    z = synth.x_vector(0, M, "int", seed=4).numpy()
    assert np.dot(B.mult_transpose(x), z) == np.dot(x, B.mult(z))
