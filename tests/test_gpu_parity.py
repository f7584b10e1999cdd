"""GPU parity: libspmat (CUDA, through the C ABI) vs the CPU oracle on seeded inputs.

Bars (BASELINE.json north_star): COO structure, contribution plans and halo plans
bit-exact; integer-valued inputs bit-exact; fp64 real-valued SpMV within relative max-norm
1e-12.  Assembled values are bit-exact in real mode too (both sides
sum contributions in ascending (src, k) order, reading Z1).
"""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

TOL = 1e-12


@pytest.fixture(scope="module")
def sp():
    import paper_2406_08646_b200 as sp
    sp.load()
    return sp


@pytest.fixture(scope="module")
def comm(sp):
    torch.cuda.set_device(0)
    c = sp.Comm(device=0, nranks=1, rank=0)
    yield c
    c.close()


def dev(t):
    return t.to("cuda")


def rel_err(y, ref):
    ref = np.asarray(ref)
    d = np.max(np.abs(np.asarray(y) - ref)) if ref.size else 0.0
    s = np.max(np.abs(ref)) if ref.size else 0.0
    return d / s if s > 0 else d


def canon(a):
    """Canonicalise -0.0 -> +0.0 for bit comparisons (reading Z18)."""
    a = np.asarray(a, dtype=np.float64).copy()
    a[a == 0] = 0.0
    return a


def check_structure(A, O, r=0):
    """Structure, colmap and contribution plan bit-exact vs the oracle rank r."""
    assert np.array_equal(A.export("rowptr_d"), O.export(r, "rowptr_d"))
    assert np.array_equal(A.export("col_d"), O.export(r, "col_d"))
    assert np.array_equal(A.export("rowptr_o"), O.export(r, "rowptr_o"))
    assert np.array_equal(A.export("col_o"), O.export(r, "col_o"))
    assert np.array_equal(A.export("colmap"), O.export(r, "colmap"))
    assert np.array_equal(A.export("jmap"), O.export(r, "jmap"))
    assert np.array_equal(A.export("csrc"), O.export(r, "csrc"))


def run_single(sp, comm, M, N, i, j, v, x, mode_values=True):
    A = sp.Mat(comm, M, N, M, N, dev(i), dev(j))
    vd = dev(v)
    A.set_values(vd)
    xd = dev(x)
    yd = torch.empty(M, dtype=torch.float64, device="cuda")
    A.mult(xd, yd)
    torch.cuda.synchronize()
    return A, yd.cpu().numpy()


CASES = {
    "c1_5pt64": lambda values: (4096, 4096) + synth.stencil_coo((64, 64), 5, values=values),
    "7pt_ragged": lambda values: (40 * 37 * 23,) * 2 + synth.stencil_coo((40, 37, 23), 7, values=values),
    "q1_9": lambda values: (9 ** 3,) * 2 + synth.q1_coo(9, variant="lap", values=values),
    "q1mass_7": lambda values: (7 ** 3,) * 2 + synth.q1_coo(7, variant="mass", values=values),
    "el_6": lambda values: (3 * 6 ** 3,) * 2 + synth.elasticity_coo(6, values=values),
    "27pt_2d9": lambda values: (81, 81) + synth.stencil_coo((9, 9), 9, values=values),
    "q2_125pt": lambda values: (9 ** 3,) * 2 + synth.stencil_coo((9, 9, 9), 125, values=values),
    "bump_45pt": lambda values: (13 * 11 * 9,) * 2 + synth.stencil_coo((13, 11, 9), 45, values=values),
}


@pytest.mark.parametrize("values", ["int", "real"])
@pytest.mark.parametrize("case", list(CASES))
def test_single_rank_parity(sp, comm, case, values):
    M, N, i, j, v = CASES[case](values)
    O = oracle.OracleMat(M, N, [M], [N], [i], [j])
    O.set_values([v])
    x = synth.x_vector(0, N, values)
    A, y = run_single(sp, comm, M, N, i, j, v, x)
    check_structure(A, O)
    # assembled values: bit-exact (canonical (src,k) order on both sides)
    assert np.array_equal(canon(A.export("val_d")), canon(O.export(0, "val_d")))
    yo = O.mult(x.numpy())
    if values == "int":
        assert np.array_equal(canon(y), canon(yo))
    else:
        assert rel_err(y, yo) <= TOL
    info = A.info()
    assert info["nnz_d"] == O.info(0, "nnz_d") and info["n_ghost"] == 0
    A.close()


def test_small_matrices_take_the_direct_kernel(sp, comm):
    """Latency-bound sizes (C1: 0.3 MB) run the direct kernel, large ones the bulk-copy one."""
    M, N, i, j, v = CASES["c1_5pt64"]("int")
    A = sp.Mat(comm, M, N, M, N, dev(i), dev(j))
    assert A.info()["spmv_kernel_id"] == 5
    A.close()


def test_p1_pins_on_gpu(sp, comm):
    """Closed forms evaluated by the GPU path: A.1 and polynomial x (P3, P4)."""
    n = 33
    M = n ** 3
    i, j, v = synth.stencil_coo((n, n, n), 7)
    A = sp.Mat(comm, M, M, M, M, dev(i), dev(j))
    A.set_values(dev(v))
    g = torch.arange(M, device="cuda")
    ix, iy, iz = g % n, (g // n) % n, g // (n * n)
    y = torch.empty(M, dtype=torch.float64, device="cuda")
    A.mult(torch.ones(M, dtype=torch.float64, device="cuda"), y)
    want = sum(((c == 0) | (c == n - 1)).double() for c in (ix, iy, iz))
    assert torch.equal(y, want)
    A.mult((ix * ix + iy * iy + iz * iz).double(), y)
    interior = (ix > 0) & (ix < n - 1) & (iy > 0) & (iy < n - 1) & (iz > 0) & (iz < n - 1)
    assert torch.all(y[interior] == -6)
    A.close()


def test_nnz_closed_forms_gpu(sp, comm):
    for (M, i, j, want) in [
        (64 * 64, *synth.stencil_coo((64, 64), 5)[:2], 5 * 64 * 64 - 4 * 64),
        (20 ** 3, *synth.stencil_coo((20,) * 3, 7)[:2], 7 * 20 ** 3 - 6 * 20 ** 2),
        (10 ** 3, *synth.q1_coo(10)[:2], (3 * 10 - 2) ** 3),
        (3 * 5 ** 3, *synth.elasticity_coo(5)[:2], 9 * (3 * 5 - 2) ** 3),
    ]:
        A = sp.Mat(comm, M, M, M, M, dev(i), dev(j))
        assert A.info()["nnz_d"] == want
        A.close()


def test_random_coo_acceptance_500(sp, comm):
    """SPEC L706 on the GPU: 500 random COO instances (<= 50 % duplicates, <= 20 % negatives,
    empty ones included) -- structure, plans and values bit-exact vs the oracle, MatMult exact
    in integers."""
    rng = np.random.default_rng(7060)
    for trial in range(500):
        M, N = int(rng.integers(1, 80)), int(rng.integers(1, 80))
        n = int(rng.integers(0, 400))
        i, j, v = synth.random_coo(M, N, n, dup_frac=float(rng.uniform(0, 0.5)),
                                   neg_frac=float(rng.uniform(0, 0.2)), seed=50000 + trial)
        O = oracle.OracleMat(M, N, [M], [N], [i], [j])
        O.set_values([v])
        A = sp.Mat(comm, M, N, M, N, dev(i), dev(j))
        check_structure(A, O)
        A.set_values(dev(v))
        assert np.array_equal(canon(A.export("val_d")), canon(O.export(0, "val_d"))), trial
        x = synth.x_vector(0, N, "int", seed=trial)
        y = torch.empty(M, dtype=torch.float64, device="cuda")
        A.mult(dev(x), y)
        assert np.array_equal(canon(y.cpu().numpy()), canon(O.mult(x.numpy()))), trial
        A.close()


@pytest.mark.parametrize("seed", range(8))
def test_random_coo_fuzz(sp, comm, seed):
    rng = np.random.default_rng(seed)
    M, N = int(rng.integers(1, 300)), int(rng.integers(1, 300))
    n = int(rng.integers(0, 4000))
    i, j, v = synth.random_coo(M, N, n, dup_frac=0.5, neg_frac=0.2, seed=seed)
    O = oracle.OracleMat(M, N, [M], [N], [i], [j])
    O.set_values([v])
    A = sp.Mat(comm, M, N, M, N, dev(i), dev(j))
    check_structure(A, O)
    A.set_values(dev(v))
    assert np.array_equal(canon(A.export("val_d")), canon(O.export(0, "val_d")))
    x = synth.x_vector(0, N, "int", seed=seed)
    y = torch.empty(M, dtype=torch.float64, device="cuda")
    A.mult(dev(x), y)
    assert np.array_equal(canon(y.cpu().numpy()), canon(O.mult(x.numpy())))
    # ADD accumulates onto the INSERTed values
    A.set_values(dev(v), sp.ADD)
    O.set_values([v], oracle.ADD)
    assert np.array_equal(canon(A.export("val_d")), canon(O.export(0, "val_d")))
    A.close()


@pytest.mark.parametrize("kernel", ["tma", "direct"])
def test_long_rows(sp, comm, kernel, monkeypatch):
    """Rows longer than the row-block cap take the CTA-reduction path (bulk-copy kernel) or
    the lane loop (direct kernel)."""
    monkeypatch.setenv("SPMAT_SPMV_KERNEL", kernel)
    M, N = 50, 6000
    rows, cols = [], []
    for r in range(M):
        L = 5000 if r in (3, 17) else (700 if r == 30 else r % 9)
        rows.append(np.full(L, r))
        cols.append(np.random.default_rng(r).choice(N, L, replace=False))
    i = torch.from_numpy(np.concatenate(rows).astype(np.int64))
    j = torch.from_numpy(np.concatenate(cols).astype(np.int64))
    v = torch.from_numpy(np.random.default_rng(1).integers(-4, 5, i.numel()).astype(np.float64))
    O = oracle.OracleMat(M, N, [M], [N], [i], [j])
    O.set_values([v])
    A = sp.Mat(comm, M, N, M, N, dev(i), dev(j))
    A.set_values(dev(v))
    assert A.info()["max_row_nnz"] == 5000
    assert A.info()["spmv_kernel_id"] == {"tma": 3, "direct": 5}[kernel]
    for values in ("int", "real"):
        x = synth.x_vector(0, N, values)
        y = torch.empty(M, dtype=torch.float64, device="cuda")
        A.mult(dev(x), y)
        yo = O.mult(x.numpy())
        if values == "int":
            assert np.array_equal(y.cpu().numpy(), yo)
        else:
            assert rel_err(y.cpu().numpy(), yo) <= TOL
    A.close()


def test_spec_example_gpu(sp, comm):
    """SPEC.md L280-291 worked example through the GPU path."""
    i = torch.tensor([0, 0, 1, -1])
    j = torch.tensor([0, 1, 1, 2])
    v = torch.tensor([1.0, 2.0, 3.0, 9.0], dtype=torch.float64)
    A = sp.Mat(comm, 2, 3, 2, 3, dev(i), dev(j))
    A.set_values(dev(v))
    x = torch.tensor([1.0, 10.0, 100.0], dtype=torch.float64, device="cuda")
    y = torch.empty(2, dtype=torch.float64, device="cuda")
    A.mult(x, y)
    assert y.tolist() == [21.0, 30.0]
    A.set_values(dev(v), sp.ADD)
    A.set_values(dev(v), sp.ADD)
    A.mult(x, y)
    assert y.tolist() == [63.0, 90.0]
    A.close()


def test_host_pointers_and_memtype(sp, comm):
    """coo_i/j and x/y may be host memory (memtype detection)."""
    M = 20 * 20
    i, j, v = synth.stencil_coo((20, 20), 5, values="real")
    A = sp.Mat(comm, M, M, M, M, i.numpy(), j.numpy())
    A.set_values(dev(v))
    x = synth.x_vector(0, M, "real")
    xh = x.pin_memory()
    yh = torch.empty(M, dtype=torch.float64).pin_memory()
    A.mult(xh, yh)
    yd = torch.empty(M, dtype=torch.float64, device="cuda")
    A.mult(dev(x), yd)
    assert torch.equal(yh, yd.cpu())
    A.close()


def test_empty_and_degenerate(sp, comm):
    # no COO at all
    A = sp.Mat(comm, 5, 5, 5, 5, torch.empty(0, dtype=torch.int64, device="cuda"),
               torch.empty(0, dtype=torch.int64, device="cuda"))
    assert A.info()["nnz_d"] == 0
    A.set_values(torch.empty(0, dtype=torch.float64, device="cuda"))
    y = torch.full((5,), 7.0, dtype=torch.float64, device="cuda")
    A.mult(torch.ones(5, dtype=torch.float64, device="cuda"), y)
    assert torch.all(y == 0)
    A.close()
    # all entries negative
    i = torch.tensor([-1, -2, 0], device="cuda")
    j = torch.tensor([0, 1, -5], device="cuda")
    A = sp.Mat(comm, 3, 3, 3, 3, i, j)
    assert A.info()["nnz_d"] == 0
    A.close()
    # 0 x 0 matrix
    A = sp.Mat(comm, 0, 0, 0, 0, torch.empty(0, dtype=torch.int64, device="cuda"),
               torch.empty(0, dtype=torch.int64, device="cuda"))
    A.close()


def test_errors(sp, comm):
    i = torch.tensor([0, 1, 7, 1], device="cuda")
    j = torch.tensor([0, 1, 0, 9], device="cuda")
    with pytest.raises(sp.SpmatError) as e:
        sp.Mat(comm, 5, 5, 5, 5, i, j)
    assert e.value.status == sp.SPMAT_ERR_RANGE and "k=2" in e.value.message
    with pytest.raises(sp.SpmatError) as e:
        sp.Mat(comm, 4, 5, 5, 5, i[:2], j[:2])
    assert e.value.status == sp.SPMAT_ERR_MISMATCH
    A = sp.Mat(comm, 5, 5, 5, 5, i[:2], j[:2])
    x = torch.ones(5, dtype=torch.float64, device="cuda")
    with pytest.raises(sp.SpmatError) as e:
        A.mult(x, torch.empty_like(x))
    assert e.value.status == sp.SPMAT_ERR_STATE  # mult before set_values
    with pytest.raises(sp.SpmatError) as e:
        A.set_values(torch.ones(2, dtype=torch.float64, device="cuda"), sp.ADD)
    assert e.value.status == sp.SPMAT_ERR_STATE  # ADD before INSERT
    A.set_values(torch.ones(2, dtype=torch.float64, device="cuda"))
    with pytest.raises(sp.SpmatError) as e:
        A.mult(x, x)
    assert e.value.status == sp.SPMAT_ERR_ARG
    A.close()


def test_sf_single_rank(sp, comm):
    """Self-edge SF: fan-in, holes, REPLACE and SUM vs the oracle graph walk."""
    rng = np.random.default_rng(3)
    nroots, nleaves, space = 50, 40, 64
    il = rng.permutation(space)[:nleaves]
    ro = rng.integers(0, nroots, nleaves)
    root = torch.from_numpy(rng.integers(-9, 9, nroots).astype(np.float64))
    leaf0 = torch.from_numpy(rng.integers(-9, 9, space).astype(np.float64))
    sf = sp.StarForest(comm, nroots, il, np.zeros(nleaves), ro)
    for op in (sp.REPLACE, sp.SUM):
        want = oracle.sf_bcast([nroots], [(il, np.zeros(nleaves), ro)], [root.numpy()],
                               [leaf0.numpy()], op)[0]
        rd = dev(root)
        leaf = dev(leaf0)
        sf.bcast_begin(rd, leaf, op)
        sf.bcast_end(rd, leaf, op)
        assert np.array_equal(leaf.cpu().numpy(), want)
        # reduce leaf -> root in (rank, leaf index) order
        wantr = oracle.sf_reduce([nroots], [(il, np.zeros(nleaves), ro)], [leaf0.numpy()],
                                 [root.numpy()], op)[0]
        rd = dev(root)
        leaf = dev(leaf0)
        sf.reduce_begin(leaf, rd, op)
        sf.reduce_end(leaf, rd, op)
        assert np.array_equal(rd.cpu().numpy(), wantr)
    sf.close()
    with pytest.raises(sp.SpmatError):
        sp.StarForest(comm, 3, None, [0], [3])  # offset >= nroots


def test_sf_state_errors(sp, comm):
    sf = sp.StarForest(comm, 3, None, [0, 0, 0], [0, 1, 2])
    r = torch.arange(3, dtype=torch.float64, device="cuda")
    l = torch.zeros(3, dtype=torch.float64, device="cuda")
    with pytest.raises(sp.SpmatError) as e:
        sf.bcast_end(r, l)
    assert e.value.status == sp.SPMAT_ERR_STATE
    sf.bcast_begin(r, l, sp.REPLACE)
    with pytest.raises(sp.SpmatError) as e:
        sf.bcast_end(r, l, sp.SUM)
    assert e.value.status == sp.SPMAT_ERR_STATE
    sf.bcast_end(r, l, sp.REPLACE)
    assert l.tolist() == [0.0, 1.0, 2.0]
    sf.close()


def test_repeated_set_values_no_replan(sp, comm):
    """Repeated numeric assembly reuses the plan."""
    M = 30 * 30
    i, j, v = synth.stencil_coo((30, 30), 5, values="real")
    A = sp.Mat(comm, M, M, M, M, dev(i), dev(j))
    for s in range(3):
        A.set_values(dev(v * (s + 1)))
    assert A.info()["plan_builds"] == 1
    O = oracle.OracleMat(M, M, [M], [M], [i], [j])
    O.set_values([v * 3])
    assert np.array_equal(canon(A.export("val_d")), canon(O.export(0, "val_d")))
    # counters of spmat_get_info: calls, and no NCCL / NVLink bytes on one rank
    x = torch.ones(M, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    for _ in range(4):
        A.mult(x, y)
    info = A.info()
    assert info["n_set_values"] == 3 and info["n_mult"] == 4 and info["halo_mode"] == 0
    assert info["nccl_bytes_sent"] == info["nccl_bytes_recv"] == info["nvlink_bytes_put"] == 0
    assert info["block_size"] == 1 and info["spmv_grid"] >= 0
    A.close()


def test_determinism(sp, comm):
    M = 64 ** 3
    i, j, v = synth.stencil_coo((64, 64, 64), 7, values="real", device="cuda")
    A = sp.Mat(comm, M, M, M, M, i, j)
    A.set_values(v)
    x = synth.x_vector(0, M, "real", device="cuda")
    y1 = torch.empty(M, dtype=torch.float64, device="cuda")
    y2 = torch.empty_like(y1)
    A.mult(x, y1)
    A.mult(x, y2)
    assert torch.equal(y1, y2)
    A.close()


def _grid_coords(M, shape, dof=1):
    """Node coordinates (fastest axis first) of every row, on the device."""
    g = torch.arange(M, device="cuda") // dof
    out = []
    for n in shape:
        out.append(g % n)
        g = g // n
    return out


def closed_form_a1(cfg, M):
    """A.1 of the integer-valued config matrix over EVERY row:
    7-point stencil: number of out-of-grid neighbours; Q1 mass x216 element assembly:
    27 * prod_d (interior_d ? 2 : 1); 3-dof Kronecker K27 (x) B3: 6 * prod_d (4 + n_d), n_d the
    node's in-grid neighbours along d."""
    c = synth.CONFIGS[cfg]
    if c["kind"] == "stencil":
        shape = synth.config_shape(cfg, 1)
        return sum(((x == 0).double() + (x == n - 1).double())
                   for x, n in zip(_grid_coords(M, shape), shape))
    n = c["n"]
    if c["kind"] == "q1":
        w = torch.ones(M, dtype=torch.float64, device="cuda") * 27
        for x in _grid_coords(M, (n, n, n)):
            w = w * torch.where((x > 0) & (x < n - 1), 2.0, 1.0).double()
        return w
    w = torch.ones(M, dtype=torch.float64, device="cuda") * 6
    for x in _grid_coords(M, (n, n, n), dof=3):
        w = w * (4 + (x > 0).double() + (x < n - 1).double())
    return w


FULL = [("c2", 1), ("c3", 1), ("c4", 1), ("c5", 1), ("c5", 3)]


@pytest.mark.parametrize("cfg,bs", FULL)
def test_full_size(sp, comm, cfg, bs):
    """BASELINE configs at full size in the bench's launch configuration (persistent grid,
    every CTA wrapping its stage ring many times; C5 at 1.94 G COO entries, 1.92 G nonzeros,
    close to the int32 / 2^32 limits of the plan):
    * integer values: nnz closed form, and A.1 over EVERY row equal to the closed form
      (exact arithmetic, so bit-exact);
    * real values: sampled rows against the oracle computed one by one from the COO
      definition (oracle.sample_rows), relative max-norm <= 1e-12."""
    i, j, v, sizes = synth.config_rank_coo(cfg, 1, 0, values="int", device="cuda")
    M = sizes[0]
    A = sp.Mat(comm, M, M, M, M, i, j)
    del i, j
    if bs == 3:
        A.set_block_size(3)
    A.set_values(v)
    del v
    torch.cuda.empty_cache()
    nnz_want = {"c2": 7 * 128 ** 3 - 6 * 128 ** 2, "c3": (3 * 160 - 2) ** 3,
                "c4": 7 * 256 ** 3 - 6 * 256 ** 2, "c5": 9 * (3 * 200 - 2) ** 3}[cfg]
    info = A.info()
    assert info["nnz_d"] == nnz_want and info["nnz_o"] == 0
    assert info["spmv_kernel_id"] == (4 if bs == 3 else 3)
    y = torch.empty(M, dtype=torch.float64, device="cuda")
    A.mult(torch.ones(M, dtype=torch.float64, device="cuda"), y)
    want = closed_form_a1(cfg, M)
    bad = torch.nonzero(y != want)
    assert bad.numel() == 0, f"{bad.numel()} rows differ, first {bad[:5].flatten().tolist()}"
    del want
    # real values: refresh the values (same plan) and compare sampled rows with the oracle
    _, _, v, _ = synth.config_rank_coo(cfg, 1, 0, values="real", device="cuda")
    A.set_values(v)
    del v
    torch.cuda.empty_cache()
    x = synth.x_vector(0, M, "real", device="cuda")
    A.mult(x, y)
    xh = x.cpu().numpy()
    c = synth.CONFIGS[cfg]
    if c["kind"] == "stencil":
        rows = torch.unique(torch.cat([torch.randint(0, M, (1500,), generator=torch.Generator().manual_seed(5)),
                                       torch.tensor([0, 1, M // 2, M - 2, M - 1])]))
        ih, jh, vh = synth.stencil_coo(synth.config_shape(cfg, 1), 7, rows=rows, values="real")
        ys = oracle.sample_rows(ih, jh, vh, rows.numpy(), xh)
    elif c["kind"] == "q1":  # the elements touching the sampled rows' nodes
        n = c["n"]
        nodes = torch.unique(torch.cat([torch.randint(0, M, (300,), generator=torch.Generator().manual_seed(5)),
                                        torch.tensor([0, M // 2, M - 1])]))
        ix, iy, iz = nodes % n, (nodes // n) % n, nodes // (n * n)
        el = []
        for dz in (0, 1):
            for dy in (0, 1):
                for dx in (0, 1):
                    ex, ey, ez = ix - dx, iy - dy, iz - dz
                    ok = (ex >= 0) & (ex < n - 1) & (ey >= 0) & (ey < n - 1) & (ez >= 0) & (ez < n - 1)
                    el.append((ex + (n - 1) * (ey + (n - 1) * ez))[ok])
        elems = torch.unique(torch.cat(el))
        ih, jh, vh = synth.q1_coo(n, elems=elems, variant="mass", values="real")
        rows = nodes
        ys = oracle.sample_rows(ih, jh, vh, rows.numpy(), xh)
    else:  # node windows at the start, middle and end of the matrix
        n = c["n"]
        N = n ** 3
        parts_i, parts_j, parts_v, rws = [], [], [], []
        for a0 in (0, 40_000, N // 2 - 17, N - 64 * n - 5, N - 64):
            ih, jh, vh = synth.elasticity_coo(n, nodes=(a0, a0 + 64), values="real")
            parts_i.append(ih); parts_j.append(jh); parts_v.append(vh)
            rws.append(torch.arange(3 * a0, 3 * (a0 + 64)))
        rows = torch.unique(torch.cat(rws))
        ys = oracle.sample_rows(torch.cat(parts_i), torch.cat(parts_j), torch.cat(parts_v), rows.numpy(), xh)
    assert rel_err(y[rows.cuda()].cpu().numpy(), ys) <= TOL
    A.close()
    del x, y
    torch.cuda.empty_cache()


@pytest.mark.parametrize("values", ["int", "real"])
def test_every_row_many_blocks_per_cta(sp, comm, values):
    """~900 k rows (~3.4 k row blocks: several per persistent CTA, so every CTA wraps its
    2-stage ring and flips the mbarrier parities) compared with the full oracle on EVERY row."""
    shape = (96, 96, 96)
    M = 96 ** 3
    i, j, v = synth.stencil_coo(shape, 7, values=values)
    O = oracle.OracleMat(M, M, [M], [M], [i], [j])
    O.set_values([v])
    x = synth.x_vector(0, M, values)
    A, y = run_single(sp, comm, M, M, i, j, v, x)
    assert A.info()["spmv_kernel_id"] == 3
    yo = O.mult(x.numpy())
    if values == "int":
        assert np.array_equal(canon(y), canon(yo))
    else:
        assert rel_err(y, yo) <= TOL
    A.close()


@pytest.mark.parametrize("kernel", ["tma", "stream", "vector", "direct"])
@pytest.mark.parametrize("case", ["7pt_ragged", "q1_9", "el_6", "c1_5pt64"])
def test_kernel_variants(sp, comm, kernel, case, monkeypatch):
    """Every diagonal SpMV variant (chosen at create time) against the oracle."""
    monkeypatch.setenv("SPMAT_SPMV_KERNEL", kernel)
    M, N, i, j, v = CASES[case]("real")
    O = oracle.OracleMat(M, N, [M], [N], [i], [j])
    O.set_values([v])
    x = synth.x_vector(0, N, "real")
    A, y = run_single(sp, comm, M, N, i, j, v, x)
    assert A.info()["spmv_kernel_id"] == {"stream": 1, "vector": 2, "tma": 3, "direct": 5}[kernel]
    assert rel_err(y, O.mult(x.numpy())) <= TOL
    # integer mode is exact in any summation order
    vi = CASES[case]("int")[4]
    A.set_values(dev(vi))
    xi = synth.x_vector(0, N, "int")
    yd = torch.empty(M, dtype=torch.float64, device="cuda")
    A.mult(dev(xi), yd)
    O.set_values([vi])
    assert np.array_equal(canon(yd.cpu().numpy()), canon(O.mult(xi.numpy())))
    A.close()


@pytest.mark.parametrize("numeric", ["ilp", "plain", "seg", "seg-4", "warp", "pipe", "pipe4", "pipe8", "one", "ilp-jmap"])
def test_numeric_kernels(sp, comm, numeric, monkeypatch):
    """Every COO numeric kernel gives the oracle's values bit for bit (Z1 order), also with
    ~20 contributions per nonzero, and with one contribution per nonzero (stencil COO: jmap is
    the identity and is not read, unless SPMAT_NUMERIC_JMAP=1)."""
    monkeypatch.setenv("SPMAT_NUMERIC_KERNEL", numeric.split("-")[0])
    if numeric.endswith("jmap"):
        monkeypatch.setenv("SPMAT_NUMERIC_JMAP", "1")
    if numeric.endswith("4"):
        monkeypatch.setenv("SPMAT_NUMERIC_SEG", "4")
    for M, i, j, v in [(9 ** 3, *synth.q1_coo(9, values="real")),
                       (20 * 17 * 9, *synth.stencil_coo((20, 17, 9), 7, values="real")),
                       (50, *synth.random_coo(50, 50, 3000, dup_frac=0.9, neg_frac=0.1, values="real")),
                       (40, *synth.random_coo(40, 40, 30000, dup_frac=0.9, neg_frac=0.1, values="real"))]:
        O = oracle.OracleMat(M, M, [M], [M], [i], [j])
        O.set_values([v])
        A = sp.Mat(comm, M, M, M, M, dev(i), dev(j))
        A.set_values(dev(v))
        assert np.array_equal(canon(A.export("val_d")), canon(O.export(0, "val_d")))
        A.set_values(dev(v), sp.ADD)
        O.set_values([v], oracle.ADD)
        assert np.array_equal(canon(A.export("val_d")), canon(O.export(0, "val_d")))
        A.close()


def test_vec_dot_and_cg_single_rank(sp, comm):
    """VecDotAsync and CGAsync analogues vs the oracle."""
    n = 24
    M = n * n
    i, j, v = synth.stencil_coo((n, n), 5, values="int")
    A = sp.Mat(comm, M, M, M, M, dev(i), dev(j))
    A.set_values(dev(v))
    a = synth.x_vector(0, M, "int", seed=1)
    b = synth.x_vector(0, M, "int", seed=2)
    res = torch.zeros(1, dtype=torch.float64, device="cuda")
    A.dot(dev(a), dev(b), res)
    assert res.item() == float(np.dot(a.numpy(), b.numpy()))  # integer products: exact
    O = oracle.OracleMat(M, M, [M], [M], [i], [j])
    O.set_values([v])
    rhs = synth.x_vector(0, M, "real", seed=3)
    for iters in (1, 5, 40):
        x = torch.zeros(M, dtype=torch.float64, device="cuda")
        hist = torch.zeros(iters + 1, dtype=torch.float64, device="cuda")
        A.cg(dev(rhs), x, iters, hist)
        xo, ho = O.cg(rhs.numpy(), np.zeros(M), iters)
        assert rel_err(x.cpu().numpy(), xo) <= 1e-10
        assert np.max(np.abs(hist.cpu().numpy() - ho) / ho[0]) <= 1e-10
    # deterministic: the same call twice is bit-identical
    x1 = torch.zeros(M, dtype=torch.float64, device="cuda")
    x2 = torch.zeros(M, dtype=torch.float64, device="cuda")
    A.cg(dev(rhs), x1, 30)
    A.cg(dev(rhs), x2, 30)
    assert torch.equal(x1, x2)
    # converged: the GPU iterate solves the system (numpy, independent)
    xs = np.linalg.solve(O.dense(), rhs.numpy())
    x = torch.zeros(M, dtype=torch.float64, device="cuda")
    A.cg(dev(rhs), x, 200)
    assert rel_err(x.cpu().numpy(), xs) <= 1e-9
    A.close()


@pytest.mark.parametrize("shape,npts", [((24, 24), 5), ((13, 13, 13), 27), ((40, 40, 8), 7)])
def test_cg_persistent_matches_graph_path(sp, comm, shape, npts, monkeypatch):
    """The one-launch CG of small single-rank matrices (every iteration in a cooperative kernel
    with grid barriers) gives the two-kernel graph path's iterates and residual history bit for
    bit, also when iterations stop early (zero residual), and both agree with the oracle."""
    M = int(np.prod(shape))
    i, j, v = synth.stencil_coo(shape, npts, values="real")
    # symmetric positive definite: A + A^T + 2*npts*I built through ADD of the transposed COO
    ii = torch.cat([i, j, torch.arange(M)])
    jj = torch.cat([j, i, torch.arange(M)])
    vv = torch.cat([v, v, torch.full((M,), 2.0 * npts, dtype=torch.float64)])
    keep = (ii >= 0) & (jj >= 0)
    ii, jj, vv = ii[keep], jj[keep], vv[keep]
    O = oracle.OracleMat(M, M, [M], [M], [ii], [jj])
    O.set_values([vv])
    rhs = synth.x_vector(0, M, "real", seed=5)
    out = {}
    for persist in ("1", "0"):
        monkeypatch.setenv("SPMAT_CG_PERSIST", persist)
        A = sp.Mat(comm, M, M, M, M, dev(ii), dev(jj))
        A.set_values(dev(vv))
        res = []
        for iters in (1, 7, 60):
            x = torch.zeros(M, dtype=torch.float64, device="cuda")
            hist = torch.zeros(iters + 1, dtype=torch.float64, device="cuda")
            A.cg(dev(rhs), x, iters, hist)
            res.append((x.cpu(), hist.cpu()))
        # zero right-hand side: stopped from the start, x stays 0
        x0 = torch.zeros(M, dtype=torch.float64, device="cuda")
        h0 = torch.ones(4, dtype=torch.float64, device="cuda")
        A.cg(torch.zeros(M, dtype=torch.float64, device="cuda"), x0, 3, h0)
        res.append((x0.cpu(), h0.cpu()))
        out[persist] = res
        A.close()
    for (xa, ha), (xb, hb) in zip(out["1"], out["0"]):
        assert torch.equal(xa, xb) and torch.equal(ha, hb)
    xo, ho = O.cg(rhs.numpy(), np.zeros(M), 60)
    assert rel_err(out["1"][2][0].numpy(), xo) <= 1e-10
    assert np.max(np.abs(out["1"][2][1].numpy() - ho) / ho[0]) <= 1e-10
    assert not out["1"][3][0].any() and torch.equal(out["1"][3][1], torch.zeros(4, dtype=torch.float64))


def test_host_pipeline_matches_device(sp, comm):
    """Host x/y take the chunked upload/compute/download pipeline for large matrices; the
    result equals the device-pointer MatMult bit for bit."""
    i, j, v, sizes = synth.config_rank_coo("c2", 1, 0, values="real", device="cuda")
    M = sizes[0]
    A = sp.Mat(comm, M, M, M, M, i, j)
    A.set_values(v)
    x = synth.x_vector(0, M, "real", device="cuda")
    yd = torch.empty(M, dtype=torch.float64, device="cuda")
    A.mult(x, yd)
    xh = x.cpu().pin_memory()
    yh = torch.full((M,), float("nan"), dtype=torch.float64).pin_memory()
    for _ in range(2):
        A.mult(xh, yh)
        assert torch.equal(yh, yd.cpu())
    # asynchronous calls: 5 different x in flight through the two staging slots, one sync
    xs = [synth.x_vector(0, M, "real", seed=20 + k, device="cuda") for k in range(5)]
    want = []
    for xk in xs:
        A.mult(xk, yd)
        want.append(yd.cpu())
    xhs = [xk.cpu().pin_memory() for xk in xs]
    yhs = [torch.full((M,), float("nan"), dtype=torch.float64).pin_memory() for _ in xs]
    s = torch.cuda.current_stream()
    for xk, yk in zip(xhs, yhs):
        A.mult_async(xk, yk, s)
    s.synchronize()
    for yk, w in zip(yhs, want):
        assert torch.equal(yk, w)
    # pipelined calls (download waited for at the next call / flush), then values changed on
    # the stream right after a call: the SpMV of that call must still see the old values
    for yk in yhs:
        yk.fill_(float("nan"))
    for xk, yk in zip(xhs, yhs):
        A.mult_pipelined(xk, yk, s)
    A.flush(s)
    s.synchronize()
    for yk, w in zip(yhs, want):
        assert torch.equal(yk, w)
    A.mult_pipelined(xhs[0], yhs[0], s)
    A.set_values(v * 2, stream=s)  # ordered after the pipelined call's SpMV
    A.mult_pipelined(xhs[1], yhs[1], s)
    A.flush(s)
    s.synchronize()
    assert torch.equal(yhs[0], want[0]) and torch.equal(yhs[1], 2 * want[1])
    A.close()


@pytest.mark.parametrize("values", ["int", "real"])
def test_block_csr_3x3(sp, comm, values):
    """3x3 block-CSR SpMV (spmat_set_block_size) on the node-block elasticity matrix vs the
    oracle; values refreshed after set_values (INSERT and ADD); unblocked matrices refuse."""
    n = 7
    M = 3 * n ** 3
    i, j, v = synth.elasticity_coo(n, values=values)
    O = oracle.OracleMat(M, M, [M], [M], [i], [j])
    O.set_values([v])
    A = sp.Mat(comm, M, M, M, M, dev(i), dev(j))
    A.set_values(dev(v))
    x = synth.x_vector(0, M, values)
    y_csr = torch.empty(M, dtype=torch.float64, device="cuda")
    A.mult(dev(x), y_csr)
    A.set_block_size(3)
    assert A.info()["spmv_kernel_id"] == 4
    y = torch.empty(M, dtype=torch.float64, device="cuda")
    A.mult(dev(x), y)
    yo = O.mult(x.numpy())
    if values == "int":
        assert np.array_equal(canon(y.cpu().numpy()), canon(yo))
    else:
        assert rel_err(y.cpu().numpy(), yo) <= TOL
    A.set_values(dev(v), sp.ADD)  # the block copy follows the assembly
    O.set_values([v], oracle.ADD)
    A.mult(dev(x), y)
    assert rel_err(y.cpu().numpy(), O.mult(x.numpy())) <= TOL
    A.set_block_size(1)
    A.close()
    # set_values AFTER set_block_size(3): the numeric step writes the block copy directly
    # (k_numeric_bsr3); the CSR values are brought up to date on demand (export, transpose,
    # back to CSR) -- all bit-exact against the oracle's assembly (canonical order, Z1)
    O = oracle.OracleMat(M, M, [M], [M], [i], [j])
    O.set_values([v])
    A = sp.Mat(comm, M, M, M, M, dev(i), dev(j))
    A.set_block_size(3)
    for mode in (sp.INSERT, sp.ADD, sp.ADD):
        A.set_values(dev(v), mode)
        if mode == sp.ADD:
            O.set_values([v], oracle.ADD)
        A.mult(dev(x), y)
        yo = O.mult(x.numpy())
        if values == "int":
            assert np.array_equal(canon(y.cpu().numpy()), canon(yo))
        else:
            assert rel_err(y.cpu().numpy(), yo) <= TOL
    assert np.array_equal(canon(A.export("val_d")), canon(O.export(0, "val_d")))
    yt = torch.empty(M, dtype=torch.float64, device="cuda")
    A.set_values(dev(v), sp.ADD)
    O.set_values([v], oracle.ADD)
    A.mult_transpose(dev(x), yt)  # gathers the transposed values from the synced CSR copy
    assert rel_err(yt.cpu().numpy(), O.mult_transpose(x.numpy())) <= TOL
    A.set_values(dev(v), sp.ADD)
    O.set_values([v], oracle.ADD)
    A.set_block_size(1)  # back to CSR: val_d synced from the block copy
    A.mult(dev(x), y)
    assert rel_err(y.cpu().numpy(), O.mult(x.numpy())) <= TOL
    assert np.array_equal(canon(A.export("val_d")), canon(O.export(0, "val_d")))
    A.close()
    i, j, v = synth.stencil_coo((9, 9, 9), 7)
    B = sp.Mat(comm, 729, 729, 729, 729, dev(i), dev(j))
    with pytest.raises(sp.SpmatError) as e:
        B.set_block_size(3)
    assert e.value.status == sp.SPMAT_ERR_ARG
    B.close()


def test_cuda_graphs(sp, comm, monkeypatch):
    """MatMult is capturable in a (torch) CUDA graph, and the graph-replayed CG iteration
    equals the eagerly launched one bit for bit."""
    n = 40
    M = n ** 3
    i, j, v = synth.stencil_coo((n, n, n), 7, values="real")
    A = sp.Mat(comm, M, M, M, M, dev(i), dev(j))
    A.set_values(dev(v))
    x = synth.x_vector(0, M, "real", device="cuda")
    y0 = torch.empty(M, dtype=torch.float64, device="cuda")
    A.mult(x, y0)
    y = torch.zeros(M, dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        A.mult(x, y, s)  # warm-up on the capture stream
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        A.mult(x, y, s)
    y.zero_()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(y, y0)
    b = synth.x_vector(0, M, "real", seed=2, device="cuda")
    outs = []
    for flag in ("1", "0"):
        monkeypatch.setenv("SPMAT_GRAPH", flag)
        xg = torch.zeros(M, dtype=torch.float64, device="cuda")
        hist = torch.zeros(21, dtype=torch.float64, device="cuda")
        A.cg(b, xg, 20, hist)
        outs.append((xg.cpu(), hist.cpu()))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
    A.close()


@pytest.mark.parametrize("cfg", ["c2", "c3"])
def test_matmult_deterministic(sp, comm, cfg):
    """the dynamically scheduled SpMV is bitwise reproducible run to run (every row
    is summed by one fixed lane group in a fixed order, whichever CTA claims its block)."""
    i, j, v, sizes = synth.config_rank_coo(cfg, 1, 0, values="real", device="cuda")
    M = sizes[0]
    A = sp.Mat(comm, M, M, M, M, i, j)
    A.set_values(v)
    del i, j, v
    x = synth.x_vector(0, M, "real", device="cuda")
    y0 = torch.empty(M, dtype=torch.float64, device="cuda")
    y1 = torch.empty_like(y0)
    A.mult(x, y0)
    for _ in range(5):
        A.mult(x, y1)
        assert torch.equal(y0, y1)
    A.close()


def test_mult_transpose(sp, comm):
    """MatMultTranspose vs the oracle: bit-exact, real values included (same summation order),
    after a value refresh (ADD), on random, element (Q1) and rectangular matrices."""
    cases = [(9 ** 3, 9 ** 3, *synth.q1_coo(9, values="real"))]
    for seed in range(4):
        M, N = 40 + 13 * seed, 70 - 11 * seed
        cases.append((M, N, *synth.random_coo(M, N, 900, dup_frac=0.4, neg_frac=0.1, values="real",
                                              seed=400 + seed)))
    for M, N, i, j, v in cases:
        O = oracle.OracleMat(M, N, [M], [N], [i], [j])
        O.set_values([v])
        A = sp.Mat(comm, M, N, M, N, dev(i), dev(j))
        A.set_values(dev(v))
        x = synth.x_vector(0, M, "real", seed=5, device="cuda")
        y = torch.full((N,), float("nan"), dtype=torch.float64, device="cuda")
        A.mult_transpose(x, y)
        assert np.array_equal(canon(y.cpu().numpy()), canon(O.mult_transpose(x.cpu().numpy())))
        A.set_values(dev(v), sp.ADD)  # values change: the transposed copy is re-gathered
        O.set_values([v], oracle.ADD)
        A.mult_transpose(x, y)
        assert np.array_equal(canon(y.cpu().numpy()), canon(O.mult_transpose(x.cpu().numpy())))
        A.close()


def test_mult_transpose_errors(sp, comm):
    """spmat_mult_transpose: host arrays, aliasing and calls before set_values are refused."""
    n = 6
    M = n ** 3
    i, j, v = synth.stencil_coo((n, n, n), 7, values="int")
    A = sp.Mat(comm, M, M, M, M, dev(i), dev(j))
    x = torch.ones(M, dtype=torch.float64, device="cuda")
    y = torch.empty(M, dtype=torch.float64, device="cuda")
    with pytest.raises(sp.SpmatError) as e:
        A.mult_transpose(x, y)
    assert e.value.status == sp.SPMAT_ERR_STATE
    A.set_values(dev(v))
    with pytest.raises(sp.SpmatError) as e:
        A.mult_transpose(x.cpu(), y)
    assert e.value.status == sp.SPMAT_ERR_ARG
    with pytest.raises(sp.SpmatError) as e:
        A.mult_transpose(x, x)
    assert e.value.status == sp.SPMAT_ERR_ARG
    A.mult_transpose(x, y)  # symmetric Laplacian: A^T 1 = A 1 = out-of-grid neighbour counts
    y2 = torch.empty_like(y)
    A.mult(x, y2)
    assert torch.equal(y, y2)
    A.close()
