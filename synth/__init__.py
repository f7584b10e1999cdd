"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module is the ONLY code both sides share (task rule ③).  It holds no arithmetic of the
method: it emits COO triplets ``(i, j, v)`` and vectors ``x`` -- the *inputs* of
``MatSetPreallocationCOO/MatSetValuesCOO/MatMult`` -- and nothing that
sorts, sums, splits or multiplies them.  Every generator is a pure function of
``(seed, global ids)`` so every rank count P sees the same global matrix and vector
(SURVEY.md §8(c) O2).  Generators are written with torch integer ops so that the same code
runs on the host (for the oracle) and on the device (for large benchmark inputs) and yields
bit-identical arrays on both.

Workload recipes (SURVEY.md §8 header table, BASELINE.json ``configs``):

* C1  2D 5-point Laplacian 64x64           -> ``stencil_coo((64, 64), 5, ...)``
* C2  3D 7-point Laplacian 128^3           -> ``stencil_coo((128,)*3, 7, ...)``
* C3  3D Q1 (27-point) element COO, 160^3 nodes, 159^3 hex elements, 64 entries per
      element as in PAPER.md L685-693 -> ``q1_coo(160, ...)``
* C4  3D 7-point 256^3 per GPU, z-slabs     -> ``stencil_coo((256, 256, 256*P), 7, rows=slab)``
* C5  3 dof/node 27-point node-block 200^3  -> ``elasticity_coo(200, ...)``

Out-of-grid stencil neighbours are emitted with ``j = -1`` (Dirichlet elimination through
PAPER.md L675-676: "negative indices ... will be ignored"), following the Listing-3 pattern
(PAPER.md L415-430): each row writes its entries at a fixed offset ``(row - lo) * S``.
"""
from __future__ import annotations

import torch

I64 = torch.int64
F64 = torch.float64

DEFAULT_SEED = 8646

# ----------------------------------------------------------------------------------------
# counter-based hash (splitmix64) on int64 tensors with two's-complement wrap-around
# ----------------------------------------------------------------------------------------


def _s64(c: int) -> int:
    """Reinterpret an unsigned 64-bit constant as a signed int64 literal."""
    return c - (1 << 64) if c >= (1 << 63) else c


_GOLDEN = _s64(0x9E3779B97F4A7C15)
_MUL1 = _s64(0xBF58476D1CE4E5B9)
_MUL2 = _s64(0x94D049BB133111EB)


def _lsr(z: torch.Tensor, k: int) -> torch.Tensor:
    """Logical right shift of an int64 tensor (torch's >> is arithmetic)."""
    return (z >> k) & ((1 << (64 - k)) - 1)


def splitmix64(z: torch.Tensor) -> torch.Tensor:
    z = z + _GOLDEN
    z = (z ^ _lsr(z, 30)) * _MUL1
    z = (z ^ _lsr(z, 27)) * _MUL2
    return z ^ _lsr(z, 31)


def hash_ids(seed: int, *ids: torch.Tensor) -> torch.Tensor:
    """Chain splitmix64 over (seed, id0, id1, ...); broadcasting like torch."""
    h = splitmix64(torch.full((), seed, dtype=I64, device=ids[0].device))
    for t in ids:
        h = splitmix64(h ^ t)
    return h


def unit_interval(h: torch.Tensor) -> torch.Tensor:
    """Top 53 bits of a hash -> float64 uniform in [0, 1)."""
    return _lsr(h, 11).to(F64) * (2.0 ** -53)


def uniform_pm1(h: torch.Tensor) -> torch.Tensor:
    """float64 uniform in [-1, 1) from a hash."""
    return 2.0 * unit_interval(h) - 1.0


# ----------------------------------------------------------------------------------------
# layouts (input choice: which rows each rank owns)
# ----------------------------------------------------------------------------------------


def split_sizes(M: int, P: int) -> list[int]:
    """PETSc-style default split: m_r = M//P + (r < M%P)."""
    return [M // P + (1 if r < M % P else 0) for r in range(P)]


def offsets_from_sizes(sizes) -> list[int]:
    out = [0]
    for s in sizes:
        out.append(out[-1] + int(s))
    return out


def slab_planes(nz: int, P: int) -> list[int]:
    """z-planes per rank: nz/P each, the remainder to the low ranks (exact when P divides nz)."""
    return [nz // P + (1 if r < nz % P else 0) for r in range(P)]


def slab_sizes(shape, P: int, dof: int = 1) -> list[int]:
    """z-slabs: whole planes per rank (nz/P when P divides nz, else the
    remainder to the low ranks), lexicographic rows."""
    plane = 1
    for s in shape[:-1]:
        plane *= s
    return [plane * k * dof for k in slab_planes(shape[-1], P)]


# ----------------------------------------------------------------------------------------
# stencil COO (C1, C2, C4)
# ----------------------------------------------------------------------------------------


def stencil_offsets(ndim: int, npts: int):
    """Neighbour offsets in ascending global-offset order (slowest axis first).

    Returned as a list of per-axis tuples ordered (d_slowest, ..., d_fastest)."""
    if npts == 2 * ndim + 1:
        offs = []
        for axis in range(ndim):  # -slowest ... -fastest
            o = [0] * ndim
            o[axis] = -1
            offs.append(tuple(o))
        offs.append(tuple([0] * ndim))
        for axis in reversed(range(ndim)):  # +fastest ... +slowest
            o = [0] * ndim
            o[axis] = 1
            offs.append(tuple(o))
        return offs
    if npts == 3 ** ndim:
        import itertools
        return [tuple(t) for t in itertools.product((-1, 0, 1), repeat=ndim)]
    if ndim == 3 and npts == 45:  # Bump_2911-density box: 3 x 3 planes x 5 along the fastest axis
        import itertools
        return [tuple(t) for t in itertools.product((-1, 0, 1), (-1, 0, 1), (-2, -1, 0, 1, 2))]
    if npts == 5 ** ndim:  # Q2-like: every node within distance 2 per axis
        import itertools
        return [tuple(t) for t in itertools.product((-2, -1, 0, 1, 2), repeat=ndim)]
    raise ValueError(f"unsupported stencil: ndim={ndim} npts={npts}")


def _coords(g: torch.Tensor, shape):
    """Lexicographic node id g = ix + nx*(iy + ny*iz) -> coords (fastest axis first)."""
    cs = []
    for n in shape:
        cs.append(g % n)
        g = g // n
    return cs


def _lex(cs, shape):
    g = torch.zeros_like(cs[0])
    for c, n in zip(reversed(cs), reversed(shape)):
        g = g * n + c
    return g


def stencil_coo(shape, npts: int, rows=None, values: str = "int", seed: int = DEFAULT_SEED,
                device="cpu"):
    """COO triplets of a Dirichlet-eliminated 5/7/9/27-point stencil.

    ``shape`` lists grid sizes fastest axis first, e.g. (nx, ny, nz).  ``rows=(lo, hi)``
    selects the generating rows (a rank's owned rows); entry ``k = (g - lo) * S + s``.
    ``rows`` may also be a 1-D tensor of row ids (entries in that order).
    values: "int"  -> Laplacian weights, centre 2*ndim (or 26 for 27-pt), neighbours -1
            "real" -> hash(seed, i, j) -> U(-1, 1)
    """
    ndim = len(shape)
    n_total = 1
    for s in shape:
        n_total *= s
    offs = stencil_offsets(ndim, npts)
    S = len(offs)
    if rows is None or isinstance(rows, tuple):
        lo, hi = (0, n_total) if rows is None else rows
        g = torch.arange(lo, hi, dtype=I64, device=device)
    else:  # explicit list of generating rows (sampled full-size parity checks)
        g = rows.to(device=device, dtype=I64)
    cs = _coords(g, shape)
    i = g.repeat_interleave(S)
    jcols = []
    for off in offs:  # off is (d_slowest, ..., d_fastest)
        d = list(reversed(off))  # fastest first, matches cs
        nc = [c + dd for c, dd in zip(cs, d)]
        inside = torch.ones_like(g, dtype=torch.bool)
        for c, n in zip(nc, shape):
            inside &= (c >= 0) & (c < n)
        jn = _lex([c.clamp(0, n - 1) for c, n in zip(nc, shape)], shape)
        jcols.append(torch.where(inside, jn, torch.full_like(jn, -1)))
    j = torch.stack(jcols, dim=1).reshape(-1)
    if values == "int":
        centre = float(npts - 1)
        w = torch.full((S,), -1.0, dtype=F64, device=device)
        w[offs.index(tuple([0] * ndim))] = centre
        v = w.repeat(g.numel())
    elif values == "real":
        v = uniform_pm1(hash_ids(seed, i, j))
    else:
        raise ValueError(values)
    return i, j, v


# ----------------------------------------------------------------------------------------
# Q1 hexahedral element COO (C3)
# ----------------------------------------------------------------------------------------

# Integer element matrices by popcount(a xor b) (derived there by 2x2x2
# Gauss quadrature on the unit cube): 12*K_Q1 and 216*M_Q1.
Q1_WEIGHTS = {"lap": (4.0, 0.0, -1.0, -1.0), "mass": (8.0, 4.0, 2.0, 1.0)}


def q1_coo(n: int, elems=None, variant: str = "lap", values: str = "int",
           seed: int = DEFAULT_SEED, device="cpu"):
    """Element-by-element COO of a Q1 operator on an n^3 node grid ((n-1)^3 elements).

    ``elems`` is (lo, hi) or a 1-D tensor of element ids e = ex + (n-1)*(ey + (n-1)*ez).
    Entry k = 64*e' + 8*a + b (e' = position of e in ``elems``), local node
    a = ax + 2*ay + 4*az, i = node(e, a), j = node(e, b) -- "entries in the same element
    matrix stored contiguously" with analytic offsets.
    """
    ne = n - 1
    if elems is None:
        e = torch.arange(0, ne ** 3, dtype=I64, device=device)
    elif isinstance(elems, tuple):
        e = torch.arange(elems[0], elems[1], dtype=I64, device=device)
    else:
        e = elems.to(device=device, dtype=I64)
    ex, ey, ez = e % ne, (e // ne) % ne, e // (ne * ne)
    a = torch.arange(8, dtype=I64, device=device)
    ax, ay, az = a & 1, (a >> 1) & 1, (a >> 2) & 1
    node = ((ex[:, None] + ax) + n * ((ey[:, None] + ay) + n * (ez[:, None] + az)))  # [E, 8]
    i = node[:, :, None].expand(-1, 8, 8).reshape(-1)
    j = node[:, None, :].expand(-1, 8, 8).reshape(-1)
    if values == "int":
        w = torch.tensor(Q1_WEIGHTS[variant], dtype=F64, device=device)
        pc = (a[:, None] ^ a[None, :])
        pc = (pc & 1) + ((pc >> 1) & 1) + ((pc >> 2) & 1)
        v = w[pc].reshape(1, 64).expand(e.numel(), 64).reshape(-1).clone()
    elif values == "real":
        ee = e[:, None, None].expand(-1, 8, 8).reshape(-1)
        aa = a[None, :, None].expand(e.numel(), -1, 8).reshape(-1)
        bb = a[None, None, :].expand(e.numel(), 8, -1).reshape(-1)
        v = uniform_pm1(hash_ids(seed, ee, aa * 8 + bb))
    else:
        raise ValueError(values)
    return i, j, v


def q1_slab_elems(n: int, P: int, r: int):
    """Elements generated by rank r under node z-slabs of n/P planes: those whose lowest
    node plane lies in the rank's slab (the top face then belongs to rank r+1, so the
    slab boundary produces off-rank COO rows that exercise the remote path)."""
    ne = n - 1
    planes = slab_planes(n, P)
    z0 = sum(planes[:r])
    z1 = min(z0 + planes[r], ne)
    return (z0 * ne * ne, max(z1, z0) * ne * ne)


# ----------------------------------------------------------------------------------------
# 3-dof node-block 27-point COO (C5)
# ----------------------------------------------------------------------------------------

B3 = ((4.0, 1.0, 1.0), (1.0, 4.0, 1.0), (1.0, 1.0, 4.0))


def elasticity_coo(n: int, nodes=None, values: str = "int", seed: int = DEFAULT_SEED,
                   device="cpu"):
    """3 dof/node, 27-point node coupling, 81 entries per row.

    Row ``3*node + c`` lists its 27 neighbours in ascending order and for each the 3 dofs d:
    ``j = 3*nbr + d`` (or -1 outside).  Integer values ``K27[offset] * B3[c][d]`` with K27 the
    tensor product of the 1-D weights (1, 4, 1) (centre 64, face 16, edge 4, corner 1).
    ``nodes=(lo, hi)`` are generating nodes; entry k = ((node-lo)*3 + c)*81 + 3*s + d.
    """
    shape = (n, n, n)
    lo, hi = (0, n ** 3) if nodes is None else nodes
    offs = stencil_offsets(3, 27)
    g = torch.arange(lo, hi, dtype=I64, device=device)
    cs = _coords(g, shape)
    jn_list, kw = [], []
    for off in offs:
        d = list(reversed(off))
        nc = [c + dd for c, dd in zip(cs, d)]
        inside = torch.ones_like(g, dtype=torch.bool)
        for c, nn in zip(nc, shape):
            inside &= (c >= 0) & (c < nn)
        jn = _lex([c.clamp(0, n - 1) for c in nc], shape)
        jn_list.append(torch.where(inside, jn, torch.full_like(jn, -1)))
        w = 1.0
        for dd in off:
            w *= 4.0 if dd == 0 else 1.0
        kw.append(w)
    nbr = torch.stack(jn_list, dim=1)  # [G, 27]
    c = torch.arange(3, dtype=I64, device=device)
    dd = torch.arange(3, dtype=I64, device=device)
    # [G, 3(c), 27(s), 3(d)]
    i = (3 * g[:, None, None, None] + c[None, :, None, None]).expand(-1, 3, 27, 3).reshape(-1)
    nb = nbr[:, None, :, None].expand(-1, 3, 27, 3)
    j = torch.where(nb >= 0, 3 * nb + dd[None, None, None, :], torch.full_like(nb, -1)).reshape(-1)
    if values == "int":
        K = torch.tensor(kw, dtype=F64, device=device)
        B = torch.tensor(B3, dtype=F64, device=device)
        blk = (B[:, None, :] * K[None, :, None])  # [3, 27, 3]
        v = blk.reshape(1, -1).expand(hi - lo, -1).reshape(-1).clone()
    elif values == "real":
        v = uniform_pm1(hash_ids(seed, i, j))
    else:
        raise ValueError(values)
    return i, j, v


# ----------------------------------------------------------------------------------------
# random COO (fuzz), vectors
# ----------------------------------------------------------------------------------------


def random_coo(M: int, N: int, n: int, dup_frac: float = 0.3, neg_frac: float = 0.1,
               values: str = "int", seed: int = DEFAULT_SEED, device="cpu"):
    """Random triplets with duplicates and negative (ignored) indices (SPEC.md L705-706
    style: <=50 % duplicates, <=20 % negatives).  Integer values lie in [-8, 8]."""
    gen = torch.Generator(device="cpu").manual_seed(seed)
    if n == 0:
        e = torch.empty(0, dtype=I64)
        return e.to(device), e.to(device), torch.empty(0, dtype=F64, device=device)
    nu = max(1, int(n * (1.0 - dup_frac)))
    iu = torch.randint(0, max(M, 1), (nu,), generator=gen, dtype=I64)
    ju = torch.randint(0, max(N, 1), (nu,), generator=gen, dtype=I64)
    pick = torch.randint(0, nu, (n,), generator=gen, dtype=I64)
    pick[:nu] = torch.arange(nu)
    perm = torch.randperm(n, generator=gen)
    i, j = iu[pick][perm], ju[pick][perm]
    neg = torch.rand(n, generator=gen) < neg_frac
    which = torch.rand(n, generator=gen) < 0.5
    i = torch.where(neg & which, torch.full_like(i, -1), i)
    j = torch.where(neg & ~which, torch.full_like(j, -3), j)
    if values == "int":
        v = torch.randint(-8, 9, (n,), generator=gen, dtype=I64).to(F64)
    else:
        v = torch.rand(n, generator=gen, dtype=F64) * 2.0 - 1.0
    return i.to(device), j.to(device), v.to(device)


def x_vector(lo: int, hi: int, values: str = "real", seed: int = DEFAULT_SEED, device="cpu"):
    """Global vector entries [lo, hi): real U(-1,1) from splitmix64(seed, g); int in
    [-2^20, 2^20]; ones; or the global index."""
    g = torch.arange(lo, hi, dtype=I64, device=device)
    if values == "real":
        return uniform_pm1(hash_ids(seed, g))
    if values == "int":
        h = hash_ids(seed, g)
        return (_lsr(h, 1) % (2 * (1 << 20) + 1) - (1 << 20)).to(F64)
    if values == "ones":
        return torch.ones(hi - lo, dtype=F64, device=device)
    raise ValueError(values)


# ----------------------------------------------------------------------------------------
# named configurations (BASELINE.json configs)
# ----------------------------------------------------------------------------------------

CONFIGS = {
    "c1": dict(kind="stencil", shape=(64, 64), npts=5, per_gpu=False),
    "c2": dict(kind="stencil", shape=(128, 128, 128), npts=7, per_gpu=False),
    "c3": dict(kind="q1", n=160, per_gpu=False),
    "c4": dict(kind="stencil", shape=(256, 256, 256), npts=7, per_gpu=True),
    "c5": dict(kind="elasticity", n=200, per_gpu=False),
    # variants: C4 per-GPU cubes in a box decomposition; Q2-like 125-point
    "c4b": dict(kind="box", local=(256, 256, 256), npts=7, per_gpu=True),
    "q2": dict(kind="stencil", shape=(96, 96, 96), npts=125, per_gpu=False),
    # the density of the paper's Bump_2911 (~3 M rows, ~128 M nonzeros):
    # a 45-point (5 x 3 x 3 box) stencil on 144^3 nodes -- 2.99 M rows, 132 M nonzeros
    "bump": dict(kind="stencil", shape=(144, 144, 144), npts=45, per_gpu=False),
}

CONFIG_TEXT = {
    "c1": "2D 5-point Laplacian 64x64 (4096 rows), COO assembly + MatMult",
    "c2": "3D 7-point Laplacian 128^3 (2.1M rows), fp64 AIJ",
    "c3": "3D Q1 27-point stencil 160^3 nodes, COO from per-element duplicates",
    "c4": "3D 7-point Laplacian 256^3 per GPU, z-slab MPIAIJ, weak scaling",
    "c5": "3D 3-dof 27-point elasticity-like 200^3, strong scaling",
    "c4b": "3D 7-point Laplacian 256^3 per GPU, box (cube) decomposition with renumbering",
    "q2": "3D 125-point (Q2-like) stencil 96^3",
    "bump": "3D 45-point (5x3x3 box) stencil 144^3: Bump_2911 density (2.99 M rows, 132 M nnz)",
}


def config_rows(name: str, P: int = 1) -> int:
    c = CONFIGS[name]
    if c["kind"] == "stencil":
        n = 1
        for s in c["shape"]:
            n *= s
        return n * (P if c["per_gpu"] else 1)
    if c["kind"] == "q1":
        return c["n"] ** 3
    if c["kind"] == "box":
        n = 1
        for sdim in config_shape(name, P):
            n *= sdim
        return n
    return 3 * c["n"] ** 3


def config_shape(name: str, P: int = 1):
    c = CONFIGS[name]
    if c["kind"] == "box":
        procs = box_procs(P)
        return tuple(l * p for l, p in zip(c["local"], procs))
    if c["kind"] != "stencil":
        raise ValueError(name)
    shape = list(c["shape"])
    if c["per_gpu"]:
        shape[-1] *= P
    return tuple(shape)


def config_rank_coo(name: str, P: int, r: int, values: str = "int", seed: int = DEFAULT_SEED,
                    device="cpu", q1_variant: str = "mass"):
    """(i, j, v, layout_sizes) that rank r of P feeds to create/set_values for config name.

    Stencil/elasticity configs: rank r generates exactly its own z-slab rows.  Q1: rank r
    generates the elements of its slab (rows on the upper face are remote)."""
    c = CONFIGS[name]
    if c["kind"] == "stencil":
        shape = config_shape(name, P)
        sizes = slab_sizes(shape, P)
        off = offsets_from_sizes(sizes)
        i, j, v = stencil_coo(shape, c["npts"], rows=(off[r], off[r + 1]), values=values,
                              seed=seed, device=device)
        return i, j, v, sizes
    if c["kind"] == "box":
        shape, procs = config_shape(name, P), box_procs(P)
        i, j, v = stencil_coo_box(shape, c["npts"], procs, r, values=values, seed=seed, device=device)
        return i, j, v, box_sizes(shape, procs)
    if c["kind"] == "q1":
        n = c["n"]
        sizes = slab_sizes((n, n, n), P)
        i, j, v = q1_coo(n, elems=q1_slab_elems(n, P, r), variant=q1_variant, values=values,
                         seed=seed, device=device)
        return i, j, v, sizes
    n = c["n"]
    sizes = slab_sizes((n, n, n), P, dof=3)
    off = offsets_from_sizes(sizes)
    i, j, v = elasticity_coo(n, nodes=(off[r] // 3, off[r + 1] // 3), values=values, seed=seed,
                             device=device)
    return i, j, v, sizes


# ----------------------------------------------------------------------------------------
# box (cube) decomposition with per-rank renumbering ("a cube of cells per
# rank"); SURVEY §8(e) variant.  Rank r = bx + px*(by + py*bz) owns the box of nodes
# [bx*nx/px, (bx+1)*nx/px) x ... and its nodes are numbered contiguously, lexicographically
# inside the box, after all nodes of ranks < r.  Halo faces are strided in the owner's
# numbering, so the owner must gather them (the SF pack path).
# ----------------------------------------------------------------------------------------


def box_procs(P: int):
    """px, py, pz for P ranks: 1 -> 1x1x1, 2 -> 2x1x1, 4 -> 2x2x1, 8 -> 2x2x2, else Px1x1."""
    return {1: (1, 1, 1), 2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)}.get(P, (P, 1, 1))


def _box_bounds(n, p, b):
    return (b * n) // p, ((b + 1) * n) // p


def box_sizes(shape, procs):
    px, py, pz = procs
    nx, ny, nz = shape
    sizes = []
    for bz in range(pz):
        for by in range(py):
            for bx in range(px):
                x0, x1 = _box_bounds(nx, px, bx)
                y0, y1 = _box_bounds(ny, py, by)
                z0, z1 = _box_bounds(nz, pz, bz)
                sizes.append((x1 - x0) * (y1 - y0) * (z1 - z0))
    return sizes


def _box_of(i, n, p):
    """Box index of coordinate i when [0, n) is cut at floor(k*n/p), k = 0..p."""
    bounds = torch.tensor([(k * n) // p for k in range(1, p)], dtype=I64, device=i.device)
    return torch.searchsorted(bounds, i, right=True) if p > 1 else torch.zeros_like(i)


def box_global_id(ix, iy, iz, shape, procs):
    """Natural coordinates -> global id under the box numbering (int64 tensors)."""
    px, py, pz = procs
    nx, ny, nz = shape
    sizes = box_sizes(shape, procs)
    offs = torch.tensor(offsets_from_sizes(sizes)[:-1], dtype=I64, device=ix.device)
    bx, by, bz = _box_of(ix, nx, px), _box_of(iy, ny, py), _box_of(iz, nz, pz)
    x0, y0, z0 = (bx * nx) // px, (by * ny) // py, (bz * nz) // pz
    lx = ((bx + 1) * nx) // px - x0
    ly = ((by + 1) * ny) // py - y0
    rank = bx + px * (by + py * bz)
    return offs[rank] + (ix - x0) + lx * ((iy - y0) + ly * (iz - z0))


def stencil_coo_box(shape, npts: int, procs, rank: int, values: str = "int",
                    seed: int = DEFAULT_SEED, device="cpu"):
    """Stencil COO of rank `rank` under the box decomposition (rows = its box's nodes in the
    box numbering; entry k = local_node * S + s).  Values: "int" Laplacian weights, or
    "real" hashed on the NATURAL (i, j) so every P sees the same operator."""
    px, py, pz = procs
    nx, ny, nz = shape
    bx, by, bz = rank % px, (rank // px) % py, rank // (px * py)
    x0, x1 = _box_bounds(nx, px, bx)
    y0, y1 = _box_bounds(ny, py, by)
    z0, z1 = _box_bounds(nz, pz, bz)
    lx, ly, lz = x1 - x0, y1 - y0, z1 - z0
    loc = torch.arange(lx * ly * lz, dtype=I64, device=device)
    ix = x0 + loc % lx
    iy = y0 + (loc // lx) % ly
    iz = z0 + loc // (lx * ly)
    offs = stencil_offsets(3, npts)
    S = len(offs)
    gi = box_global_id(ix, iy, iz, shape, procs)
    nat_i = ix + nx * (iy + ny * iz)
    i = gi.repeat_interleave(S)
    jcols, nat_j = [], []
    for off in offs:
        dz, dy, dx = off
        jx, jy, jz = ix + dx, iy + dy, iz + dz
        inside = (jx >= 0) & (jx < nx) & (jy >= 0) & (jy < ny) & (jz >= 0) & (jz < nz)
        g = box_global_id(jx.clamp(0, nx - 1), jy.clamp(0, ny - 1), jz.clamp(0, nz - 1), shape, procs)
        jcols.append(torch.where(inside, g, torch.full_like(g, -1)))
        nat_j.append(jx + nx * (jy + ny * jz))
    j = torch.stack(jcols, dim=1).reshape(-1)
    if values == "int":
        w = torch.full((S,), -1.0, dtype=F64, device=device)
        w[offs.index((0, 0, 0))] = float(npts - 1)
        v = w.repeat(loc.numel())
    else:
        nj = torch.stack(nat_j, dim=1).reshape(-1)
        v = uniform_pm1(hash_ids(seed, nat_i.repeat_interleave(S), nj))
    return i, j, v
