/*
 * oracle.c -- plain, slow, serial CPU oracle for the distributed MatMult hot path of
 * arXiv 2406.08646 (PETSc/TAO on GPU-based exascale systems).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code, header,
 * table or helper with the CUDA product path (paper_2406_08646_b200/csrc, include/).
 *
 * Compiled with gcc -O2 -ffp-contract=off (no FMA contraction, IEEE binary64
 * round-to-nearest-even, no reassociation) so every floating-point step below happens
 * exactly as written.
 *
 * What it computes, and where the paper defines it (PAPER.md line numbers, "P:n"):
 *
 *  - Layout: MPI parallel matrices are "distributed row-wise across MPI processes with
 *    diagonal (intra-process coupling) and off-diagonal (inter-process coupling) blocks
 *    stored separately as two sequential CSR matrices".  Rank r owns rows
 *    [rstart_r, rend_r) and columns [cstart_r, cend_r) (contiguous, ascending).
 *
 *  - COO assembly: "the assembled matrix A is defined as the sum of each contribution v[k]
 *    to entry a_{i[k],j[k]}"; "negative indices in i/j[] ... the corresponding
 *    entries will be ignored"; MatSetPreallocationCOO "analyzes indices ...,
 *    exchanges information about remote entries, finalizes the sparsity pattern of the
 *    diagonal and off-diagonal blocks ... and builds MPI communication plans";
 *    MatSetValuesCOO with v "of the same length and ... same order as i/j";
 *    "each entry ... is destined for the owned diagonal, owned off-diagonal block, or a
 *    send buffer".
 *
 *  - Star forest: "Leaves are locally indexed with integers, while roots are globally
 *    indexed via tuples of (owner rank, offset)"; Bcast "broadcasts root values
 *    to leaves" with op REPLACE or add.
 *
 *  - MatMult: y = A x with ghost x entries fetched through the halo SF (P:433-434,
 *    P:477-478), y_local = A_d x_local + A_o lvec.
 *
 *  - MatMultTranspose (what the SF reduce enables): lvec = A_o^T x, y = A_d^T x,
 *    then the halo SF reduces lvec into the owners' y with SUM (root value first, then the
 *    contributions in ascending source rank).
 *
 * Readings of points the paper leaves open:
 *  Z1  duplicate contributions are summed in ascending (src rank, k) order, one accumulator
 *      starting from +0.0;
 *  Z2  INSERT: a = +0.0 + sum;  ADD: a = a_old + sum;
 *  Z3  an entry is ignored when i < 0 OR j < 0;
 *  Z4  i >= M or j >= N is an error naming (rank, k), checked before anything else;
 *  Z5  diagonal block = columns in the rank's column ownership range;
 *  Z7  columns ascending within a row; colmap = sorted unique off-diagonal global columns;
 *  Z8  the MatMult halo is a REPLACE broadcast;
 *  O5  y_i = S_d, or S_d + S_o when the row has off-diagonal entries; S_d/S_o are
 *      left-to-right sums from +0.0 of separately rounded products.
 *
 * Multi-rank runs are simulated in-process: the oracle loops over ranks and moves data
 * between them by direct indexing (SURVEY.md §4 "Multi-rank without a cluster").
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_ERR_ARG 1
#define ORC_ERR_RANGE 2
#define ORC_ERR_STATE 3
#define ORC_ERR_OOM 5

typedef struct {
  int64_t i, j;
  int64_t src, k;
} orc_tuple;

typedef struct {
  int64_t rstart, rend, cstart, cend;
  /* diagonal block: CSR over owned rows x owned columns, local column ids */
  int64_t nnz_d;
  int64_t *rowptr_d, *col_d;
  double *val_d;
  /* off-diagonal block: CSR over owned rows (full rowptr) x ghost columns, columns are
     indices into colmap */
  int64_t nnz_o;
  int64_t *rowptr_o, *col_o;
  double *val_o;
  int64_t n_ghost;
  int64_t *colmap;
  /* contributions of every stored nonzero, block order = diag nonzeros (CSR order) then
     offdiag nonzeros (CSR order): jmap[z]..jmap[z+1] index csrc/ck */
  int64_t *jmap, *csrc, *ck, ncontrib;
  /* COO send plan of this rank: for each destination rank (ascending, != self) the k's it
     sends, ascending; send_count[P]; recv_count[P] = entries received from each src */
  int64_t *send_count, *send_k, nsend;
  int64_t *recv_count;
  /* halo SF: leaf g (0..n_ghost-1) -> (leaf_owner[g], leaf_offset[g]) */
  int64_t *leaf_owner, *leaf_offset;
  /* root side: for each requester rank p (ascending), root_count[p] offsets, concatenated */
  int64_t *root_count, *root_offsets, nroot_offsets;
  int values_set;
} orc_rank;

typedef struct {
  int P;
  int64_t M, N;
  int64_t *roff, *coff; /* P+1 */
  orc_rank *rk;
} orc_sys;

static int cmp_tuple(const void *a, const void *b) {
  const orc_tuple *x = (const orc_tuple *)a, *y = (const orc_tuple *)b;
  if (x->i != y->i) return x->i < y->i ? -1 : 1;
  if (x->j != y->j) return x->j < y->j ? -1 : 1;
  if (x->src != y->src) return x->src < y->src ? -1 : 1;
  if (x->k != y->k) return x->k < y->k ? -1 : 1;
  return 0;
}

static int cmp_i64(const void *a, const void *b) {
  int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* owner of global index g under offsets off[0..P]: the r with off[r] <= g < off[r+1]
   (plain linear scan; empty ranks are skipped naturally) */
static int owner_of(const int64_t *off, int P, int64_t g) {
  for (int r = 0; r < P; ++r)
    if (off[r] <= g && g < off[r + 1]) return r;
  return -1;
}

static void *xcalloc(size_t n, size_t s) { return calloc(n ? n : 1, s); }

void orc_destroy(orc_sys *S) {
  if (!S) return;
  for (int r = 0; r < S->P; ++r) {
    orc_rank *R = &S->rk[r];
    free(R->rowptr_d); free(R->col_d); free(R->val_d);
    free(R->rowptr_o); free(R->col_o); free(R->val_o);
    free(R->colmap); free(R->jmap); free(R->csrc); free(R->ck);
    free(R->send_count); free(R->send_k); free(R->recv_count);
    free(R->leaf_owner); free(R->leaf_offset);
    free(R->root_count); free(R->root_offsets);
  }
  free(S->rk); free(S->roff); free(S->coff); free(S);
}

/*
 * orc_create_coo: MatSetPreallocationCOO(A, n, i, j) on every simulated rank.
 *   P ranks, global sizes M x N, row offsets roff[P+1], column offsets coff[P+1].
 *   The COO of all ranks is concatenated: rank r owns entries [cooff[r], cooff[r+1]) of
 *   gi/gj, its local k = global position - cooff[r].
 *   On a range error returns ORC_ERR_RANGE and sets *bad_rank/*bad_k to the first offender
 *   (lowest rank, then lowest k).
 */
int orc_create_coo(int P, int64_t M, int64_t N, const int64_t *roff, const int64_t *coff,
                   const int64_t *cooff, const int64_t *gi, const int64_t *gj, orc_sys **out,
                   int64_t *bad_rank, int64_t *bad_k) {
  *out = NULL;
  if (P < 1 || M < 0 || N < 0) return ORC_ERR_ARG;
  if (roff[0] != 0 || roff[P] != M || coff[0] != 0 || coff[P] != N) return ORC_ERR_ARG;
  for (int r = 0; r < P; ++r)
    if (roff[r + 1] < roff[r] || coff[r + 1] < coff[r]) return ORC_ERR_ARG;

  /* Z4: range check before anything else */
  for (int r = 0; r < P; ++r)
    for (int64_t t = cooff[r]; t < cooff[r + 1]; ++t) {
      if (gi[t] < 0 || gj[t] < 0) continue; /* Z3: ignored, never an error */
      if (gi[t] >= M || gj[t] >= N) {
        *bad_rank = r;
        *bad_k = t - cooff[r];
        return ORC_ERR_RANGE;
      }
    }

  orc_sys *S = (orc_sys *)calloc(1, sizeof(orc_sys));
  S->P = P; S->M = M; S->N = N;
  S->roff = (int64_t *)malloc(sizeof(int64_t) * (P + 1));
  S->coff = (int64_t *)malloc(sizeof(int64_t) * (P + 1));
  memcpy(S->roff, roff, sizeof(int64_t) * (P + 1));
  memcpy(S->coff, coff, sizeof(int64_t) * (P + 1));
  S->rk = (orc_rank *)calloc(P, sizeof(orc_rank));

  /* 1. every rank routes its valid entries to the row owner; the send plan lists, per
        destination ascending, the k's ascending (a "send buffer") */
  for (int r = 0; r < P; ++r) {
    orc_rank *R = &S->rk[r];
    R->rstart = roff[r]; R->rend = roff[r + 1];
    R->cstart = coff[r]; R->cend = coff[r + 1];
    R->send_count = (int64_t *)xcalloc(P, sizeof(int64_t));
    R->recv_count = (int64_t *)xcalloc(P, sizeof(int64_t));
    R->root_count = (int64_t *)xcalloc(P, sizeof(int64_t));
    int64_t nsend = 0;
    for (int64_t t = cooff[r]; t < cooff[r + 1]; ++t) {
      if (gi[t] < 0 || gj[t] < 0) continue;
      int d = owner_of(roff, P, gi[t]);
      if (d != r) { R->send_count[d]++; nsend++; }
    }
    R->nsend = nsend;
    R->send_k = (int64_t *)xcalloc(nsend, sizeof(int64_t));
    int64_t w = 0;
    for (int d = 0; d < P; ++d) {
      if (d == r) continue;
      for (int64_t t = cooff[r]; t < cooff[r + 1]; ++t) {
        if (gi[t] < 0 || gj[t] < 0) continue;
        if (owner_of(roff, P, gi[t]) == d) R->send_k[w++] = t - cooff[r];
      }
    }
  }

  /* 2. on every owner: gather tuples (i, j, src, k) of all entries it owns, sort by the
        total order (i, j, src, k), unique (i, j) -> nonzeros (Z1, Z7) */
  for (int r = 0; r < P; ++r) {
    orc_rank *R = &S->rk[r];
    int64_t m = R->rend - R->rstart;
    int64_t nt = 0;
    for (int src = 0; src < P; ++src)
      for (int64_t t = cooff[src]; t < cooff[src + 1]; ++t)
        if (gi[t] >= 0 && gj[t] >= 0 && owner_of(roff, P, gi[t]) == r) nt++;
    orc_tuple *T = (orc_tuple *)xcalloc(nt, sizeof(orc_tuple));
    int64_t w = 0;
    for (int src = 0; src < P; ++src)
      for (int64_t t = cooff[src]; t < cooff[src + 1]; ++t)
        if (gi[t] >= 0 && gj[t] >= 0 && owner_of(roff, P, gi[t]) == r) {
          T[w].i = gi[t]; T[w].j = gj[t]; T[w].src = src; T[w].k = t - cooff[src];
          if (src != r) R->recv_count[src]++;
          w++;
        }
    qsort(T, nt, sizeof(orc_tuple), cmp_tuple);

    /* count nonzeros per row and block */
    R->rowptr_d = (int64_t *)xcalloc(m + 1, sizeof(int64_t));
    R->rowptr_o = (int64_t *)xcalloc(m + 1, sizeof(int64_t));
    int64_t nnz_d = 0, nnz_o = 0;
    for (int64_t a = 0; a < nt; ++a) {
      if (a > 0 && T[a].i == T[a - 1].i && T[a].j == T[a - 1].j) continue;
      int64_t lr = T[a].i - R->rstart;
      if (T[a].j >= R->cstart && T[a].j < R->cend) { R->rowptr_d[lr + 1]++; nnz_d++; }
      else { R->rowptr_o[lr + 1]++; nnz_o++; }
    }
    for (int64_t q = 0; q < m; ++q) {
      R->rowptr_d[q + 1] += R->rowptr_d[q];
      R->rowptr_o[q + 1] += R->rowptr_o[q];
    }
    R->nnz_d = nnz_d; R->nnz_o = nnz_o;
    R->col_d = (int64_t *)xcalloc(nnz_d, sizeof(int64_t));
    R->col_o = (int64_t *)xcalloc(nnz_o, sizeof(int64_t));
    R->val_d = (double *)xcalloc(nnz_d, sizeof(double));
    R->val_o = (double *)xcalloc(nnz_o, sizeof(double));

    /* colmap = sorted unique global off-diagonal columns (Z7) */
    int64_t *oc = (int64_t *)xcalloc(nnz_o, sizeof(int64_t));
    int64_t no = 0;
    for (int64_t a = 0; a < nt; ++a) {
      if (a > 0 && T[a].i == T[a - 1].i && T[a].j == T[a - 1].j) continue;
      if (!(T[a].j >= R->cstart && T[a].j < R->cend)) oc[no++] = T[a].j;
    }
    qsort(oc, no, sizeof(int64_t), cmp_i64);
    int64_t ng = 0;
    for (int64_t a = 0; a < no; ++a)
      if (a == 0 || oc[a] != oc[a - 1]) oc[ng++] = oc[a];
    R->n_ghost = ng;
    R->colmap = (int64_t *)xcalloc(ng, sizeof(int64_t));
    memcpy(R->colmap, oc, sizeof(int64_t) * ng);
    free(oc);

    /* fill columns and the contribution lists; nonzero z in block order: diag nonzeros
       first (CSR order), then offdiag nonzeros (CSR order) */
    int64_t nnz = nnz_d + nnz_o;
    int64_t *cnt = (int64_t *)xcalloc(nnz + 1, sizeof(int64_t));
    int64_t *zof = (int64_t *)xcalloc(nt, sizeof(int64_t)); /* tuple -> nonzero id */
    int64_t pd = 0, po = 0, z = -1;
    for (int64_t a = 0; a < nt; ++a) {
      int newnz = !(a > 0 && T[a].i == T[a - 1].i && T[a].j == T[a - 1].j);
      if (newnz) {
        if (T[a].j >= R->cstart && T[a].j < R->cend) {
          R->col_d[pd] = T[a].j - R->cstart;
          z = pd++;
        } else {
          /* binary search the ghost index of T[a].j in colmap */
          int64_t lo = 0, hi = ng - 1, g = -1;
          while (lo <= hi) {
            int64_t mid = lo + (hi - lo) / 2;
            if (R->colmap[mid] == T[a].j) { g = mid; break; }
            if (R->colmap[mid] < T[a].j) lo = mid + 1; else hi = mid - 1;
          }
          R->col_o[po] = g;
          z = nnz_d + po++;
        }
      }
      zof[a] = z;
      cnt[z + 1]++;
    }
    for (int64_t q = 0; q < nnz; ++q) cnt[q + 1] += cnt[q];
    R->jmap = cnt;
    R->ncontrib = nt;
    R->csrc = (int64_t *)xcalloc(nt, sizeof(int64_t));
    R->ck = (int64_t *)xcalloc(nt, sizeof(int64_t));
    int64_t *fill = (int64_t *)xcalloc(nnz + 1, sizeof(int64_t));
    for (int64_t a = 0; a < nt; ++a) { /* tuples are in (i,j,src,k) order within a nonzero */
      int64_t zz = zof[a];
      int64_t at = cnt[zz] + fill[zz]++;
      R->csrc[at] = T[a].src;
      R->ck[at] = T[a].k;
    }
    free(fill); free(zof); free(T);

    /* halo SF leaves: g -> (owner(colmap[g]), colmap[g] - cstart_owner) */
    R->leaf_owner = (int64_t *)xcalloc(ng, sizeof(int64_t));
    R->leaf_offset = (int64_t *)xcalloc(ng, sizeof(int64_t));
    for (int64_t g = 0; g < ng; ++g) {
      int q = owner_of(coff, P, R->colmap[g]);
      R->leaf_owner[g] = q;
      R->leaf_offset[g] = R->colmap[g] - coff[q];
    }
  }

  /* 3. root side of every halo SF: owner q lists, per requester p ascending, the offsets
        p's leaves request in p's leaf order */
  for (int q = 0; q < P; ++q) {
    orc_rank *Q = &S->rk[q];
    int64_t tot = 0;
    for (int p = 0; p < P; ++p) {
      orc_rank *Rp = &S->rk[p];
      for (int64_t g = 0; g < Rp->n_ghost; ++g)
        if (Rp->leaf_owner[g] == q) { Q->root_count[p]++; tot++; }
    }
    Q->nroot_offsets = tot;
    Q->root_offsets = (int64_t *)xcalloc(tot, sizeof(int64_t));
    int64_t w = 0;
    for (int p = 0; p < P; ++p) {
      orc_rank *Rp = &S->rk[p];
      for (int64_t g = 0; g < Rp->n_ghost; ++g)
        if (Rp->leaf_owner[g] == q) Q->root_offsets[w++] = Rp->leaf_offset[g];
    }
  }
  *out = S;
  return ORC_OK;
}

/*
 * orc_set_values_coo: MatSetValuesCOO(A, v, mode) on every rank.
 *   gv is the concatenation of every rank's v (same order as its i/j).
 *   mode 0 = INSERT (a = +0.0 + s), 1 = ADD (a = a_old + s)   (Z2)
 *   s = +0.0; for each contribution in ascending (src, k): s = s + v_src[k]   (Z1)
 */
int orc_set_values_coo(orc_sys *S, const int64_t *cooff, const double *gv, int mode) {
  if (!S) return ORC_ERR_STATE;
  if (mode != 0 && mode != 1) return ORC_ERR_ARG;
  for (int r = 0; r < S->P; ++r) {
    orc_rank *R = &S->rk[r];
    int64_t nnz = R->nnz_d + R->nnz_o;
    for (int64_t z = 0; z < nnz; ++z) {
      double s = +0.0;
      for (int64_t t = R->jmap[z]; t < R->jmap[z + 1]; ++t)
        s = s + gv[cooff[R->csrc[t]] + R->ck[t]];
      double *a = z < R->nnz_d ? &R->val_d[z] : &R->val_o[z - R->nnz_d];
      if (mode == 0) *a = +0.0 + s;
      else *a = *a + s;
    }
    R->values_set = 1;
  }
  return ORC_OK;
}

/*
 * orc_sf_bcast_halo: lvec_r[g] = x_{owner}[offset] for every rank's halo leaves
 * (REPLACE broadcast, Z8).  gx is the global x (concatenation of every rank's x).
 */
static void orc_halo(const orc_sys *S, int r, const double *gx, double *lvec) {
  const orc_rank *R = &S->rk[r];
  for (int64_t g = 0; g < R->n_ghost; ++g)
    lvec[g] = gx[S->coff[R->leaf_owner[g]] + R->leaf_offset[g]];
}

/*
 * orc_mult: y = A x, distributed form (O5).  gx: global x (length N), gy: global y (M).
 *   S_d = sum over diag entries left to right of (a * x_loc[c]),  from +0.0
 *   S_o = same over offdiag entries with lvec
 *   y_i = S_d if the row has no offdiag entries, else S_d + S_o
 */
int orc_mult(const orc_sys *S, const double *gx, double *gy) {
  if (!S) return ORC_ERR_STATE;
  for (int r = 0; r < S->P; ++r) {
    const orc_rank *R = &S->rk[r];
    if (!R->values_set && R->nnz_d + R->nnz_o > 0) return ORC_ERR_STATE;
    double *lvec = (double *)xcalloc(R->n_ghost, sizeof(double));
    orc_halo(S, r, gx, lvec);
    const double *xl = gx + R->cstart;
    int64_t m = R->rend - R->rstart;
    for (int64_t q = 0; q < m; ++q) {
      double sd = +0.0;
      for (int64_t t = R->rowptr_d[q]; t < R->rowptr_d[q + 1]; ++t) {
        double p = R->val_d[t] * xl[R->col_d[t]];
        sd = sd + p;
      }
      double y = sd;
      if (R->rowptr_o[q + 1] > R->rowptr_o[q]) {
        double so = +0.0;
        for (int64_t t = R->rowptr_o[q]; t < R->rowptr_o[q + 1]; ++t) {
          double p = R->val_o[t] * lvec[R->col_o[t]];
          so = so + p;
        }
        y = sd + so;
      }
      gy[R->rstart + q] = y;
    }
    free(lvec);
  }
  return ORC_OK;
}

/*
 * orc_mult_transpose: y = A^T x in PETSc's MPIAIJ order (MatMultTranspose; the halo star
 * forest used in reverse, PetscSFReduce with SUM).  gx: global x (length M, the row
 * layout), gy: global y (length N, the column layout).
 *   per rank:  y_loc[c] = sum over the rank's rows q ascending of a_d(q,c) * x[q], from +0.0
 *              lvec[g]  = same over the off-diagonal entries of ghost column g
 *   then, for every rank s ascending, the owner adds lvec_s[g] to y[colmap_s[g]]
 *   (SF reduce order: the root's value first, then ascending source rank).
 */
int orc_mult_transpose(const orc_sys *S, const double *gx, double *gy) {
  if (!S) return ORC_ERR_STATE;
  for (int r = 0; r < S->P; ++r) {
    const orc_rank *R = &S->rk[r];
    if (!R->values_set && R->nnz_d + R->nnz_o > 0) return ORC_ERR_STATE;
    for (int64_t c = R->cstart; c < R->cend; ++c) gy[c] = +0.0;
    const int64_t m = R->rend - R->rstart;
    for (int64_t q = 0; q < m; ++q)
      for (int64_t t = R->rowptr_d[q]; t < R->rowptr_d[q + 1]; ++t) {
        double p = R->val_d[t] * gx[R->rstart + q];
        gy[R->cstart + R->col_d[t]] = gy[R->cstart + R->col_d[t]] + p;
      }
  }
  for (int s = 0; s < S->P; ++s) {
    const orc_rank *R = &S->rk[s];
    double *lvec = (double *)xcalloc(R->n_ghost, sizeof(double));
    const int64_t m = R->rend - R->rstart;
    for (int64_t q = 0; q < m; ++q)
      for (int64_t t = R->rowptr_o[q]; t < R->rowptr_o[q + 1]; ++t) {
        double p = R->val_o[t] * gx[R->rstart + q];
        lvec[R->col_o[t]] = lvec[R->col_o[t]] + p;
      }
    for (int64_t g = 0; g < R->n_ghost; ++g) gy[R->colmap[g]] = gy[R->colmap[g]] + lvec[g];
    free(lvec);
  }
  return ORC_OK;
}

/* per-rank sizes: what = 0 rstart, 1 rend, 2 cstart, 3 cend, 4 nnz_d, 5 nnz_o, 6 n_ghost,
   7 ncontrib, 8 nsend, 9 nroot_offsets, 10 number of rows with offdiag entries */
int64_t orc_info(const orc_sys *S, int r, int what) {
  const orc_rank *R = &S->rk[r];
  switch (what) {
    case 0: return R->rstart;
    case 1: return R->rend;
    case 2: return R->cstart;
    case 3: return R->cend;
    case 4: return R->nnz_d;
    case 5: return R->nnz_o;
    case 6: return R->n_ghost;
    case 7: return R->ncontrib;
    case 8: return R->nsend;
    case 9: return R->nroot_offsets;
    case 10: {
      int64_t c = 0, m = R->rend - R->rstart;
      for (int64_t q = 0; q < m; ++q) c += R->rowptr_o[q + 1] > R->rowptr_o[q];
      return c;
    }
  }
  return -1;
}

/* copy a per-rank array out; returns elements copied.  int64 arrays unless noted:
   0 rowptr_d[m+1] 1 col_d 2 val_d(f64) 3 rowptr_o[m+1] 4 col_o 5 val_o(f64) 6 colmap
   7 jmap[nnz+1] 8 csrc 9 ck 10 send_count[P] 11 send_k 12 recv_count[P]
   13 leaf_owner 14 leaf_offset 15 root_count[P] 16 root_offsets */
int64_t orc_export(const orc_sys *S, int r, int what, void *buf) {
  const orc_rank *R = &S->rk[r];
  int64_t m = R->rend - R->rstart, nnz = R->nnz_d + R->nnz_o, P = S->P;
  const void *src = NULL;
  int64_t n = 0;
  switch (what) {
    case 0: src = R->rowptr_d; n = m + 1; break;
    case 1: src = R->col_d; n = R->nnz_d; break;
    case 2: src = R->val_d; n = R->nnz_d; break;
    case 3: src = R->rowptr_o; n = m + 1; break;
    case 4: src = R->col_o; n = R->nnz_o; break;
    case 5: src = R->val_o; n = R->nnz_o; break;
    case 6: src = R->colmap; n = R->n_ghost; break;
    case 7: src = R->jmap; n = nnz + 1; break;
    case 8: src = R->csrc; n = R->ncontrib; break;
    case 9: src = R->ck; n = R->ncontrib; break;
    case 10: src = R->send_count; n = P; break;
    case 11: src = R->send_k; n = R->nsend; break;
    case 12: src = R->recv_count; n = P; break;
    case 13: src = R->leaf_owner; n = R->n_ghost; break;
    case 14: src = R->leaf_offset; n = R->n_ghost; break;
    case 15: src = R->root_count; n = P; break;
    case 16: src = R->root_offsets; n = R->nroot_offsets; break;
    default: return -1;
  }
  if (buf && n) memcpy(buf, src, (size_t)n * 8);
  return n;
}

/*
 * orc_sf_bcast: brute-force graph walk of an explicit star forest (
 * SPEC.md L148 "brute-force graph walk").  For every rank p and leaf l:
 *   leaf_p[ilocal(l)]  = root_{rank(l)}[offset(l)]          (op 0, REPLACE)
 *   leaf_p[ilocal(l)] += root_{rank(l)}[offset(l)]          (op 1, SUM)
 * Arrays are concatenated over ranks: leaves of rank p are [lvoff[p], lvoff[p+1]);
 * ilocal may be NULL (identity); root data of rank q starts at rdoff[q]; leaf data of
 * rank p starts at ldoff[p].  Returns ORC_ERR_RANGE if an offset is outside the owner's
 * nroots = rdoff[q+1]-rdoff[q].
 */
int orc_sf_bcast(int P, const int64_t *lvoff, const int64_t *ilocal, const int64_t *rrank,
                 const int64_t *roffset, const int64_t *rdoff, const int64_t *ldoff,
                 const double *rootdata, double *leafdata, int op) {
  for (int p = 0; p < P; ++p)
    for (int64_t l = lvoff[p]; l < lvoff[p + 1]; ++l) {
      int64_t q = rrank[l];
      if (q < 0 || q >= P) return ORC_ERR_RANGE;
      if (roffset[l] < 0 || roffset[l] >= rdoff[q + 1] - rdoff[q]) return ORC_ERR_RANGE;
      int64_t li = ilocal ? ilocal[l] : l - lvoff[p];
      double rv = rootdata[rdoff[q] + roffset[l]];
      if (op == 0) leafdata[ldoff[p] + li] = rv;
      else leafdata[ldoff[p] + li] = leafdata[ldoff[p] + li] + rv;
    }
  return ORC_OK;
}

/*
 * orc_sf_reduce: brute-force walk of PetscSFReduce ("the latter reduces leaf
 * values into roots"), same array conventions as orc_sf_bcast.  Contributions to a root are
 * applied in ascending (source rank, leaf index) order (SPEC.md L139-141 reading):
 *   op 1 SUM:     root = root + leaf, one contribution at a time in that order
 *   op 0 REPLACE: root = the last contribution in that order
 * Leaf index = ilocal(l).  Roots nobody references are untouched.
 */
int orc_sf_reduce(int P, const int64_t *lvoff, const int64_t *ilocal, const int64_t *rrank,
                  const int64_t *roffset, const int64_t *rdoff, const int64_t *ldoff,
                  const double *leafdata, double *rootdata, int op) {
  for (int q = 0; q < P; ++q)        /* every root, in rank order */
    for (int64_t r = 0; r < rdoff[q + 1] - rdoff[q]; ++r)
      for (int p = 0; p < P; ++p) {  /* sources ascending */
        /* leaves of p on root (q, r), ascending leaf index: selection by repeated minimum */
        int64_t last = -1;
        for (;;) {
          int64_t best = -1, bestl = -1;
          for (int64_t l = lvoff[p]; l < lvoff[p + 1]; ++l) {
            if (rrank[l] != q || roffset[l] != r) continue;
            int64_t li = ilocal ? ilocal[l] : l - lvoff[p];
            if (li > last && (best < 0 || li < bestl)) { best = l; bestl = li; }
          }
          if (best < 0) break;
          double c = leafdata[ldoff[p] + bestl];
          double *root = &rootdata[rdoff[q] + r];
          *root = op == 0 ? c : *root + c;
          last = bestl;
        }
      }
  return ORC_OK;
}

/*
 * orc_sample_rows: y_i for a sorted list of sampled rows straight from the COO definition
 * A_ij = sum_k v[k] over entries with i[k]=i, j[k]=j, i,j >= 0,
 * for full-size parity checks where assembling the whole matrix on the host is too slow.
 * Per row the entries are gathered in k order, sorted stably by column (so duplicates keep
 * k order), summed per column from +0.0, and y_i = left-to-right sum over ascending columns
 * of a_ij * x_j.  (This is the P=1 summation order; at P>1 the row-split order differs,
 * so callers compare real-mode values with the 1e-12 tolerance.)
 */
typedef struct { int64_t j, k; double v; } orc_rowent;
static int cmp_rowent(const void *a, const void *b) {
  const orc_rowent *x = (const orc_rowent *)a, *y = (const orc_rowent *)b;
  if (x->j != y->j) return x->j < y->j ? -1 : 1;
  return x->k < y->k ? -1 : (x->k > y->k ? 1 : 0);
}
int orc_sample_rows(int64_t ncoo, const int64_t *gi, const int64_t *gj, const double *gv,
                    int64_t nsample, const int64_t *rows, const double *gx, double *yout) {
  /* rows must be sorted ascending and unique */
  int64_t *cnt = (int64_t *)xcalloc(nsample + 1, sizeof(int64_t));
  for (int64_t k = 0; k < ncoo; ++k) {
    if (gi[k] < 0 || gj[k] < 0) continue;
    int64_t lo = 0, hi = nsample - 1;
    while (lo <= hi) {
      int64_t mid = lo + (hi - lo) / 2;
      if (rows[mid] == gi[k]) { cnt[mid + 1]++; break; }
      if (rows[mid] < gi[k]) lo = mid + 1; else hi = mid - 1;
    }
  }
  for (int64_t s = 0; s < nsample; ++s) cnt[s + 1] += cnt[s];
  orc_rowent *E = (orc_rowent *)xcalloc(cnt[nsample], sizeof(orc_rowent));
  int64_t *fill = (int64_t *)xcalloc(nsample, sizeof(int64_t));
  for (int64_t k = 0; k < ncoo; ++k) {
    if (gi[k] < 0 || gj[k] < 0) continue;
    int64_t lo = 0, hi = nsample - 1;
    while (lo <= hi) {
      int64_t mid = lo + (hi - lo) / 2;
      if (rows[mid] == gi[k]) {
        orc_rowent *e = &E[cnt[mid] + fill[mid]++];
        e->j = gj[k]; e->k = k; e->v = gv[k];
        break;
      }
      if (rows[mid] < gi[k]) lo = mid + 1; else hi = mid - 1;
    }
  }
  for (int64_t s = 0; s < nsample; ++s) {
    orc_rowent *R = E + cnt[s];
    int64_t n = cnt[s + 1] - cnt[s];
    qsort(R, n, sizeof(orc_rowent), cmp_rowent);
    double y = +0.0;
    int64_t a = 0;
    while (a < n) {
      double aij = +0.0;
      int64_t b = a;
      while (b < n && R[b].j == R[a].j) { aij = aij + R[b].v; ++b; }
      double p = aij * gx[R[a].j];
      y = y + p;
      a = b;
    }
    yout[s] = y;
  }
  free(fill); free(E); free(cnt);
  return ORC_OK;
}

/*
 * orc_csr_direct: the COO definition A_ij = +0.0 + sum of v[k] (negatives ignored
 * P:675-676, INSERT reading Z2) for the special case of a COO whose valid entries are already
 * in CSR order with no duplicate positions: rows ascending, columns strictly ascending within
 * a row -- the Listing-3 stencil COO is of this form.  Every nonzero then has
 * exactly one contribution, so a_ij = +0.0 + v[k] and the CSR is the valid entries in input
 * order.  This is the "direct CSR generation" of SURVEY.md §8(d) for matrices too large for
 * the tuple sort of orc_create_coo (full-size oracle timing); any input not of that form is
 * refused with ORC_ERR_ARG (never silently assembled), an index >= M or >= N with ORC_ERR_RANGE.
 * rowptr: int64[M+1]; col: int64[>= valid entries]; val: f64[same]; *nnz_out = valid entries.
 */
int orc_csr_direct(int64_t M, int64_t N, int64_t ncoo, const int64_t *gi, const int64_t *gj,
                   const double *gv, int64_t *rowptr, int64_t *col, double *val, int64_t *nnz_out) {
  int64_t nnz = 0, row = 0, last_i = -1, last_j = -1;
  rowptr[0] = 0;
  for (int64_t k = 0; k < ncoo; ++k) {
    if (gi[k] < 0 || gj[k] < 0) continue;
    if (gi[k] >= M || gj[k] >= N) return ORC_ERR_RANGE;
    if (gi[k] < last_i || (gi[k] == last_i && gj[k] <= last_j)) return ORC_ERR_ARG;
    while (row < gi[k]) rowptr[++row] = nnz;  /* close rows up to gi[k] - 1 */
    col[nnz] = gj[k];
    val[nnz] = +0.0 + gv[k];
    ++nnz;
    last_i = gi[k];
    last_j = gj[k];
  }
  while (row < M) rowptr[++row] = nnz;
  *nnz_out = nnz;
  return ORC_OK;
}

/*
 * orc_csr_mult: y = A x for one rank's CSR with no off-diagonal block -- per row the same
 * left-to-right sum from +0.0 of separately rounded products as orc_mult's S_d (O5), so the
 * result is bit-identical to orc_mult.  nthreads > 1 splits the rows into nthreads contiguous
 * slices, one POSIX thread each, every row still computed by that same serial loop (the
 * "all host cores" leg of the oracle timed beside the GPU); the slicing
 * cannot change any value.  Timing aid only: the checks use orc_mult.
 */
typedef struct {
  int64_t r0, r1;
  const int64_t *rowptr, *col;
  const double *val, *x;
  double *y;
} orc_slice;

static void *orc_csr_rows(void *arg) {
  const orc_slice *s = (const orc_slice *)arg;
  for (int64_t q = s->r0; q < s->r1; ++q) {
    double sd = +0.0;
    for (int64_t t = s->rowptr[q]; t < s->rowptr[q + 1]; ++t) {
      double p = s->val[t] * s->x[s->col[t]];
      sd = sd + p;
    }
    s->y[q] = sd;
  }
  return NULL;
}

int orc_csr_mult(int64_t m, const int64_t *rowptr, const int64_t *col, const double *val,
                 const double *x, double *y, int nthreads) {
  if (nthreads < 1 || nthreads > 4096) return ORC_ERR_ARG;
  orc_slice *S = (orc_slice *)xcalloc((size_t)nthreads, sizeof(orc_slice));
  pthread_t *T = (pthread_t *)xcalloc((size_t)nthreads, sizeof(pthread_t));
  int st = ORC_OK, started = 0;
  for (int t = 0; t < nthreads; ++t) {
    S[t].r0 = m * t / nthreads;
    S[t].r1 = m * (t + 1) / nthreads;
    S[t].rowptr = rowptr; S[t].col = col; S[t].val = val; S[t].x = x; S[t].y = y;
  }
  if (nthreads == 1) {
    orc_csr_rows(&S[0]);
  } else {
    for (int t = 0; t < nthreads; ++t) {
      if (pthread_create(&T[t], NULL, orc_csr_rows, &S[t]) != 0) { st = ORC_ERR_OOM; break; }
      ++started;
    }
    for (int t = 0; t < started; ++t) pthread_join(T[t], NULL);
  }
  free(T); free(S);
  return st;
}

/* dot product, left to right from +0.0 (VecDot) */
static double orc_dot(int64_t n, const double *a, const double *b) {
  double s = +0.0;
  for (int64_t i = 0; i < n; ++i) {
    double p = a[i] * b[i];
    s = s + p;
  }
  return s;
}

/*
 * orc_cg: unpreconditioned conjugate gradients, the MatMult consumer of the paper's
 * CG/CGAsync experiment.  The paper fixes the structure -- MatMult, vector dot
 * products and AXPYs per iteration, a user-given maximum iteration count and no convergence
 * test inside the loop -- and leaves the iteration itself to the textbook
 * (Hestenes & Stiefel 1952), written out here step by step:
 *   r = b - A x;  p = r;  rr = r.r
 *   repeat maxit times:  q = A p;  alpha = rr / p.q;  x = x + alpha p;  r = r - alpha q;
 *                        rrn = r.r;  beta = rrn / rr;  p = r + beta p;  rr = rrn
 * A x uses orc_mult (the distributed MatMult of the simulated ranks).  rr_hist[k] = r_k.r_k
 * for k = 0..maxit.  If p.q or rr becomes exactly 0 the iteration stops (x, r unchanged) and
 * the remaining history repeats the last rr.  Requires a square matrix (M == N).
 */
int orc_cg(const orc_sys *S, const double *b, double *x, int maxit, double *rr_hist) {
  if (!S || S->M != S->N || maxit < 0) return ORC_ERR_ARG;
  const int64_t n = S->M;
  double *r = (double *)xcalloc(n, sizeof(double));
  double *p = (double *)xcalloc(n, sizeof(double));
  double *q = (double *)xcalloc(n, sizeof(double));
  int st = orc_mult(S, x, q);
  if (st != ORC_OK) { free(r); free(p); free(q); return st; }
  for (int64_t i = 0; i < n; ++i) {
    r[i] = b[i] - q[i];
    p[i] = r[i];
  }
  double rr = orc_dot(n, r, r);
  if (rr_hist) rr_hist[0] = rr;
  int stopped = 0;
  for (int k = 0; k < maxit; ++k) {
    if (!stopped) {
      orc_mult(S, p, q);
      double pq = orc_dot(n, p, q);
      if (pq == 0.0 || rr == 0.0) {
        stopped = 1;
      } else {
        double alpha = rr / pq;
        for (int64_t i = 0; i < n; ++i) {
          double t = alpha * p[i];
          x[i] = x[i] + t;
          double u = alpha * q[i];
          r[i] = r[i] - u;
        }
        double rrn = orc_dot(n, r, r);
        double beta = rrn / rr;
        for (int64_t i = 0; i < n; ++i) {
          double t = beta * p[i];
          p[i] = r[i] + t;
        }
        rr = rrn;
      }
    }
    if (rr_hist) rr_hist[k + 1] = rr;
  }
  free(r); free(p); free(q);
  return ORC_OK;
}
