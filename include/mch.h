/*
 * mch.h — C ABI of the B200-native hot path of hierarchical multicontinuum
 * homogenization (arXiv 2503.01276).
 *
 * The library computes, for every macropoint x_p of every level n of the
 * hierarchy, the constrained local cell problems of Eqs. (3)/(4) (level 1) and
 * the correction problems of Eqs. (12)/(13) (levels n >= 2) on the level-n FE
 * grid of mesh h*eta^(n-1), after the linear interpolation of preceding-level
 * solutions (Eq. 11), followed by the energy reductions of Eq. (7):
 *
 *   PAPER.md:147-170 (Eqs. 3-4), 171 (c_mj), 211-224 (Eq. 7),
 *   249-266 (Algorithm 1), 270-294 (S_n, Eq. 10), 366-374 (V_n),
 *   382-419 (Eqs. 11-13).
 *
 * Readings of the paper: vertex-centred
 * macropoints x_p = H*k, k in {0..M}^d (R1); R_p^+ = x_p +- (l+1/2)H clipped to
 * Omega, subcells = dual blocks of the vertices within l*H (R2); natural BC on
 * the window (R3); c_mj from K_p used in every R_q (R8); local-coordinate
 * transport of parents (R9); d-linear parents on T_{n-1} (R10); exact Galerkin
 * level operators (R11); Eq. (7) with prefactor 1 over K_p (R12); zero-measure
 * constraint rows dropped (R13).
 *
 * All entry points return 0 (MCH_OK) or a negative MCH_E* code; they never
 * throw.  mch_last_error() returns a message for the last failing call on the
 * context (or the last failed mch_create when ctx is NULL).  All device work is
 * ordered on params.stream (NULL = legacy default stream).
 */
#ifndef MCH_H_
#define MCH_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MCH_OK             0
#define MCH_EINVAL        -1  /* bad argument: d, N, n, M, L, eta, kappa <= 0 / non-finite, id >= N, sizes */
#define MCH_EDIVISIBILITY -2  /* M does not divide n; H/(2h) or H/(2h eta^(L-1)) not integer; eta^(L-1) does not divide M */
#define MCH_ERANK         -3  /* a continuum is absent from some K_p (c_mj undefined) */
#define MCH_ENOCONV       -4  /* projected PCG did not reach the tolerance within max_iter */
#define MCH_EORDER        -5  /* levels must be solved 1..L in order; coefficients need all levels */
#define MCH_ECUDA         -6  /* CUDA runtime failure */
#define MCH_ENOMEM        -7  /* device allocation failed */
#define MCH_EPLAN         -8  /* hierarchy cannot be built (no covering parent, reading R9) */
#define MCH_ENCCL         -9  /* NCCL unavailable or a collective failed (world > 1) */

typedef struct mch_ctx mch_ctx;

typedef struct {
  int      d;              /* 2 or 3 */
  int64_t  n;              /* fine cells per dimension; Omega = [0,1]^d, h = 1/n */
  int      num_continua;   /* N, 1..4 (continuum ids are 0..N-1) */
  int64_t  M;              /* macro cells per dimension, H = 1/M; (M+1)^d vertex macropoints */
  int      levels;         /* L >= 1 */
  int      eta;            /* coarsening factor >= 2 */
  int      oversample;     /* l >= 1: R_p^+ = x_p +- (l+1/2)H (BASELINE: 1, i.e. a 3H window) */
  double   rtol;           /* projected-residual tolerance of the PCG (default 1e-12 if <= 0) */
  int      max_iter;       /* PCG iteration cap (default 20000 if <= 0) */
  int      rank, world;    /* macropoint sharding across processes (one per GPU; world <= 1: all
                              macropoints here).  Each S_n (lexicographic order, i.e. slabs of the
                              macrogrid) is cut into `world` contiguous runs of near-equal work
                              (level-n window nodes); rank r solves run r (mch_shard_plan).
                              PAPER.md:201 (macropoints independent), 256-261 (levels in order). */
  int      keep_all;       /* 1: keep every macropoint's fine local solution (for
                              mch_local_solution); 0: keep only parents (T_{L-1}) */
  void*    stream;         /* cudaStream_t */
  int      interp;         /* interpolation of preceding levels (Eq. 11): MCH_INTERP_DLINEAR (0,
                              default) = d-linear on the corners of the T_{n-1} cell (reading
                              R10); MCH_INTERP_NEAREST_S1 (1) = the single nearest S_1 point,
                              weight 1, as in the paper's experiments, shifted to
                              the child in local coordinates (R9); MCH_INTERP_PHYSICAL_S1 (2) =
                              the nearest S_1 point evaluated at PHYSICAL coordinates, the level-1
                              windows enlarged by eta^(L-1)/2 layers to contain every child's
                              window (NEXT-4; d = 2, vertex layout) */
  int      layout;         /* macropoint layout: MCH_LAYOUT_VERTEX (0, default) = x_p = H k,
                              k in {0..M}^d (reading R1); MCH_LAYOUT_BLOCK (1) = block centres
                              x_p = (k + 1/2) H, k in {0..M-1}^d, K_p the block, T_n as in the
                              paper's Figures 2-3 */
  /* optional device allocator for every buffer the context owns (e.g. PyTorch's caching
     allocator, so the framework's pool holds the memory); both NULL: cudaMalloc / cudaFree.
     alloc(bytes, stream, alloc_user) returns a device pointer or NULL (-> MCH_ENOMEM);
     free(ptr, stream, alloc_user).  stream is params.stream. */
  void*  (*alloc)(size_t bytes, void* stream, void* user);
  void   (*free)(void* ptr, void* stream, void* user);
  void*    alloc_user;
  /* ncclComm_t of the `world` ranks (from mch_comm_init, or the caller's own), or NULL.  With a
     communicator and world > 1, mch_solve_level sends each level's parent solutions to the ranks
     whose children need them and mch_effective_coeffs / mch_load_vectors all-reduce, so both are
     collective and every rank returns the full results.  NULL with world > 1: no exchange (the
     caller moves pool slots itself, see mch_shard_plan / mch_pool_slot; tests). */
  void*    nccl_comm;
} mch_params;

#define MCH_INTERP_DLINEAR    0
#define MCH_INTERP_NEAREST_S1 1
#define MCH_INTERP_PHYSICAL_S1 2
#define MCH_LAYOUT_VERTEX     0
#define MCH_LAYOUT_BLOCK      1

typedef struct {
  int64_t  macropoints;    /* macropoints of this level solved by this context */
  int64_t  problems;       /* macropoints * N(1+d) right-hand sides */
  int64_t  iters_total;    /* sum of PCG iterations over problems */
  int64_t  iters_max;
  int64_t  unknowns_level; /* sum over macropoints of level-n nodes of the window */
  int64_t  cells_level;    /* sum over macropoints of level-n cells of the window */
  double   relres_max;     /* max final projected relative residual */
  double   ms_total;       /* device time of mch_solve_level(level) */
  double   ms_pcg;         /* device time of the PCG kernels */
  double   ms_setup;       /* device time of targets, operators, transport and projector setup */
  double   ms_gram;        /* device time of combine + Eq. (7) reductions */
  double   pcg_bytes;      /* algorithmic bytes moved by the PCG: see DESIGN.md §6 */
  int64_t  launches;       /* kernels launched by mch_solve_level(level) */
  int64_t  rank_deficient; /* windows whose level-n constraint rows were dependent (reading R20:
                              constraints imposed in the least-squares sense) */
  double   ms_comm;        /* device time of the parent exchange after this level (world > 1) */
  double   bytes_comm;     /* bytes this rank sent + received in that exchange */
  double   node_iters;     /* sum over problems of level-n window nodes x PCG iterations (the
                              solver work of the paper's cost model) */
  double   ms_transport;   /* device time of the transport (Eqs. 11-13: I_p, b, g), part of ms_setup */
  double   transport_units;/* fine window nodes x right-hand sides the transport processed */
  double   transport_flops;/* its algorithmic FP64 flops: per unit 2 npar (I_p) + 60 (the kappa-
                              weighted Q1 rows, z restriction, constraint sums) */
} mch_level_stats;

/* Algorithm 1 REQUIRE (macropoint set T, coarsening factor eta, fine mesh h,
 * levels L) with the medium kappa, psi_j.  Validate params and inputs, copy
 * kappa (float64, n^d, x fastest) and continuum ids (uint8, n^d, x fastest; psi_j = [id == j])
 * into library-owned device memory, build the hierarchy T_n / S_n (Eq. 10), the
 * parents of every macropoint (Eq. 11) and the sharding plan.  inputs_on_device: 1 if the
 * pointers are device pointers.  The caller keeps ownership of its buffers.  *out is NULL on error.
 * Errors: MCH_EINVAL, MCH_EDIVISIBILITY, MCH_EPLAN, MCH_ENOMEM, MCH_ECUDA, MCH_ENCCL. */
int mch_create(const mch_params* params, const double* kappa, const uint8_t* continuum_id,
               int inputs_on_device, mch_ctx** out);

/* Algorithm 1 lines 4-7 for level `level` (1..L, strictly in order): solve the
 * N(1+d) constrained problems of every macropoint of S_level owned by this
 * context and compute their Eq. (7) Gram matrices.  Stream-ordered; returns
 * after the level's device work is complete.  With params.nccl_comm and world > 1 it is
 * collective: afterwards every parent of S_level that a child on another rank needs has been
 * sent there (point-to-point NCCL, grouped).  Errors: MCH_EORDER, MCH_ERANK, MCH_ENOCONV
 * (message names macropoint, rhs, residual), MCH_ECUDA, MCH_ENCCL. */
int mch_solve_level(mch_ctx* ctx, int level);

/* Copy the Eq. (7) coefficients of all macropoints into out,
 * layout [P][n_rhs][n_rhs] with P = (M+1)^d (vertex layout) or M^d (block layout),
 * n_rhs = N(1+d), macropoints in
 * lexicographic vertex order (x fastest); G[a][b] = int_{K_p} kappa grad(Phi_a).grad(Phi_b)
 * with Phi = (phi_0..phi_{N-1}, phi_0^0..phi_0^{d-1}, .., phi_{N-1}^{d-1}), i.e.
 * B_ji = G[j][i], B^m_ji = G[j][N+i*d+m], Bbar^n_ji = G[N+j*d+n][i],
 * B^{mn}_ji = G[N+j*d+n][N+i*d+m].  Requires all levels (MCH_EORDER).  world > 1: with
 * params.nccl_comm the call is collective (all-reduce of the owner-only tensors, exact because
 * non-owned entries are 0) and returns every macropoint; without a communicator the entries of
 * macropoints owned by other ranks are 0.  Synchronises params.stream. */
int mch_effective_coeffs(mch_ctx* ctx, double* out, size_t out_len, int out_on_device);

/* Replace the medium of an existing context: validate and copy kappa (float64, n^d) and
 * continuum ids (uint8, n^d) exactly as mch_create does, keeping the hierarchy, the per-level
 * plans and all device buffers, and rewind the level counter (as mch_reset).  The coefficients
 * of the previous medium are discarded.  PAPER.md:124-125 (kappa, psi_j define the problem;
 * the macropoint hierarchy of Algorithm 1, depends only on the grid).  The
 * copy is ordered on params.stream; the call returns after the inputs were validated.  Errors:
 * MCH_EINVAL (NULL pointers, kappa <= 0 / non-finite, id >= N), MCH_ECUDA. */
int mch_set_medium(mch_ctx* ctx, const double* kappa, const uint8_t* continuum_id, int inputs_on_device);

/* NEXT-2 (upscaled system).  Source term f for the load vectors of Eq. (7) (PAPER.md:221,
 * b_j = |K_p|/|R_p| int_{R_p} f phi_j with R_p = K_p): float64, n^d, x fastest,
 * constant per fine cell (the paper's f, sampled at cell centres by the caller).
 * The loads are then computed alongside the Gram matrices of every level solved afterwards,
 * b_j(p) = sum_{cells e of K_p} f_e (h^d/2^d) sum_{corners a of e} phi_j(a) (exact for Q1 phi_j).
 * f = NULL removes the source.  Must be called before level 1 (or after mch_reset /
 * mch_set_medium): MCH_EORDER otherwise.  Errors: MCH_EINVAL (non-finite host f), MCH_ECUDA. */
int mch_set_source(mch_ctx* ctx, const double* f, int input_on_device);

/* Copy the load vectors b[P][N] (macropoints in lexicographic order, P as for the coefficients;
 * entries of macropoints owned by other ranks are 0).  Errors: MCH_EINVAL (no source, out_len <
 * P*N), MCH_EORDER (levels missing). */
int mch_load_vectors(mch_ctx* ctx, double* out, size_t out_len, int out_on_device);

/* Solve the upscaled system, Eq. (6), through its bilinear form with U_i,
 * V_j and their gradients taken at the block midpoints, on the block-centred layout only
 * (MCH_EINVAL otherwise): U_i continuous Q1 on the coarse vertex grid {0..M}^d, U_i = 0 on the
 * boundary (Eq. 1), a(U,V) = sum_p t_p(V)^T G_p t_p(U) with t_p = (U_0..U_{N-1}, grad U_0, ..,
 * grad U_{N-1}) at x_p, l(V) = sum_p sum_j V_j(x_p) b_j(p) (reading R23).  G
 * [P][n_rhs][n_rhs] and b [P][N] as returned by mch_effective_coeffs / mch_load_vectors; pass
 * both NULL to use this context's own (world == 1, all levels solved, source set).
 * inputs_on_device applies to G and b.  U receives [N][(M+1)^d] nodal values (x fastest).
 * Deterministic one-CTA Jacobi-PCG to ||r|| <= rtol ||F|| (rtol <= 0: 1e-12; max_iter <= 0:
 * 100000); *iters (may be NULL) receives the iteration count.  Errors: MCH_EINVAL, MCH_EORDER,
 * MCH_ENOCONV (tolerance not reached), MCH_ECUDA. */
int mch_macro_solve(mch_ctx* ctx, const double* G, const double* b, int inputs_on_device, double* U,
                    size_t U_len, int out_on_device, double rtol, int max_iter, int* iters);

/* NEXT-3 (validation workload).  Global fine-grid reference solution of Eq. (2):
 * u in Q1 on the n^d fine cells of Omega = [0,1]^d, u = 0 on the boundary (Eq. 1), with this
 * context's kappa and the cellwise source f (float64, n^d, x fastest; f_on_device as for kappa).
 * u receives the (n+1)^d nodal values (x fastest).  Matrix-free Jacobi-PCG in fp64, one
 * persistent cooperative kernel, to ||r|| <= rtol ||F|| (rtol <= 0: 1e-10; max_iter <= 0: 10^6);
 * *iters (may be NULL) receives the iteration count.  Deterministic for a given GPU model (the
 * grid is sized from the SM count).  Errors: MCH_EINVAL, MCH_ENOCONV, MCH_ECUDA. */
int mch_fine_solve(mch_ctx* ctx, const double* f, int f_on_device, double* u, size_t u_len, int u_on_device,
                   double rtol, int max_iter, int* iters);

/* Fine block averages of the error metric e_2: out[p][i] =
 * (1/|K_p cap Omega_i|) int_{K_p cap Omega_i} u for the (n+1)^d nodal Q1 field u (e.g. from
 * mch_fine_solve), Omega_i = the cells of continuum i, K_p as for the coefficients (block or
 * clipped dual block); NaN where K_p holds no cell of continuum i.  out [P][N].  Errors:
 * MCH_EINVAL, MCH_ECUDA. */
int mch_fine_block_averages(mch_ctx* ctx, const double* u, int u_on_device, double* out, size_t out_len,
                            int out_on_device);

/* Rewind the level counter so the same context (inputs, plan, pool, scratch) solves levels
 * 1..L again — for repeated runs (benchmarks, serving) without re-creating the context. */
int mch_reset(mch_ctx* ctx);

/* |S_level| (all ranks). */
int mch_num_macropoints(const mch_ctx* ctx, int level, int64_t* count);

/* Lexicographic indices of S_level in solve order (position i is owned by rank i mod world). */
int mch_level_macropoints(const mch_ctx* ctx, int level, int64_t* out, size_t cap);

/* Fine-grid combined local solution phi_p (Eq. 11) of macropoint `macropoint`
 * (lexicographic vertex index) for right-hand side `rhs` on its clipped window,
 * x fastest; ext receives the node counts per dimension.  Available for
 * parents (T_{L-1}) or, with keep_all, for every solved macropoint. */
int mch_local_solution(mch_ctx* ctx, int64_t macropoint, int rhs, double* out, size_t out_len,
                       int64_t ext[3]);

/* Per-level counters of the last solve of `level` on this context (SURVEY.md §8(d) metric:
 * macropoint solves per level; PCG / fine-pass / exchange device times; iterations; the
 * algorithmic PCG bytes of DESIGN.md §6).  Errors: MCH_EINVAL. */
int mch_get_level_stats(const mch_ctx* ctx, int level, mch_level_stats* out);

/* PCG iteration count of every problem of the last solve of `level` on this context: out[i*n_rhs + r]
 * for the i-th macropoint this context solved (the order of mch_level_macropoints restricted to
 * this rank) and right-hand side r.  cap: capacity of out in elements.  Diagnostics (load
 * balance, preconditioner studies).  Errors: MCH_EINVAL, MCH_EORDER (level not solved). */
int mch_level_iterations(const mch_ctx* ctx, int level, int32_t* out, size_t cap);

/* Parent-pool layout for the multi-GPU exchange (one process per GPU): device
 * pointer of the pool of fine parent solutions, and for macropoint index m its
 * element offset and length (-1, 0 if not stored). */
int mch_pool_info(const mch_ctx* ctx, double** pool, int64_t* pool_len);
int mch_pool_slot(const mch_ctx* ctx, int64_t macropoint, int64_t* offset, int64_t* length);
/* device pointer of the [(M+1)^d][n_rhs][n_rhs] coefficient array */
int mch_coeffs_device(const mch_ctx* ctx, double** G);

/* ---- checkpoint / resume between levels (SURVEY.md §5 auxiliaries) ----
 * The levels are solved in order and level n reads only what levels < n left behind
 * (Algorithm 1: "for n = 1..L"): the pool of stored fine local solutions
 * (the parents' phi, Eq. 11), the coefficient array G (Eq. 7) and, with a source set, the load
 * vectors.  mch_checkpoint_save writes those arrays of this rank, the number of solved levels and
 * the parameters that fix their layout (d, n, N, M, L, eta, l, interp, layout, keep_all, rank,
 * world) to `path` (host file, little-endian, raw fp64: bitwise).  mch_checkpoint_load restores
 * them into a context created with the same parameters and the same medium (the medium is NOT in
 * the file; a fingerprint of kappa / ids taken on the device is, and must match) and marks
 * those levels solved (their count in *solved_levels if not NULL), so mch_solve_level continues
 * at the next one with bitwise the same result as an uninterrupted run.  Level statistics of the restored levels are not kept.
 * Errors: MCH_EINVAL (NULL, file unreadable / not a checkpoint / parameters or medium differ),
 * MCH_ECUDA, MCH_ENOMEM. */
int mch_checkpoint_save(mch_ctx* ctx, const char* path);
int mch_checkpoint_load(mch_ctx* ctx, const char* path, int* solved_levels);

/* ---- multi-GPU plumbing; NCCL is loaded at run time (libnccl.so.2) ----
 * mch_comm_id: a new NCCL unique id (id_len >= 128 bytes) on one rank, to be broadcast to the
 * others by the caller (e.g. torch.distributed).  mch_comm_init: ncclCommInitRank(world, id, rank)
 * into *comm (collective over the ranks; call after cudaSetDevice).  mch_comm_destroy: release.
 * Errors: MCH_EINVAL, MCH_ENCCL. */
int mch_comm_id(void* id, size_t id_len);
int mch_comm_init(void** comm, int world, int rank, const void* id, size_t id_len);
int mch_comm_destroy(void* comm);

/* Sharding plan of params (rank, world) at `level`, host only (no device work, no context):
 * owned[0..*n_owned) = lexicographic indices of the macropoints of S_level this rank solves;
 * xfers[3*i .. 3*i+2] = (macropoint, src rank, dst rank) of the parent solutions of S_level that
 * move after level `level` (every rank lists all transfers; sorted by src, dst, macropoint).
 * NULL buffers return only the counts.  Errors: MCH_EINVAL (also capacity too small),
 * MCH_EDIVISIBILITY, MCH_EPLAN. */
int mch_shard_plan(const mch_params* params, int level, int64_t* owned, size_t owned_cap, int64_t* n_owned,
                   int64_t* xfers, size_t xfer_cap, int64_t* n_xfers);

const char* mch_last_error(const mch_ctx* ctx);
void mch_destroy(mch_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* MCH_H_ */
