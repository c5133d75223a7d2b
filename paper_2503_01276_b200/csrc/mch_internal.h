// Internal structures shared by the host planner, the C ABI and the kernels.
#pragma once
#include <cstdint>
#include <vector_types.h>

#define MCH_MAXPAR 8  // 2^d parents at most (d-linear interpolation, Eq. 11)
constexpr int kAzCap = 4;  // (A z_a) list entries per window node (two-level preconditioner, 2D)

// One macropoint solved at its level (device-visible POD).
struct ProbDesc {
  int k[3];          // macro vertex multi-index (x_p = H k)
  int lo[3];         // window R_p^+ lower fine-cell index (global)
  int ncf[3];        // window fine cells per dimension
  int nc[3];         // window level-n cells per dimension (ncf / s)
  int glo[3];        // global level-n cell index of the window origin (lo / s)
  int kp_lo[3];      // K_p fine-cell range [kp_lo, kp_hi) (global)
  int kp_hi[3];
  int64_t lin;       // lexicographic macropoint index
  int64_t node_off;  // offset of this macropoint's level-n node block (dinv)
  int64_t vec_off;   // offset of rhs 0 of the level-n vectors; rhs r at vec_off + r*nodes
  int64_t fine_off;  // offset of rhs 0 in the fine workspace (levels >= 2)
  int64_t pool_off;  // offset of rhs 0 in the parent pool, -1 if not stored
  int npar;
  int par_k[MCH_MAXPAR][3];
  int par_lo[MCH_MAXPAR][3];
  int par_ncf[MCH_MAXPAR][3];
  int64_t par_pool[MCH_MAXPAR];
  double par_w[MCH_MAXPAR];
};

// Per-level constants passed by value to every kernel.
struct LevelArgs {
  int D, N, n_rhs, l, w;   // w = 2l+1 subcells per dimension
  int nsub, ncon;          // w^D subcells, ncon = nsub*N constraint rows
  int level, s;            // s = eta^(level-1)
  int n, c;                // fine cells per dim, fine cells per H
  int coff;                // subcell of fine cell f: (f + coff) / c - k + l (c/2 vertex layout, 0 block)
  int gn;                  // global level-n cells per dim (n/s)
  double h;
  float inv_c;             // 1/c
  const double* kappa;     // fine, n^D, x fastest
  const uint8_t* ids;
  const double* W;         // level >= 2: per global level-n cell, D*3^(D-1) operator weights
  const double* Mc;        // level >= 2: per global level-n cell, N*2^D constraint weights
  const ProbDesc* probs;
  int nprob_mp;            // macropoints in this batch
  int nprob_level;         // macropoints of S_level over all ranks (launch heuristics)
  // per-macropoint arrays (indexed by batch-local macropoint index)
  double* g0;              // [mp][ncon][n_rhs] original targets (Eqs. 3/4)
  double* g;               // [mp][ncon][n_rhs] targets of the solved problem (Eq. 12/13)
  double* meas;            // [mp][ncon] int_{R_q} psi_j
  double* cm;              // [mp][D][N] centring constants c_mj
  int* flags;              // [mp] bit0: continuum absent from K_p
  double* dinv;            // level-n node blocks
  double* NWt;             // [node blocks][N][nodes] interior-node constraint weights
  double* Sinv;            // [mp][ncon][ncon]
  double* pinv_ds;         // [mp][ncon] row scales of S~ (reading R20 windows)
  // per-problem vectors (problem = mp*n_rhs + r)
  double* X; double* R; double* P; double* Q; double* B;
  double* FI; double* FY;  // fine workspace (levels >= 2): I_p / phi and A1 I_p
  double* FK;              // fused 3D path (fine3d.cu): phi_p on the K_p node box, [mp][n_rhs][nkp_max]
  int nkp_max;             // K_p box nodes per (macropoint, rhs) slot of FK
  double* pool;            // parent pool
  double* G;               // [(M+1)^D][n_rhs][n_rhs]
  int band;                // 0: dense S^-1 per macropoint; > 0: banded Cholesky factor of the
                           //  equilibrated S (half-bandwidth band, 2D large l), Sinv[mp][nc][band+1]
  // two-level preconditioner (generic k_pcg, level 1, dense projector): M^-1 = D^-1 + Z E^-1 Z^T with
  // Z = indicators of the 8- (26-) connected components of nodes touching a high-kappa cell
  int coarse;              // bit 0: build and use the coarse space; bit 1: second labelling pass (k_coarse_setup)
  int ncmax;               // components per window capacity (more: the window runs without)
  int* cmap;               // [nodes] component of each level-1 node, -1 none (node_off based)
  int* ncomp;              // [mp]
  int* cbox;               // [mp][ncmax][6] node bounding box per component (lo, hi inclusive)
  double* Einv;            // [mp][ncmax] 1 / (z_a^T A z_a)
  double* CZ;              // [mp][ncon][ncmax] C z_a
  int* cptr;               // [mp][ncmax+1] start of each component's node list in clist
  int* clist;              // [nodes] node indices of each component, in node order (node_off based)
  int* azp;                // [mp][ncmax+1] start of each component's (A z_a) list (2D on-chip kernels)
  int* azi;                // [kAzCap * nodes] node of each entry, packed x | y << 16
  double* azw;             // [kAzCap * nodes] (A z_a) at that node
  int phys;                // 1: parents at physical coordinates (NEXT-4), 0: local coordinates (R9)
  int tphase;              // k_transport: 0 all phases; 1 only I_p; 2 only the restriction (3D split path)
  int psplit;              // k_proj_setup: 0 whole; 1 only S = C D^-1 C^T (into Sinv); 2 the rest from it
  const double* f;         // NEXT-2: cellwise source, n^D, x fastest (NULL: no load vectors)
  double* bload;           // NEXT-2: [P][N] load vectors b_j = int_{K_p} f phi_j (Eq. 7)
  int* iters; double* relres;  // [problem]
  double* diag;            // [problem][4]: final rz, reference rz, floor, breakdown flag
  double rtol; int max_iter;
  // on-chip 2D PCG (pcg2d.cu)
  const short4* segs;      // [mp][maxseg] row chunks: (first node row, rows, subcell row, subcell row
                           //  of the lower elements of the first row if it is an interface row, else -1)
  const int* nseg;         // [mp]
  int maxseg;
  int tm_cols;             // TMEM columns allocated per CTA
  double* STC;             // levels >= 2: per window node 9 stencil coefficients, SoA [9][nodes]
  double* dbg;             // debug: per-iteration scalars of problem dbg_prob (NULL: off)
  int dbg_prob, dbg_cap;
  int need_nwt;            // k_proj_setup fills NWt (generic k_pcg only)
  int stc_pad;             // 3D levels >= 2 on k_pcg3d / k_pcg3dc: STC / MLR per window at a fixed node
                           // stride NXM^3 (window i at i * 27 * NXM^3), so the solvers address them
                           // with compile-time offsets; 0: node_off layout with stride nn
  double* MLR;             // levels >= 2: per node constraint side sums, SoA [4N][nodes]:
                           //  [L|R][j] over lower+upper elements, then [L|R][j] lower elements only
};
