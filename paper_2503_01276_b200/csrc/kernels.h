#pragma once
#include <cuda_runtime.h>
#include "mch_internal.h"

cudaError_t launch_level_ops(const LevelArgs& A, cudaStream_t st);
cudaError_t launch_targets(const LevelArgs& A, cudaStream_t st);
cudaError_t launch_transport(const LevelArgs& A, int threads, cudaStream_t st);
cudaError_t launch_proj_setup(const LevelArgs& A, int threads, cudaStream_t st);
cudaError_t launch_pinv(const LevelArgs& A, cudaStream_t st);  // R20 windows flagged by proj_setup
cudaError_t launch_pcg(const LevelArgs& A, int threads, cudaStream_t st);
cudaError_t launch_combine(const LevelArgs& A, int threads, cudaStream_t st);
cudaError_t launch_gram(const LevelArgs& A, int threads, cudaStream_t st);
cudaError_t launch_fingerprint(const double* kappa, const uint8_t* ids, int64_t cnt, unsigned long long* out,
                               cudaStream_t st);
cudaError_t launch_validate(const double* kappa, const uint8_t* ids, int64_t cnt, int N, int* bad,
                            cudaStream_t st);

// on-chip 2D projected PCG (pcg2d.cu).  Variants: level 1 with kappa/ids in shared memory, and
// the precomputed per-node operator for windows of <= 49 / 25 / 97 nodes per side.
#define PCG2D_V_L1 0
#define PCG2D_V_GN49 1
#define PCG2D_V_GN25 2
#define PCG2D_V_GN97 3
void pcg2d_variant(int variant, int* rpt, int* nxm, int* maxw, int* l1op, int* sstc, int* smlr);
size_t pcg2d_smem_t(int N, bool l1op, int nxm, int maxw, bool sstc, bool smlr, bool crs = false);
cudaError_t launch_node_ops2d(const LevelArgs& A, int max_nodes, cudaStream_t st);
cudaError_t launch_pcg2d(const LevelArgs& A, int variant, int threads, cudaStream_t st);
void pcg2d_phase_dump(const char* tag);  // PCG2D_TIMING builds: per-phase cycle counters

// upscaled system (macro.cu, NEXT-2): one-CTA matrix-free Jacobi-PCG on the coarse vertex grid
size_t macro_workspace_doubles(int D, int N, int64_t M);
cudaError_t launch_macro_pcg(int D, int N, int64_t M, const double* G, const double* b, double* U, double* ws,
                             double rtol, int max_iter, int* iters, double* relres, cudaStream_t st);

// on-chip 3D PCG at levels >= 2 (pcg3d.cu): windows of <= 7 / 13 / 25 level nodes per side
int pcg3d_nxm(int max_nodes_per_side);
size_t pcg3d_smem(int N, int nxm);
cudaError_t launch_node_ops3d(const LevelArgs& A, int max_nodes, cudaStream_t st);
cudaError_t launch_pcg3d(const LevelArgs& A, int nxm, cudaStream_t st);
// level 1 (windows of <= 49 fine nodes per side)
size_t pcg3d_l1_smem(int N);
// level 1 with a thread-block cluster of cs CTAs per problem (pcg3d_cl.cu)
size_t pcg3d_l1c_smem(int N);
int pcg3d_l1c_cluster(int level_problems, int sms);
cudaError_t launch_pcg3d_l1c(const LevelArgs& A, int cs, cudaStream_t st);
// levels >= 2 (windows of 13 / 25 level nodes per side) with a cluster of cs CTAs per problem
size_t pcg3dc_smem(int N, int nxm, int cs);
int pcg3dc_cluster(int nxm, int level_problems, int sms);
cudaError_t launch_pcg3dc(const LevelArgs& A, int nxm, int cs, cudaStream_t st);
// windows of <= 7 level nodes per side, N <= 2: one CTA per macropoint, one warp per rhs
size_t pcg3d_w7_smem(int N);
cudaError_t launch_pcg3d_w7(const LevelArgs& A, cudaStream_t st);
cudaError_t launch_pcg3d_l1(const LevelArgs& A, cudaStream_t st);

// validation workload (fine.cu, NEXT-3): global fine reference solve of Eq. (2), block averages
size_t fine_workspace_doubles(int D, int64_t n, int grid);
int fine_grid_size(int D);
cudaError_t launch_fine_pcg(int D, int64_t n, const double* kappa, const double* f, double* ws, unsigned* bar,
                            int grid, double rtol, int max_iter, int* iters, double* relres, cudaStream_t st);
cudaError_t launch_fine_block_avg(int D, const double* u, const uint8_t* ids, const int* kbox, int64_t P, int64_t n,
                                  int N, double* out, cudaStream_t st);
// 3D transport split (levels >= 2): Y = A_1 I_p and g = g0 - C_1 I_p on the fine window
cudaError_t launch_tapply3d(const LevelArgs& A, cudaStream_t st);
// dynamic shared memory of k_pcg / k_proj_setup_band at these arguments
size_t pcg_smem(const LevelArgs& A);
size_t proj_setup_band_smem(const LevelArgs& A);
// dynamic shared memory of k_pcg / k_proj_setup_band at these arguments
size_t pcg_smem(const LevelArgs& A);
size_t proj_setup_band_smem(const LevelArgs& A);
// two-level preconditioner setup (generic k_pcg, level 1)
cudaError_t launch_coarse_setup(const LevelArgs& A, cudaStream_t st);

// fused 3D fine-window passes at levels >= 2 (fine3d.cu): transport + A_1 I_p + C_1 I_p +
// restriction in one kernel; combine on K_p (and the whole window for stored parents)
size_t fine3d_transport_smem(int N);
cudaError_t launch_fine3d_transport(const LevelArgs& A, cudaStream_t st);
cudaError_t launch_fine3d_combine(const LevelArgs& A, int max_fine_nodes, cudaStream_t st);
// Eq. (7) of all rhs in one pass over the K_p cells (fused 3D path, no source term; n_rhs 4 or 8)
cudaError_t launch_gram3_kp(const LevelArgs& A, cudaStream_t st);
