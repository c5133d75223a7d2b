#pragma once
#include <cuda_runtime.h>
#include "mch_internal.h"

cudaError_t launch_level_ops(const LevelArgs& A, cudaStream_t st);
cudaError_t launch_targets(const LevelArgs& A, cudaStream_t st);
cudaError_t launch_transport(const LevelArgs& A, int threads, cudaStream_t st);
cudaError_t launch_proj_setup(const LevelArgs& A, int threads, cudaStream_t st);
cudaError_t launch_pcg(const LevelArgs& A, int threads, cudaStream_t st);
cudaError_t launch_combine(const LevelArgs& A, int threads, cudaStream_t st);
cudaError_t launch_gram(const LevelArgs& A, int threads, cudaStream_t st);
cudaError_t launch_validate(const double* kappa, const uint8_t* ids, int64_t cnt, int N, int* bad,
                            cudaStream_t st);

// on-chip 2D projected PCG (pcg2d.cu)
#define PCG2D_RPT_L1 17  // rows per thread, level 1 (kappa/ids in shared memory)
#define PCG2D_RPT_GN 9   // rows per thread, levels >= 2 (precomputed per-node operator)
#define PCG2D_NXMAX_L1 97  // widest window (nodes) of the level-1 variant: 3H at 32 cells per H
#define PCG2D_NXMAX_GN 97  // and of the precomputed-operator variant
size_t pcg2d_smem(int nx, int ny, int nc, int nwarps, bool l1op);
cudaError_t launch_node_ops2d(const LevelArgs& A, int max_nodes, cudaStream_t st);
cudaError_t launch_pcg2d(const LevelArgs& A, bool l1op, int threads, size_t smem, cudaStream_t st);
