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
