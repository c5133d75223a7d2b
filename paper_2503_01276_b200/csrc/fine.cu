// Validation workload (NEXT-3): the global fine-grid reference solve of Eq. (2) and the fine
// block averages of the error metric e_2.
//
// Eq. (2) on the n^d fine Q1 grid of the whole domain, u = 0 on the boundary
// (Eq. 1): matrix-free Jacobi-PCG in fp64 over the interior nodes, one persistent cooperative
// kernel (every CTA resident; a grid barrier between the two phases of an iteration).  Operator
// per interior node from the kappa of its 2^d cells (the Q1 element rows, as in the local
// solvers); load F_a = sum_{e ni a} f_e h^d / 2^d.  p is double-buffered so the p update of
// iteration k+1 is fused into its stencil pass (neighbours read z and the old p, which no CTA
// writes in that phase): two grid barriers per iteration.  Dot products: per-CTA fixed-order
// partial sums, then every CTA sums the partials in CTA order, so all CTAs take identical
// decisions and results are bitwise reproducible for a given grid.
#include <cuda_runtime.h>

#include <cstdint>

#include "device_common.cuh"
#include "kernels.h"

namespace {

constexpr int FT = 256;  // threads per CTA

struct FineArgs {
  int D, n;
  double h;
  const double* kappa;  // n^D cells, x fastest
  const double* f;      // n^D cells
  double *x, *r, *z, *pa, *pb, *q, *dinv;  // (n+1)^D nodes
  double* part;         // [grid][4]
  unsigned* bar;        // [2]: arrival count, generation
  double rtol;
  int max_iter;
  int* iters;
  double* relres;
};

__device__ __forceinline__ void grid_sync(unsigned* bar) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = bar + 1;
    const unsigned g = *gen;
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g) __nanosleep(64);
    }
    __threadfence();
  }
  __syncthreads();
}

// fixed-order CTA sum of NV values (all threads get the totals)
template <int NV>
__device__ __forceinline__ void cta_sum(double (&v)[NV], double* sh) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; i++)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_down_sync(FULLMASK, v[i], o);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < NV; i++) sh[w * NV + i] = v[i];
  __syncthreads();
#pragma unroll
  for (int i = 0; i < NV; i++) {
    double s = 0.0;
    for (int k = 0; k < FT / 32; k++) s += sh[k * NV + i];
    v[i] = s;
  }
}

// grid total of partial slot i (fixed order over CTAs; __ldcg: written by other SMs)
__device__ __forceinline__ double grid_total(const double* part, int i, double* sh) {
  double s = 0.0;
  if (threadIdx.x < 32) {
    for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) s += __ldcg(part + b * 4 + i);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(FULLMASK, s, o);
    if (threadIdx.x == 0) sh[0] = s;
  }
  __syncthreads();
  s = sh[0];
  __syncthreads();
  return s;
}

template <int D>
struct FGeo {
  int n, nv;
  int64_t nn;
  __device__ void xyz(int64_t k, int* c) const {
    for (int i = 0; i < D; i++) {
      c[i] = (int)(k % nv);
      k /= nv;
    }
  }
  __device__ bool interior(const int* c) const {
    for (int i = 0; i < D; i++)
      if (c[i] == 0 || c[i] == n) return false;
    return true;
  }
};

// (A v)_k at an interior node with v given on the fly by val(node index)
template <int D, typename V>
__device__ __forceinline__ double apply_fine(const FineArgs& A, const FGeo<D>& g, const int* c, int64_t k, V&& val) {
  const int64_t sy = g.nv, sz = (int64_t)g.nv * g.nv;
  if (D == 2) {
    const double* kp = A.kappa + (int64_t)(c[1] - 1) * g.n + (c[0] - 1);
    const double kLL = kp[0], kLR = kp[1], kUL = kp[g.n], kUR = kp[g.n + 1];
    const double sL = kLL + kUL, sR = kLR + kUR, sD = kLL + kLR, sU = kUL + kUR;
    const double a0 = val(k - sy - 1), b0 = val(k - sy), c0 = val(k - sy + 1);
    const double a1 = val(k - 1), b1 = val(k), c1 = val(k + 1);
    const double a2 = val(k + sy - 1), b2 = val(k + sy), c2 = val(k + sy + 1);
    double acc = 4.0 * (sL + sR) * b1 - sR * c1 - sL * a1 - sU * b2 - sD * b0;
    acc -= 2.0 * (kUR * c2 + kUL * a2 + kLR * c0 + kLL * a0);
    return acc * (1.0 / 6.0);
  } else {
    double nb[3][3][3];
#pragma unroll
    for (int dz = 0; dz < 3; dz++)
#pragma unroll
      for (int dy = 0; dy < 3; dy++)
#pragma unroll
        for (int dx = 0; dx < 3; dx++) nb[dz][dy][dx] = val(k + (dz - 1) * sz + (dy - 1) * sy + (dx - 1));
    double acc = 0.0;
#pragma unroll
    for (int o = 0; o < 8; o++) {
      const int ox = o & 1, oy = (o >> 1) & 1, oz = o >> 2;
      const double kap =
          A.kappa[((int64_t)(c[2] - 1 + oz) * g.n + (c[1] - 1 + oy)) * g.n + (c[0] - 1 + ox)];
      const int a = (~o) & 7;
      auto pb = [&](int b) { return nb[oz + ((b >> 2) & 1)][oy + ((b >> 1) & 1)][ox + (b & 1)]; };
      acc += kap * (4.0 * pb(a) - pb(a ^ 3) - pb(a ^ 5) - pb(a ^ 6) - pb(a ^ 7));
    }
    return acc * A.h * (1.0 / 12.0);
  }
}

template <int D>
__global__ void __launch_bounds__(FT) k_fine_pcg(FineArgs A) {
  __shared__ double sh[FT / 32 * 4];
  FGeo<D> g;
  g.n = A.n;
  g.nv = A.n + 1;
  g.nn = 1;
  for (int i = 0; i < D; i++) g.nn *= g.nv;
  const int64_t chunk = (g.nn + gridDim.x - 1) / gridDim.x;
  const int64_t k0 = (int64_t)blockIdx.x * chunk, k1 = min(g.nn, k0 + chunk);
  const double hd = (D == 2) ? A.h * A.h * 0.25 : A.h * A.h * A.h * 0.125;
  // init: x = 0, r = F, D^-1, z = D^-1 r; partials rz, |F|^2
  {
    double v[2] = {0.0, 0.0};
    for (int64_t k = k0 + threadIdx.x; k < k1; k += FT) {
      int c[3];
      g.xyz(k, c);
      double F = 0.0, di = 0.0;
      if (g.interior(c)) {
        double ks = 0.0;
        for (int o = 0; o < (1 << D); o++) {
          int64_t e = 0;
          for (int i = D - 1; i >= 0; i--) e = e * g.n + (c[i] - 1 + ((o >> i) & 1));
          F += A.f[e];
          ks += A.kappa[e];
        }
        F *= hd;
        di = 1.0 / ((D == 2) ? ks * (2.0 / 3.0) : ks * A.h * (1.0 / 3.0));
      }
      A.x[k] = 0.0;
      A.r[k] = F;
      A.dinv[k] = di;
      const double zz = di * F;
      A.z[k] = zz;
      A.pa[k] = 0.0;
      A.pb[k] = 0.0;
      A.q[k] = 0.0;
      v[0] += F * zz;
      v[1] += F * F;
    }
    cta_sum<2>(v, sh);
    if (threadIdx.x == 0) {
      A.part[blockIdx.x * 4 + 0] = v[0];
      A.part[blockIdx.x * 4 + 1] = v[1];
    }
  }
  grid_sync(A.bar);
  double rz = grid_total(A.part, 0, sh);
  const double bnorm = sqrt(grid_total(A.part, 1, sh));
  double rn = bnorm, beta = 0.0;
  int it = 0;
  double* pold = A.pa;
  double* pnew = A.pb;
  grid_sync(A.bar);  // everyone has read the partials before they are overwritten
  for (; bnorm > 0.0 && it < A.max_iter && rn > A.rtol * bnorm; it++) {
    // phase 1: p_new = z + beta p_old (fused), q = A p_new, pq
    double v[1] = {0.0};
    for (int64_t k = k0 + threadIdx.x; k < k1; k += FT) {
      int c[3];
      g.xyz(k, c);
      if (!g.interior(c)) continue;
      auto pv = [&](int64_t m) { return __ldcg(A.z + m) + beta * __ldcg(pold + m); };
      const double qk = apply_fine<D>(A, g, c, k, pv);
      const double pk = pv(k);
      pnew[k] = pk;
      A.q[k] = qk;
      v[0] += pk * qk;
    }
    cta_sum<1>(v, sh);
    if (threadIdx.x == 0) A.part[blockIdx.x * 4 + 2] = v[0];
    grid_sync(A.bar);
    const double alpha = rz / grid_total(A.part, 2, sh);
    // phase 2: x += alpha p, r -= alpha q, z = D^-1 r, rz, rr (own nodes only)
    double w[2] = {0.0, 0.0};
    for (int64_t k = k0 + threadIdx.x; k < k1; k += FT) {
      const double di = A.dinv[k];
      if (di == 0.0) continue;  // boundary node
      A.x[k] += alpha * pnew[k];
      const double rk = A.r[k] - alpha * A.q[k];
      A.r[k] = rk;
      const double zz = di * rk;
      A.z[k] = zz;
      w[0] += rk * zz;
      w[1] += rk * rk;
    }
    cta_sum<2>(w, sh);
    if (threadIdx.x == 0) {
      A.part[blockIdx.x * 4 + 0] = w[0];
      A.part[blockIdx.x * 4 + 1] = w[1];
    }
    grid_sync(A.bar);
    const double rz_new = grid_total(A.part, 0, sh);
    rn = sqrt(grid_total(A.part, 1, sh));
    beta = rz_new / rz;
    rz = rz_new;
    double* t = pold;
    pold = pnew;
    pnew = t;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *A.iters = it;
    *A.relres = (bnorm > 0.0) ? rn / bnorm : 0.0;
  }
}

// fine block averages: one CTA per macropoint, out[p][i] = mean over the cells of continuum i in
// K_p of the cell mean of u (equal cell volumes); NaN if K_p holds no cell of continuum i
template <int D>
__global__ void k_fine_block_avg(const double* u, const uint8_t* ids, const int* kbox, int n, int N, double* out) {
  const int p = blockIdx.x;
  const int* b = kbox + p * 6;
  int ext[3] = {1, 1, 1};
  for (int i = 0; i < D; i++) ext[i] = b[3 + i] - b[i];
  const int64_t cnt = (int64_t)ext[0] * ext[1] * ext[2];
  const int64_t nv = n + 1;
  __shared__ double scratch[32 * 16];
  __shared__ double tot[16];
  double v[16];
  for (int i = 0; i < 16; i++) v[i] = 0.0;
  for (int64_t idx = threadIdx.x; idx < cnt; idx += blockDim.x) {
    int e[3] = {b[0] + (int)(idx % ext[0]), b[1] + (int)((idx / ext[0]) % ext[1]), 0};
    if (D == 3) e[2] = b[2] + (int)(idx / ((int64_t)ext[0] * ext[1]));
    int64_t ce = 0, nd = 0;
    for (int i = D - 1; i >= 0; i--) {
      ce = ce * n + e[i];
      nd = nd * nv + e[i];
    }
    double s = 0.0;
    for (int a = 0; a < (1 << D); a++) {
      int64_t m = 0;
      for (int i = D - 1; i >= 0; i--) m = m * nv + e[i] + ((a >> i) & 1);
      s += u[m];
    }
    s *= 1.0 / (double)(1 << D);
    const int id = ids[ce];
    for (int j = 0; j < N; j++) {
      v[j] += (id == j) ? s : 0.0;
      v[8 + j] += (id == j) ? 1.0 : 0.0;
    }
    (void)nd;
  }
  block_sum<16>(v, scratch, tot);
  if (threadIdx.x < N) {
    const double c = tot[8 + threadIdx.x];
    out[(int64_t)p * N + threadIdx.x] = (c > 0.0) ? tot[threadIdx.x] / c : __longlong_as_double(0x7ff8000000000000LL);
  }
}

}  // namespace

size_t fine_workspace_doubles(int D, int64_t n, int grid) {
  int64_t nn = 1;
  for (int i = 0; i < D; i++) nn *= n + 1;
  return (size_t)(7 * nn + 4 * (int64_t)grid);
}

int fine_grid_size(int D) {
  int dev = 0, sms = 0, nb = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (D == 2) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_fine_pcg<2>, FT, 0);
  else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_fine_pcg<3>, FT, 0);
  return sms * (nb > 0 ? nb : 1);
}

cudaError_t launch_fine_pcg(int D, int64_t n, const double* kappa, const double* f, double* ws, unsigned* bar,
                            int grid, double rtol, int max_iter, int* iters, double* relres, cudaStream_t st) {
  FineArgs A;
  A.D = D;
  A.n = (int)n;
  A.h = 1.0 / (double)n;
  A.kappa = kappa;
  A.f = f;
  int64_t nn = 1;
  for (int i = 0; i < D; i++) nn *= n + 1;
  A.x = ws; A.r = ws + nn; A.z = ws + 2 * nn; A.pa = ws + 3 * nn; A.pb = ws + 4 * nn; A.q = ws + 5 * nn;
  A.dinv = ws + 6 * nn;
  A.part = ws + 7 * nn;
  A.bar = bar;
  A.rtol = rtol;
  A.max_iter = max_iter;
  A.iters = iters;
  A.relres = relres;
  cudaError_t e = cudaMemsetAsync(bar, 0, 2 * sizeof(unsigned), st);
  if (e != cudaSuccess) return e;
  void* args[] = {&A};
  if (D == 2) return cudaLaunchCooperativeKernel((const void*)k_fine_pcg<2>, grid, FT, args, 0, st);
  return cudaLaunchCooperativeKernel((const void*)k_fine_pcg<3>, grid, FT, args, 0, st);
}

cudaError_t launch_fine_block_avg(int D, const double* u, const uint8_t* ids, const int* kbox, int64_t P, int64_t n,
                                  int N, double* out, cudaStream_t st) {
  if (D == 2) k_fine_block_avg<2><<<(unsigned)P, 256, 0, st>>>(u, ids, kbox, (int)n, N, out);
  else k_fine_block_avg<3><<<(unsigned)P, 256, 0, st>>>(u, ids, kbox, (int)n, N, out);
  return cudaGetLastError();
}
