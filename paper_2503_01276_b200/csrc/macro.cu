// Upscaled multicontinuum system (NEXT-2): Eq. (6) through the bilinear form of PAPER.md:187-199,
// on the block-centred layout (K_p = coarse block p, "U_i, V_j and their gradients are taken at
// ... the midpoint of the coarse block").  Unknowns: U_i continuous Q1 on the coarse vertex grid
// {0..M}^D, homogeneous Dirichlet on the boundary (Eq. 1).
//
//   a(U, V) = sum_p t_p(V)^T G_p t_p(U),  t_p(U) = (U_0..U_{N-1}, d_0U_0..d_{D-1}U_0, .., d_{D-1}U_{N-1})
//   l(V)    = sum_p sum_j V_j(x_p) b_j(p)                       (reading R23)
//
// t_p at the block centre from the corner values: U_i(x_p) = mean of the 2^D corners,
// d_m U_i(x_p) = sum_a sgn_m(a) U_i(a) / (H 2^(D-1)).
//
// One CTA, matrix-free Jacobi-PCG (the system has (M+1)^D N unknowns: coarse and small, SURVEY
// §8(f) item 2).  K p is applied in two phases so every sum has a fixed order (bitwise
// deterministic): (1) per block, y_p = G_p t_p(p) into a block buffer; (2) per node and
// continuum, the E^T y_p contributions of the adjacent blocks in corner order.
#include <cuda_runtime.h>

#include <cstdint>

#include "device_common.cuh"
#include "kernels.h"

namespace {

constexpr int MT = 1024;  // threads of the one CTA

struct MacroArgs {
  int N, M;
  double H;
  const double* G;  // [P][nr][nr]
  const double* b;  // [P][N]
  double* U;        // out [N][(M+1)^D]
  double *x, *r, *z, *p, *q, *dinv, *y;  // workspace: 6 x nodes*N, blocks*nr
  double rtol;
  int max_iter;
  int* iters;       // out
  double* relres;   // out: final ||r|| / ||F||
};

// fixed-order sums of NV values over the CTA (shuffle tree per warp, then warps in order)
template <int NV>
__device__ __forceinline__ void cta_sum(double (&v)[NV], double* scratch, double* out) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; i++)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_down_sync(0xffffffffu, v[i], o);
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < NV; i++) scratch[wid * NV + i] = v[i];
  __syncthreads();
  if (threadIdx.x < NV) {
    double s = 0.0;
    for (int w = 0; w < MT / 32; w++) s += scratch[w * NV + threadIdx.x];
    out[threadIdx.x] = s;
  }
  __syncthreads();
}

template <int D>
struct MGeo {
  int M, nv;
  int64_t nodes, blocks;
  __device__ void node_xyz(int64_t v, int* c) const {
    for (int i = 0; i < D; i++) { c[i] = (int)(v % nv); v /= nv; }
  }
  __device__ int64_t node_of(const int* c) const {
    int64_t v = 0;
    for (int i = D - 1; i >= 0; i--) v = v * nv + c[i];
    return v;
  }
  __device__ int64_t block_of(const int* c) const {
    int64_t v = 0;
    for (int i = D - 1; i >= 0; i--) v = v * M + c[i];
    return v;
  }
  __device__ bool interior(const int* c) const {
    for (int i = 0; i < D; i++)
      if (c[i] == 0 || c[i] == M) return false;
    return true;
  }
};

// phase 1: y_p = G_p E u_p for every block (u = src, node-major, continuum fastest)
template <int D>
__device__ void blocks_apply(const MacroArgs& A, const MGeo<D>& g, const double* src) {
  const int N = A.N, nr = N * (1 + D);
  const double gs = 1.0 / (A.H * (double)(1 << (D - 1)));
  const double vs = 1.0 / (double)(1 << D);
  for (int64_t pb = threadIdx.x; pb < g.blocks; pb += MT) {
    int kb[3] = {0, 0, 0};
    int64_t rem = pb;
    for (int i = 0; i < D; i++) { kb[i] = (int)(rem % g.M); rem /= g.M; }
    double t[16];
    for (int i = 0; i < nr; i++) t[i] = 0.0;
    for (int a = 0; a < (1 << D); a++) {
      int cc[3];
      for (int i = 0; i < D; i++) cc[i] = kb[i] + ((a >> i) & 1);
      const double* u = src + g.node_of(cc) * N;
      for (int i = 0; i < N; i++) {
        const double ui = u[i];
        t[i] += vs * ui;
        for (int m = 0; m < D; m++) t[N + i * D + m] += (((a >> m) & 1) ? gs : -gs) * ui;
      }
    }
    const double* Gp = A.G + pb * nr * nr;
    double* yp = A.y + pb * nr;
    for (int rr = 0; rr < nr; rr++) {
      double s = 0.0;
      for (int cc = 0; cc < nr; cc++) s += Gp[rr * nr + cc] * t[cc];
      yp[rr] = s;
    }
  }
}

// phase 2 contribution of the adjacent blocks to node (c, continuum i): sum_a E^T y  (or F from b)
template <int D>
__device__ double gather_node(const MacroArgs& A, const MGeo<D>& g, const int* c, int i, bool load) {
  const int N = A.N, nr = N * (1 + D);
  const double gs = 1.0 / (A.H * (double)(1 << (D - 1)));
  const double vs = 1.0 / (double)(1 << D);
  double s = 0.0;
  for (int a = 0; a < (1 << D); a++) {  // node c is corner a of block c - bits(a)
    int kb[3];
    bool ok = true;
    for (int m = 0; m < D; m++) {
      kb[m] = c[m] - ((a >> m) & 1);
      ok = ok && kb[m] >= 0 && kb[m] < g.M;
    }
    if (!ok) continue;
    const int64_t pb = g.block_of(kb);
    if (load) {
      s += vs * A.b[pb * N + i];
      continue;
    }
    const double* yp = A.y + pb * nr;
    double v = vs * yp[i];
    for (int m = 0; m < D; m++) v += (((a >> m) & 1) ? gs : -gs) * yp[N + i * D + m];
    s += v;
  }
  return s;
}

template <int D>
__device__ double diag_node(const MacroArgs& A, const MGeo<D>& g, const int* c, int i) {
  const int N = A.N, nr = N * (1 + D);
  const double gs = 1.0 / (A.H * (double)(1 << (D - 1)));
  const double vs = 1.0 / (double)(1 << D);
  double s = 0.0;
  for (int a = 0; a < (1 << D); a++) {
    int kb[3];
    bool ok = true;
    for (int m = 0; m < D; m++) {
      kb[m] = c[m] - ((a >> m) & 1);
      ok = ok && kb[m] >= 0 && kb[m] < g.M;
    }
    if (!ok) continue;
    const double* Gp = A.G + g.block_of(kb) * nr * nr;
    int idx[4];
    double e[4];
    idx[0] = i; e[0] = vs;
    for (int m = 0; m < D; m++) { idx[1 + m] = N + i * D + m; e[1 + m] = ((a >> m) & 1) ? gs : -gs; }
    for (int u = 0; u <= D; u++)
      for (int w = 0; w <= D; w++) s += e[u] * Gp[idx[u] * nr + idx[w]] * e[w];
  }
  return s;
}

template <int D>
__global__ void __launch_bounds__(MT, 1) k_macro_pcg(MacroArgs A) {
  __shared__ double scratch[32 * 2];
  __shared__ double tot[2];
  MGeo<D> g;
  g.M = A.M;
  g.nv = A.M + 1;
  g.nodes = 1;
  g.blocks = 1;
  for (int i = 0; i < D; i++) { g.nodes *= g.nv; g.blocks *= g.M; }
  const int N = A.N;
  const int64_t nu = g.nodes * N;
  // F, r = F (x = 0), dinv, z, p
  double acc[2] = {0.0, 0.0};
  for (int64_t u = threadIdx.x; u < nu; u += MT) {
    int c[3];
    g.node_xyz(u / N, c);
    const int i = (int)(u % N);
    double f = 0.0, di = 1.0;
    if (g.interior(c)) {
      f = gather_node<D>(A, g, c, i, true);
      const double dg = diag_node<D>(A, g, c, i);
      di = dg > 0.0 ? 1.0 / dg : 1.0;
    }
    A.x[u] = 0.0;
    A.r[u] = f;
    A.dinv[u] = di;
    const double zz = di * f;
    A.z[u] = zz;
    A.p[u] = zz;
    acc[0] += f * zz;
    acc[1] += f * f;
  }
  cta_sum<2>(acc, scratch, tot);
  double rz = tot[0];
  const double bnorm = sqrt(tot[1]);
  double rn = bnorm;
  int it = 0;
  if (bnorm > 0.0) {
    for (; it < A.max_iter && rn > A.rtol * bnorm; it++) {
      blocks_apply<D>(A, g, A.p);
      __syncthreads();
      double pq[1] = {0.0};
      for (int64_t u = threadIdx.x; u < nu; u += MT) {
        int c[3];
        g.node_xyz(u / N, c);
        const double qq = g.interior(c) ? gather_node<D>(A, g, c, (int)(u % N), false) : 0.0;
        A.q[u] = qq;
        pq[0] += A.p[u] * qq;
      }
      cta_sum<1>(pq, scratch, tot);
      const double alpha = rz / tot[0];
      double a2[2] = {0.0, 0.0};
      for (int64_t u = threadIdx.x; u < nu; u += MT) {
        A.x[u] += alpha * A.p[u];
        const double rr = A.r[u] - alpha * A.q[u];
        A.r[u] = rr;
        const double zz = A.dinv[u] * rr;
        A.z[u] = zz;
        a2[0] += rr * zz;
        a2[1] += rr * rr;
      }
      cta_sum<2>(a2, scratch, tot);
      const double beta = tot[0] / rz;
      rz = tot[0];
      rn = sqrt(tot[1]);
      for (int64_t u = threadIdx.x; u < nu; u += MT) A.p[u] = A.z[u] + beta * A.p[u];
      __syncthreads();
    }
  }
  for (int64_t u = threadIdx.x; u < nu; u += MT) A.U[(u % N) * g.nodes + u / N] = A.x[u];
  if (threadIdx.x == 0) {
    *A.iters = it;
    *A.relres = bnorm > 0.0 ? rn / bnorm : 0.0;
  }
}

}  // namespace

size_t macro_workspace_doubles(int D, int N, int64_t M) {
  int64_t nodes = 1, blocks = 1;
  for (int i = 0; i < D; i++) { nodes *= M + 1; blocks *= M; }
  return (size_t)(6 * nodes * N + blocks * N * (1 + D));
}

cudaError_t launch_macro_pcg(int D, int N, int64_t M, const double* G, const double* b, double* U, double* ws,
                             double rtol, int max_iter, int* iters, double* relres, cudaStream_t st) {
  MacroArgs A;
  A.N = N;
  A.M = (int)M;
  A.H = 1.0 / (double)M;
  A.G = G;
  A.b = b;
  A.U = U;
  int64_t nodes = 1;
  for (int i = 0; i < D; i++) nodes *= M + 1;
  const int64_t nu = nodes * N;
  A.x = ws; A.r = ws + nu; A.z = ws + 2 * nu; A.p = ws + 3 * nu; A.q = ws + 4 * nu; A.dinv = ws + 5 * nu;
  A.y = ws + 6 * nu;
  A.rtol = rtol;
  A.max_iter = max_iter;
  A.iters = iters;
  A.relres = relres;
  if (D == 2) k_macro_pcg<2><<<1, MT, 0, st>>>(A);
  else k_macro_pcg<3><<<1, MT, 0, st>>>(A);
  return cudaGetLastError();
}
