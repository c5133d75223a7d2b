// Device helpers shared by the hot-path kernels: window geometry, the element
// operator (exact Galerkin Q1 stiffness in "directional weight" form), the
// element constraint weights, and deterministic block reductions.
//
// Element operator (weak form Eq. 2; level spaces PAPER.md:369):
// for a (coarse) cell E of side Hc with fine cellwise kappa, coarse Q1 basis
// N_a = prod_i l_{a_i}(x_i),
//   (K_E p)_a = sum_k s(a_k) sum_{b_o} W^k[t(a_o,b_o)] (p[b_k=1,b_o] - p[b_k=0,b_o]),
//   W^k[t] = Hc^-2 int_E kappa prod_{o != k} l_{a_o} l_{b_o}   (t = type of the pair per
//   other dimension: 00 -> 0, 01/10 -> 1, 11 -> 2),  s(0) = -1, s(1) = +1.
// At level 1 (E = fine cell) W^k[t] = kappa h^(D-2) prod_o m1[t_o], m1 = (1/3, 1/6, 1/3).
// Element constraint weights (Eq. 3/4 constraint rows): m_{E,j,a} = int_E psi_j N_a;
// at level 1 m = [id_E = j] h^D / 2^D.
#pragma once
#include <cstdint>
#include "mch_internal.h"

#define FULLMASK 0xffffffffu

template <int D> struct DimC {
  static constexpr int NC = 1 << D;              // element corners
  static constexpr int NT = (D == 2) ? 3 : 9;    // pair types over the other D-1 dims
  static constexpr int NW = D * NT;              // operator weights per element
  static constexpr int NB = (D == 2) ? 9 : 27;   // 3^D node neighbourhood
};

template <int D> struct Geo {
  int nc[3];      // cells per dim (element grid)
  int nn[3];      // nodes per dim
  int nnodes;
  int s;          // fine cells per element edge
  bool fineop;    // element data from fine kappa/ids (level-1 form)
  float inv0, inv01;  // 1/nn[0], 1/(nn[0] nn[1]) for division-free index decoding
};

// floor(a / b) for 0 <= a < 2^22, 1 <= b < 2^11, given inv = 1/b in float (exact: the +0.5 keeps
// the product away from integers by more than the float rounding error)
__device__ __forceinline__ int fdiv(int a, float inv) { return (int)(((float)a + 0.5f) * inv); }

template <int D>
__device__ __forceinline__ Geo<D> level_geo(const LevelArgs& A, const ProbDesc& P) {
  Geo<D> g;
  g.nnodes = 1;
  for (int i = 0; i < 3; i++) {
    g.nc[i] = (i < D) ? P.nc[i] : 0;
    g.nn[i] = (i < D) ? P.nc[i] + 1 : 1;
    g.nnodes *= g.nn[i];
  }
  g.s = A.s;
  g.fineop = (A.level == 1);
  g.inv0 = 1.0f / (float)g.nn[0];
  g.inv01 = 1.0f / (float)(g.nn[0] * g.nn[1]);
  return g;
}

template <int D>
__device__ __forceinline__ Geo<D> fine_geo(const ProbDesc& P) {
  Geo<D> g;
  g.nnodes = 1;
  for (int i = 0; i < 3; i++) {
    g.nc[i] = (i < D) ? P.ncf[i] : 0;
    g.nn[i] = (i < D) ? P.ncf[i] + 1 : 1;
    g.nnodes *= g.nn[i];
  }
  g.s = 1;
  g.fineop = true;
  g.inv0 = 1.0f / (float)g.nn[0];
  g.inv01 = 1.0f / (float)(g.nn[0] * g.nn[1]);
  return g;
}

template <int D>
__device__ __forceinline__ void node_xyz(const Geo<D>& g, int k, int* x) {
  if (D == 2) {
    x[1] = fdiv(k, g.inv0);
    x[0] = k - x[1] * g.nn[0];
    x[2] = 0;
  } else {
    x[2] = fdiv(k, g.inv01);
    const int t = k - x[2] * g.nn[0] * g.nn[1];
    x[1] = fdiv(t, g.inv0);
    x[0] = t - x[1] * g.nn[0];
  }
}

template <int D>
__device__ __forceinline__ int node_id(const Geo<D>& g, const int* x) {
  return (D == 2) ? x[0] + g.nn[0] * x[1] : x[0] + g.nn[0] * (x[1] + g.nn[1] * x[2]);
}

template <int D>
__device__ __forceinline__ int64_t fine_cell_index(const LevelArgs& A, const ProbDesc& P, const Geo<D>& g,
                                                   const int* e, const int* sub) {
  // fine cell of element e (+ sub-offset inside a coarse element)
  int64_t f = 0;
#pragma unroll
  for (int i = D - 1; i >= 0; i--) f = f * A.n + (P.lo[i] + e[i] * g.s + (sub ? sub[i] : 0));
  return f;
}

template <int D>
__device__ __forceinline__ int64_t level_cell_index(const LevelArgs& A, const ProbDesc& P, const int* e) {
  int64_t f = 0;
#pragma unroll
  for (int i = D - 1; i >= 0; i--) f = f * A.gn + (P.glo[i] + e[i]);
  return f;
}

// subcell index q of element e (dual block of vertex v, slot = v - k + l)
template <int D>
__device__ __forceinline__ int elem_subcell(const LevelArgs& A, const ProbDesc& P, const Geo<D>& g, const int* e) {
  int q = 0;
#pragma unroll
  for (int i = D - 1; i >= 0; i--) {
    int f = P.lo[i] + e[i] * g.s;
    int slot = fdiv(f + A.coff, A.inv_c) - P.k[i] + A.l;
    q = q * A.w + slot;
  }
  return q;
}

template <int D>
__device__ __forceinline__ void elem_W(const LevelArgs& A, const ProbDesc& P, const Geo<D>& g, const int* e,
                                       double* W) {
  if (g.fineop) {
    const double kap = A.kappa[fine_cell_index<D>(A, P, g, e, nullptr)];
    const double m1[3] = {1.0 / 3.0, 1.0 / 6.0, 1.0 / 3.0};
    if (D == 2) {
#pragma unroll
      for (int k = 0; k < 2; k++)
#pragma unroll
        for (int t = 0; t < 3; t++) W[k * 3 + t] = kap * m1[t];
    } else {
      const double kh = kap * A.h;
#pragma unroll
      for (int k = 0; k < 3; k++)
#pragma unroll
        for (int t2 = 0; t2 < 3; t2++)
#pragma unroll
          for (int t1 = 0; t1 < 3; t1++) W[k * 9 + t1 + 3 * t2] = kh * m1[t1] * m1[t2];
    }
  } else {
    const double* src = A.W + level_cell_index<D>(A, P, e) * DimC<D>::NW;
#pragma unroll
    for (int i = 0; i < DimC<D>::NW; i++) W[i] = src[i];
  }
}

// m_{E,j,a}
template <int D>
__device__ __forceinline__ double elem_m(const LevelArgs& A, const ProbDesc& P, const Geo<D>& g, const int* e,
                                         int j, int a) {
  if (g.fineop) {
    const int id = A.ids[fine_cell_index<D>(A, P, g, e, nullptr)];
    return (id == j) ? ((D == 2) ? 0.25 * A.h * A.h : 0.125 * A.h * A.h * A.h) : 0.0;
  }
  return A.Mc[level_cell_index<D>(A, P, e) * (A.N << D) + j * (1 << D) + a];
}

// pair type over the other dimensions of direction k
template <int D>
__device__ __forceinline__ int pair_type(int k, int a, int b) {
  int t = 0, mul = 1;
#pragma unroll
  for (int i = 0; i < D; i++) {
    if (i == k) continue;
    t += mul * (((a >> i) & 1) + ((b >> i) & 1));
    mul *= 3;
  }
  return t;
}

// (K_E c)_a for one corner a
template <int D>
__device__ __forceinline__ double elem_row(const double* W, const double* c, int a) {
  double y = 0.0;
#pragma unroll
  for (int k = 0; k < D; k++) {
    double acc = 0.0;
#pragma unroll
    for (int b = 0; b < (1 << D); b++) {
      if ((b >> k) & 1) continue;               // b has b_k = 0; partner b | (1<<k)
      const int t = pair_type<D>(k, a, b);
      acc += W[k * DimC<D>::NT + t] * (c[b | (1 << k)] - c[b]);
    }
    y += ((a >> k) & 1) ? acc : -acc;
  }
  return y;
}

// (K_E)_aa
template <int D>
__device__ __forceinline__ double elem_diag(const double* W, int a) {
  double y = 0.0;
#pragma unroll
  for (int k = 0; k < D; k++) y += W[k * DimC<D>::NT + pair_type<D>(k, a, a)];
  return y;
}

// (A v)_k by gathering the 2^D elements around node k (natural BC: elements outside skipped),
// from the node's 3^D neighbourhood.  Level 1 uses the Q1 element rows written out
// (2D: kappa/6 (4 v_a - v_{a^1} - v_{a^2} - 2 v_{a^3}); 3D: kappa h/12 (4 v_a - the 4 corners
// differing in >= 2 coordinates)); levels >= 2 the exact-Galerkin weights W.
template <int D>
__device__ __forceinline__ double apply_xyz(const LevelArgs& A, const ProbDesc& P, const Geo<D>& g,
                                            const double* __restrict__ v, const int* xx, int k) {
  constexpr int NB = DimC<D>::NB;
  const int sy = g.nn[0], sz = g.nn[0] * g.nn[1];
  double nb[NB];
#pragma unroll
  for (int c = 0; c < NB; c++) {
    const int dx = c % 3 - 1, dy = (c / 3) % 3 - 1, dz = (D == 3) ? c / 9 - 1 : 0;
    const bool ok = (xx[0] + dx >= 0) && (xx[0] + dx < g.nn[0]) && (xx[1] + dy >= 0) && (xx[1] + dy < g.nn[1]) &&
                    (D == 2 || ((xx[2] + dz >= 0) && (xx[2] + dz < g.nn[2])));
    nb[c] = ok ? v[k + dx + dy * sy + dz * sz] : 0.0;
  }
  double out = 0.0;
#pragma unroll
  for (int o = 0; o < (1 << D); o++) {
    int e[3] = {0, 0, 0};
    bool ok = true;
#pragma unroll
    for (int i = 0; i < D; i++) {
      e[i] = xx[i] - 1 + ((o >> i) & 1);
      ok = ok && (e[i] >= 0) && (e[i] < g.nc[i]);
    }
    if (!ok) continue;
    const int a = (~o) & ((1 << D) - 1);
    auto nbv = [&](int b) {
      const int dx = (b & 1) - (a & 1), dy = ((b >> 1) & 1) - ((a >> 1) & 1);
      const int dz = (D == 3) ? ((b >> 2) & 1) - ((a >> 2) & 1) : 0;
      return nb[(dx + 1) + 3 * (dy + 1) + (D == 3 ? 9 * (dz + 1) : 0)];
    };
    if (g.fineop) {
      const double kap = A.kappa[fine_cell_index<D>(A, P, g, e, nullptr)];
      if (D == 2)
        out += kap * (1.0 / 6.0) * (4.0 * nbv(a) - nbv(a ^ 1) - nbv(a ^ 2) - 2.0 * nbv(a ^ 3));
      else
        out += kap * A.h * (1.0 / 12.0) * (4.0 * nbv(a) - nbv(a ^ 3) - nbv(a ^ 5) - nbv(a ^ 6) - nbv(a ^ 7));
    } else {
      double W[DimC<D>::NW];
      elem_W<D>(A, P, g, e, W);
      double c[1 << D];
#pragma unroll
      for (int b = 0; b < (1 << D); b++) c[b] = nbv(b);
      out += elem_row<D>(W, c, a);
    }
  }
  return out;
}

template <int D>
__device__ __forceinline__ double apply_node(const LevelArgs& A, const ProbDesc& P, const Geo<D>& g,
                                             const double* v, int k) {
  int x[3];
  node_xyz<D>(g, k, x);
  return apply_xyz<D>(A, P, g, v, x, k);
}

template <int D>
__device__ __forceinline__ double diag_node(const LevelArgs& A, const ProbDesc& P, const Geo<D>& g, int k) {
  int x[3];
  node_xyz<D>(g, k, x);
  double y = 0.0;
#pragma unroll
  for (int ep = 0; ep < (1 << D); ep++) {
    int e[3] = {0, 0, 0};
    bool ok = true;
#pragma unroll
    for (int i = 0; i < D; i++) {
      e[i] = x[i] - 1 + ((ep >> i) & 1);
      ok = ok && (e[i] >= 0) && (e[i] < g.nc[i]);
    }
    if (!ok) continue;
    double W[DimC<D>::NW];
    elem_W<D>(A, P, g, e, W);
    y += elem_diag<D>(W, (~ep) & ((1 << D) - 1));
  }
  return y;
}

// (C^T yhat)_k = sum_{E∋k} sum_j m_{E,j,a} yhat[q(E)*N + j]
template <int D>
__device__ __forceinline__ double ct_node(const LevelArgs& A, const ProbDesc& P, const Geo<D>& g,
                                          const double* yhat, int k) {
  int x[3];
  node_xyz<D>(g, k, x);
  double y = 0.0;
#pragma unroll
  for (int ep = 0; ep < (1 << D); ep++) {
    int e[3] = {0, 0, 0};
    bool ok = true;
#pragma unroll
    for (int i = 0; i < D; i++) {
      e[i] = x[i] - 1 + ((ep >> i) & 1);
      ok = ok && (e[i] >= 0) && (e[i] < g.nc[i]);
    }
    if (!ok) continue;
    const int a = (~ep) & ((1 << D) - 1);
    const int q = elem_subcell<D>(A, P, g, e);
    if (g.fineop) {
      const int id = A.ids[fine_cell_index<D>(A, P, g, e, nullptr)];
      y += yhat[q * A.N + id];
    } else {
      for (int j = 0; j < A.N; j++) y += elem_m<D>(A, P, g, e, j, a) * yhat[q * A.N + j];
    }
  }
  if (g.fineop) y *= (D == 2) ? 0.25 * A.h * A.h : 0.125 * A.h * A.h * A.h;
  return y;
}

// (C^T yhat)_k with the subcell-interior fast path: if every element around node k lies in one
// subcell q, (C^T yhat)_k = sum_j nw[j][k] yhat[q][j] (nw precomputed per window, shared by the
// right-hand sides); interface nodes take the per-element path.
template <int D>
__device__ __forceinline__ double ct_fast(const LevelArgs& A, const ProbDesc& P, const Geo<D>& g,
                                          const double* __restrict__ nw, const double* yhat, int k) {
  int x[3];
  node_xyz<D>(g, k, x);
  bool interior = true;
  int q = 0;
#pragma unroll
  for (int i = D - 1; i >= 0; i--) {
    const int xi = x[i];
    const int t = P.lo[i] + xi * g.s + A.coff;
    const int v = fdiv(t, A.inv_c);
    if (xi > 0 && xi < g.nn[i] - 1 && v * A.c == t) interior = false;  // on a dual-block face
    const int e = (xi < g.nc[i]) ? xi : xi - 1;
    const int slot = fdiv(P.lo[i] + e * g.s + A.coff, A.inv_c) - P.k[i] + A.l;
    q = q * A.w + slot;
  }
  if (!interior) return ct_node<D>(A, P, g, yhat, k);
  double y = 0.0;
  for (int j = 0; j < A.N; j++) y += nw[(int64_t)j * g.nnodes + k] * yhat[q * A.N + j];
  return y;
}

// ---------------------------------------------------------------------------------------
// deterministic reductions

// sum `nv` values across the block; every thread gets the totals in out[] (smem, nv entries).
// scratch: >= 32*nv doubles.  Must be called by all threads.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* scratch, double* out) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int i = 0; i < NV; i++) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_down_sync(FULLMASK, v[i], o);
  }
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < NV; i++) scratch[wid * NV + i] = v[i];
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    double s = 0.0;
    for (int w = 0; w < nw; w++) s += scratch[w * NV + threadIdx.x];
    out[threadIdx.x] = s;
  }
  __syncthreads();
}

// Subcell element boxes at the problem's geometry: for each subcell q its element range.
// eb[q*6 + 0..2] = lo, eb[q*6 + 3..5] = extent (0 if the subcell is outside Omega).
template <int D>
__device__ void subcell_boxes(const LevelArgs& A, const ProbDesc& P, const Geo<D>& g, int* eb, int* ntask) {
  // thread 0 fills (nsub <= 125)
  if (threadIdx.x == 0) {
    int total = 0;
    for (int q = 0; q < A.nsub; q++) {
      int rem = q, cnt = 1;
      for (int i = 0; i < 3; i++) {
        int lo = 0, ext = (i < D) ? 0 : 1;
        if (i < D) {
          const int slot = rem % A.w;
          rem /= A.w;
          const int v = P.k[i] - A.l + slot;
          int flo = v * A.c - A.coff, fhi = flo + A.c;
          if (flo < 0) flo = 0;
          if (fhi > A.n) fhi = A.n;
          if (fhi <= flo) {
            ext = 0;
          } else {
            lo = (flo - P.lo[i]) / g.s;
            ext = (fhi - flo) / g.s;
          }
        }
        eb[q * 6 + i] = lo;
        eb[q * 6 + 3 + i] = ext;
        cnt *= ext;
      }
      eb[A.nsub * 6 + q] = total;  // task prefix (tasks of 32 elements)
      total += (cnt + 31) / 32;
    }
    eb[A.nsub * 6 + A.nsub] = total;
    *ntask = total;
  }
  __syncthreads();
}

// Contribution of element idx (< cnt) of subcell box bx to the N constraint rows of its subcell.
template <int D, typename UF>
__device__ __forceinline__ void cell_constraint_part(const LevelArgs& A, const ProbDesc& P, const Geo<D>& g,
                                                     const int* bx, int idx, UF uf, double (&part)[4]) {
  int e[3];
  const int i2 = (D == 3) ? fdiv(idx, 1.0f / (float)(bx[3] * bx[4])) : 0;
  const int r2 = idx - i2 * bx[3] * bx[4];
  const int i1 = fdiv(r2, 1.0f / (float)bx[3]);
  e[0] = bx[0] + r2 - i1 * bx[3];
  e[1] = bx[1] + i1;
  e[2] = bx[2] + i2;
  double u[1 << D];
#pragma unroll
  for (int b = 0; b < (1 << D); b++) {
    int xb[3] = {e[0] + (b & 1), e[1] + ((b >> 1) & 1), (D == 3) ? e[2] + ((b >> 2) & 1) : 0};
    u[b] = uf(node_id<D>(g, xb));
  }
  if (g.fineop) {
    const int id = A.ids[fine_cell_index<D>(A, P, g, e, nullptr)];
    double s = 0.0;
#pragma unroll
    for (int b = 0; b < (1 << D); b++) s += u[b];
    s *= (D == 2) ? 0.25 * A.h * A.h : 0.125 * A.h * A.h * A.h;
#pragma unroll
    for (int j = 0; j < 4; j++) part[j] = (j == id) ? s : 0.0;
  } else {
    for (int j = 0; j < A.N; j++) {
      double s = 0.0;
#pragma unroll
      for (int b = 0; b < (1 << D); b++) s += elem_m<D>(A, P, g, e, j, b) * u[b];
      part[j] = s;
    }
  }
}

// Large constraint counts (banded projector, 2D l >= 4): warp w owns the subcells q = w mod
// nwarps and sums each over its elements in a fixed order; out: ncon (no per-warp bins).
template <int D, typename UF>
__device__ void constraint_apply_owned(const LevelArgs& A, const ProbDesc& P, const Geo<D>& g, const int* eb, UF uf,
                                       double* out) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  for (int q = wid; q < A.nsub; q += nw) {
    const int* bx = eb + q * 6;
    const int cnt = bx[3] * bx[4] * bx[5];
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int idx = lane; idx < cnt; idx += 32) {
      double part[4] = {0.0, 0.0, 0.0, 0.0};
      cell_constraint_part<D>(A, P, g, bx, idx, uf, part);
#pragma unroll
      for (int j = 0; j < 4; j++) acc[j] += part[j];
    }
    for (int j = 0; j < A.N; j++) {
      double v = acc[j];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(FULLMASK, v, o);
      if (lane == 0) out[q * A.N + j] = v;
    }
  }
  __syncthreads();
}

// c[q*N+j] = sum_{E in R_q} sum_a m_{E,j,a} u(node(E,a)), u given by functor uf(node).
// eb: subcell boxes (see subcell_boxes); bins: nwarps*ncon scratch; out: ncon.
template <int D, typename UF>
__device__ void constraint_apply(const LevelArgs& A, const ProbDesc& P, const Geo<D>& g, const int* eb,
                                 int ntask, UF uf, double* bins, double* out) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  for (int i = threadIdx.x; i < nw * A.ncon; i += blockDim.x) bins[i] = 0.0;
  __syncthreads();
  const int* pref = eb + A.nsub * 6;
  for (int t = wid; t < ntask; t += nw) {
    int q = 0;
    while (pref[q + 1] <= t) q++;
    const int* bx = eb + q * 6;
    const int idx = (t - pref[q]) * 32 + lane;
    const int cnt = bx[3] * bx[4] * bx[5];
    double part[4] = {0.0, 0.0, 0.0, 0.0};
    if (idx < cnt) {
      int e[3];
      const int i2 = (D == 3) ? fdiv(idx, 1.0f / (float)(bx[3] * bx[4])) : 0;
      const int r2 = idx - i2 * bx[3] * bx[4];
      const int i1 = fdiv(r2, 1.0f / (float)bx[3]);
      e[0] = bx[0] + r2 - i1 * bx[3];
      e[1] = bx[1] + i1;
      e[2] = bx[2] + i2;
      double u[1 << D];
#pragma unroll
      for (int b = 0; b < (1 << D); b++) {
        int xb[3] = {e[0] + (b & 1), e[1] + ((b >> 1) & 1), (D == 3) ? e[2] + ((b >> 2) & 1) : 0};
        u[b] = uf(node_id<D>(g, xb));
      }
      if (g.fineop) {
        const int id = A.ids[fine_cell_index<D>(A, P, g, e, nullptr)];
        double s = 0.0;
#pragma unroll
        for (int b = 0; b < (1 << D); b++) s += u[b];
        s *= (D == 2) ? 0.25 * A.h * A.h : 0.125 * A.h * A.h * A.h;
#pragma unroll
        for (int j = 0; j < 4; j++) part[j] = (j == id) ? s : 0.0;
      } else {
        for (int j = 0; j < A.N; j++) {
          double s = 0.0;
#pragma unroll
          for (int b = 0; b < (1 << D); b++) s += elem_m<D>(A, P, g, e, j, b) * u[b];
          part[j] = s;
        }
      }
    }
    for (int j = 0; j < A.N; j++) {
      double v = part[j];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(FULLMASK, v, o);
      if (lane == 0) bins[wid * A.ncon + q * A.N + j] += v;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < A.ncon; i += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < nw; w++) s += bins[w * A.ncon + i];
    out[i] = s;
  }
  __syncthreads();
}
