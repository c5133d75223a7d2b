// On-chip projected PCG for 3D windows at levels >= 2 (sm_100a) and its per-node setup.
//
// Same method as k_pcg (kernels.cu) and k_pcg2d (pcg2d.cu): for each problem (macropoint p,
// right-hand side r) the correction problem of Eqs. (12)/(13) on the level-n
// grid, min 1/2 x^T A x - b^T x s.t. C x = g, by projected Jacobi-PCG with the residual
// re-projected every iteration (readings R16, R19).
//
//   p          shared memory, zero halo planes in y and z; x-neighbours by warp shuffles
//   r, q, x    global memory (L2-resident: <= 125 KB each per problem)
//   A_n        per-node 27-point stencil rows of A_n = P_n^T A_1 P_n (reading R11), precomputed
//              per window by k_node_ops3d (streamed from L2, shared by the right-hand sides)
//   C_n        per-node constraint weights m_{E,j,a} = int_E psi_j N_a merged over the elements
//              around the node that lie in one subcell, per octant (k_node_ops3d)
//
// Thread layout: warp y owns node row y of every plane, lane x its node x (windows of at most
// NXM <= 25 nodes per side, so a row fits a warp); every thread walks its column in z.  The
// constraint vector c = C D^-1 r is accumulated per thread for the current subcell layer in z,
// merged across x by one shuffle, reduced per warp with a segmented scan keyed by the subcell
// column and written to per-row bins; the bins are summed over rows in a fixed order, so every
// run gives bitwise identical results.  Five block barriers per iteration.
#include <cuda_runtime.h>

#include <cstdio>

#include "device_common.cuh"
#include "kernels.h"

#include "pcg3d_common.cuh"

#ifndef MCH_P13_MINB
#define MCH_P13_MINB 3  // CTAs per SM of the 13-node windows: 3 (80 registers, some spills) beat 2 (128): c5 level-3 PCG 31.0 -> 28.1 ms
#endif

// ------------------------------------------------------------------------------------------
// per-node stencil rows STC[27][nodes] (offset (dx+1) + 3(dy+1) + 9(dz+1)) and octant-merged
// constraint weights MW[8][N][nodes] (octant o = xs + 2 ys + 4 zs, sides as in Sides) of every
// window of the batch.  grid (ceil(max nodes / 128), macropoints)
template <int N>
__global__ void k_node_ops3d(LevelArgs A) {
  const int mp = blockIdx.y;
  const ProbDesc& P = A.probs[mp];
  const Geo<3> g = level_geo<3>(A, P);
  const int nn = g.nnodes;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nn) return;
  int X[3];
  node_xyz<3>(g, k, X);
  double st[27];
  double mw[8][N];
  for (int i = 0; i < 27; i++) st[i] = 0.0;
  for (int o = 0; o < 8; o++)
    for (int j = 0; j < N; j++) mw[o][j] = 0.0;
  Sides sd[3];
  for (int i = 0; i < 3; i++) sd[i] = sides_of(A, P, i, X[i], g.nc[i]);
  for (int o = 0; o < 8; o++) {
    int e[3];
    bool ok = true;
    int t = 0;
    for (int i = 0; i < 3; i++) {
      const int ob = (o >> i) & 1;
      e[i] = X[i] - 1 + ob;
      ok = ok && e[i] >= 0 && e[i] < g.nc[i];
      const int tb = (sd[i].pm == 3) ? ob : ((sd[i].pm == 2) ? 1 : 0);
      t |= tb << i;
    }
    if (!ok) continue;
    double W[DimC<3>::NW];
    elem_W<3>(A, P, g, e, W);
    const int a = (~o) & 7;  // corner of the node in element e
    for (int b = 0; b < 8; b++) {
      // (K_E)_ab = elem_row(W, e_b, a) written out: per direction k one weight, sign + if a_k = 1,
      // times + if b_k = 1 (the pair partner b ^ (1 << k) has b_k = 0)
      double kab = 0.0;
#pragma unroll
      for (int kk = 0; kk < 3; kk++) {
        const double w = W[kk * DimC<3>::NT + pair_type<3>(kk, a, b)];
        kab += ((((a ^ b) >> kk) & 1) ? -w : w);
      }
      const int dx = e[0] + (b & 1) - X[0], dy = e[1] + ((b >> 1) & 1) - X[1], dz = e[2] + ((b >> 2) & 1) - X[2];
      st[(dx + 1) + 3 * (dy + 1) + 9 * (dz + 1)] += kab;
    }
    for (int j = 0; j < N; j++) mw[t][j] += elem_m<3>(A, P, g, e, j, a);
  }
  const int64_t base = A.stc_pad ? (int64_t)mp * A.stc_pad : P.node_off;
  const int stride = A.stc_pad ? A.stc_pad : nn;
  double* so = A.STC + base * 27;
  for (int c = 0; c < 27; c++) so[(int64_t)c * stride + k] = st[c];
  double* mo = A.MLR + base * 8 * N;
  for (int o = 0; o < 8; o++)
    for (int j = 0; j < N; j++) mo[(int64_t)(o * N + j) * stride + k] = mw[o][j];
}

// ------------------------------------------------------------------------------------------
// the solver: one CTA per problem (macropoint, rhs).  A row of the window occupies LPR lanes
// (32, 16 or 8: the smallest that holds NXM nodes), so a warp carries RPW = 32 / LPR rows at a
// time; NW warps, RW rounds of rows each.
template <int N, int NXM, int RW, int MINB>
__global__ void __launch_bounds__(32 * ((NXM + (32 / ((NXM > 16) ? 32 : ((NXM > 8) ? 16 : 8))) * RW - 1) /
                                        ((32 / ((NXM > 16) ? 32 : ((NXM > 8) ? 16 : 8))) * RW)),
                                  MINB) k_pcg3d(LevelArgs A) {
  constexpr int LPR = (NXM > 16) ? 32 : ((NXM > 8) ? 16 : 8);  // lanes per row
  constexpr int RPW = 32 / LPR;                                 // rows per warp and round
  constexpr int NW = (NXM + RPW * RW - 1) / (RPW * RW);
  constexpr int PY = NXM + 2;   // p_s rows per plane (zero halo rows y = -1, ny)
  constexpr int PZ = PY * NXM;  // p_s plane (x pitch NXM, no x halo: x-neighbours by shuffle)
  constexpr int NQ = 27 * N;    // constraint rows of a 3x3x3-subcell window
  const int prob = blockIdx.x;
  const int mp = prob / A.n_rhs, rhs = prob - mp * A.n_rhs;
  const ProbDesc& P = A.probs[mp];
  const int nx = P.nc[0] + 1, ny = P.nc[1] + 1, nz = P.nc[2] + 1, nn = nx * ny * nz;
  const int ncx = nx - 1;
  const int nc = A.ncon;  // == NQ (host check)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int x = lane & (LPR - 1), ry = lane / LPR;
  const bool xin = x < NXM;
  // current row of this lane group: set by set_row
  int y = warp;
  bool wact = false, lact = false;  // wact warp-uniform (some row of the warp is in the window)

  extern __shared__ __align__(16) double smem[];
  double* p_s = smem;                  // [NXM+2][PY][NXM], zero halo planes / rows
  double* bins = p_s + (NXM + 2) * PZ;  // [NXM rows][NQ]
  double* Ysh = bins + NXM * NQ;        // [NQ] yhat
  double* csh = Ysh + NQ;               // [NQ] c
  double* slots = csh + NQ;             // [5][32] scalar partial sums
  double* zr = slots + 5 * 32;          // [256] coarse: E^-1 Z^T r
  double* vv = zr + 256;                // [256] coarse: coarse part of z
  int* zsm = reinterpret_cast<int*>(vv + 256);  // [NXM][3] z sides (pm, k0, k1)

  for (int i = threadIdx.x; i < (NXM + 2) * PZ; i += blockDim.x) p_s[i] = 0.0;
  for (int i = threadIdx.x; i < NXM * NQ + 2 * NQ + 5 * 32; i += blockDim.x) bins[i] = 0.0;
  for (int z = threadIdx.x; z < nz; z += blockDim.x) {
    const Sides s = sides_of(A, P, 2, z, nz - 1);
    zsm[z * 3] = s.pm;
    zsm[z * 3 + 1] = s.k0;
    zsm[z * 3 + 2] = s.k1;
  }
  Sides sx{0, 0, 0}, sy{0, 0, 0}, syr[RW];
  if (x < nx) sx = sides_of(A, P, 0, x, ncx);
#pragma unroll
  for (int ri = 0; ri < RW; ri++) {
    const int yy = (warp + ri * NW) * RPW + ry;
    syr[ri] = (yy < ny) ? sides_of(A, P, 1, yy, ny - 1) : Sides{0, 0, 0};
  }
  const int kxe = (x < ncx) ? slot3(A, P, 0, x) : 1000;  // subcell column of element x
  const int kseg = ry * 1024 + kxe;                      // scan key: never equal across rows
  auto set_row = [&](int ri) {
    const int yb = (warp + ri * NW) * RPW;
    y = yb + ry;
    wact = yb < ny;
    lact = (y < ny) && x < nx;
    sy = syr[ri];
  };
  __syncthreads();

  constexpr int PAD = NXM * NXM * NXM;  // fixed node stride of STC / MLR (A.stc_pad): offsets c PAD are immediates
  const double* S27 = A.STC + (int64_t)mp * 27 * PAD;
  const double* MW = A.MLR + (int64_t)mp * 8 * N * PAD;
  const double* dg = A.dinv + P.node_off;
  double* Xv = A.X + P.vec_off + (int64_t)rhs * nn;
  double* Rv = A.R + P.vec_off + (int64_t)rhs * nn;
  double* Qv = A.Q + P.vec_off + (int64_t)rhs * nn;
  const double* Si = A.Sinv + (int64_t)mp * nc * nc;
  const double* gsrc = A.g;  // levels >= 2 only
  const double* bvec = A.B + P.vec_off + (int64_t)rhs * nn;

  auto rows = [&](auto&& f) {
#pragma unroll
    for (int ri = 0; ri < RW; ri++) {
      set_row(ri);
      f();
    }
  };
  auto nidx = [&](int z) { return (z * ny + y) * nx + x; };
  auto pidx = [&](int z) { return (z + 1) * PZ + (y + 1) * NXM + x; };

  // (C^T yhat)_k over the present octants
  auto ct_at = [&](int z, int k) -> double {
    const int pmz = zsm[z * 3];
    double ct = 0.0;
#pragma unroll
    for (int zs = 0; zs < 2; zs++) {
      if (!((pmz >> zs) & 1)) continue;
      const int kz = zsm[z * 3 + 1 + zs];
#pragma unroll
      for (int ys = 0; ys < 2; ys++) {
        if (!((sy.pm >> ys) & 1)) continue;
        const int ky = ys ? sy.k1 : sy.k0;
#pragma unroll
        for (int xs = 0; xs < 2; xs++) {
          if (!((sx.pm >> xs) & 1)) continue;
          const int kx = xs ? sx.k1 : sx.k0;
          const int o = xs + 2 * ys + 4 * zs;
          const double* yq = Ysh + ((kz * 3 + ky) * 3 + kx) * N;
#pragma unroll
          for (int j = 0; j < N; j++) ct += __ldg(MW + (o * N + j) * PAD + k) * yq[j];
        }
      }
    }
    return ct;
  };

  // constraint accumulation: acc[ys][xs][j] for the current subcell layer in z
  double acc[2][2][N];
  auto acc_zero = [&]() {
#pragma unroll
    for (int a = 0; a < 2; a++)
#pragma unroll
      for (int b = 0; b < 2; b++)
#pragma unroll
        for (int j = 0; j < N; j++) acc[a][b][j] = 0.0;
  };
  auto acc_add = [&](int zs, int k, double u) {
#pragma unroll
    for (int ys = 0; ys < 2; ys++) {
      if (!((sy.pm >> ys) & 1)) continue;
#pragma unroll
      for (int xs = 0; xs < 2; xs++) {
        if (!((sx.pm >> xs) & 1)) continue;
        const int o = xs + 2 * ys + 4 * zs;
#pragma unroll
        for (int j = 0; j < N; j++) acc[ys][xs][j] += __ldg(MW + (o * N + j) * PAD + k) * u;
      }
    }
  };
  // warp-collective (wact warps): layer kz of each row -> bins[y]
  auto flush = [&](int kz) {
#pragma unroll
    for (int ys = 0; ys < 2; ys++) {
      const bool has = (sy.pm >> ys) & 1;  // per row (acc is zero where the side is absent)
      const int ky = ys ? sy.k1 : sy.k0;
      double v[N];
#pragma unroll
      for (int j = 0; j < N; j++) {
        const double t = __shfl_down_sync(FULLMASK, acc[ys][0][j], 1);  // element x of lane x+1
        v[j] = acc[ys][1][j] + ((x < LPR - 1) ? t : 0.0);
      }
      const int kup = __shfl_up_sync(FULLMASK, kseg, 1);
      const unsigned hm = __ballot_sync(FULLMASK, lane == 0 || kseg != kup);
      const int head = 31 - __clz(hm & (0xffffffffu >> (31 - lane)));
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
        for (int j = 0; j < N; j++) {
          const double t = __shfl_up_sync(FULLMASK, v[j], d);
          if (lane - d >= head) v[j] += t;
        }
      }
      const bool tail = (lane == 31) || ((hm >> (lane + 1)) & 1u);
      if (tail && kxe < 1000 && has && y < ny) {
        double* B = bins + y * NQ + ((kz * 3 + ky) * 3 + kxe) * N;
#pragma unroll
        for (int j = 0; j < N; j++) B[j] = v[j];
      }
    }
    acc_zero();
  };
  // walk the column accumulating u(z, k) into the constraint bins (wact warps)
  auto sweep_c = [&](auto&& ufun) {
    acc_zero();
    int layer = 0;
    for (int z = 0; z < nz; z++) {
      const int k = nidx(z);
      const double u = ufun(z, k);
      const int pmz = zsm[z * 3];
      if (pmz == 3) {
        if (lact) acc_add(0, k, u);
        flush(zsm[z * 3 + 1]);
        if (lact) acc_add(1, k, u);
        layer = zsm[z * 3 + 2];
      } else {
        if (lact) acc_add((pmz == 2) ? 1 : 0, k, u);
        layer = (pmz == 2) ? zsm[z * 3 + 2] : zsm[z * 3 + 1];
      }
    }
    flush(layer);
  };
  // (A p)_k from p_s: f(z, k, Ap, p_k)  (wact warps; lanes >= nx carry zeros)
  auto sweep_stencil = [&](auto&& f) {
    const double* pb = p_s + (y + 1) * NXM + x;
    double v[3][3];  // [dy][dz]
#pragma unroll
    for (int dy = 0; dy < 3; dy++) {
      v[dy][0] = xin ? pb[(dy - 1) * NXM] : 0.0;
      v[dy][1] = xin ? pb[PZ + (dy - 1) * NXM] : 0.0;
    }
    for (int z = 0; z < nz; z++) {
#pragma unroll
      for (int dy = 0; dy < 3; dy++) v[dy][2] = xin ? pb[(z + 2) * PZ + (dy - 1) * NXM] : 0.0;
      const int k = nidx(z);
      double cf[27];  // all 27 coefficient loads in flight before the first use
#pragma unroll
      for (int c = 0; c < 27; c++) cf[c] = lact ? __ldg(S27 + c * PAD + k) : 0.0;
      double Ap = 0.0;
#pragma unroll
      for (int dz = 0; dz < 3; dz++)
#pragma unroll
        for (int dy = 0; dy < 3; dy++) {
          const double c0 = v[dy][dz];
          double l = __shfl_up_sync(FULLMASK, c0, 1);
          double r = __shfl_down_sync(FULLMASK, c0, 1);
          if (x == 0) l = 0.0;
          if (x == LPR - 1) r = 0.0;
          const int cb = 9 * dz + 3 * dy;
          Ap += cf[cb] * l + cf[cb + 1] * c0 + cf[cb + 2] * r;
        }
      f(z, k, Ap, v[1][1]);
#pragma unroll
      for (int dy = 0; dy < 3; dy++) {
        v[dy][0] = v[dy][1];
        v[dy][1] = v[dy][2];
      }
    }
  };

  auto slot_put = [&](int which, double v) {
    v = wsum0(v);
    if (lane == 0) slots[which * 32 + warp] = v;
  };
  auto slot_fin = [&](int which) { return wsum0((lane < NW) ? slots[which * 32 + lane] : 0.0); };
  // c = sum over rows of the bins (fixed order) into csh; call between barriers
  auto reduce_c = [&]() {  // one warp per constraint row, fixed tree over the row bins
    for (int i = warp; i < nc; i += NW) {
      double s = 0.0;
      for (int yy = lane; yy < ny; yy += 32) s += bins[yy * NQ + i];
      s = wsum0(s);
      if (lane == 0) csh[i] = s;
    }
  };
  // Ysh = S^-1 csh (rows over warps), slots[3] = per-warp partial c.yhat; call between barriers
  auto solve_y = [&]() {
    double cyw = 0.0;
    for (int i = warp; i < nc; i += NW) {
      double s = 0.0;
      for (int j = lane; j < nc; j += 32) s += __ldg(Si + (int64_t)i * nc + j) * csh[j];
      s = wsum0(s);
      if (lane == 0) Ysh[i] = s;
      cyw += s * csh[i];
    }
    if (lane == 0) slots[3 * 32 + warp] = cyw;
  };

  // two-level preconditioner, as in k_pcg3d_l1
  const bool crs = A.coarse && A.ncomp[mp] > 0;
  const int nca = crs ? A.ncomp[mp] : 0;
  const int* cmp = A.cmap + P.node_off;
  const int* cpt = A.cptr + (int64_t)mp * (A.ncmax + 1);
  const int* cls = A.clist + P.node_off;
  const double* Eiv = A.Einv + (int64_t)mp * A.ncmax;
  const double* CZm = A.CZ + (int64_t)mp * nc * A.ncmax;
  auto coarse_c = [&]() {  // zr, slot 4, csh += (CZ) zr; two barriers
    double part = 0.0;
    const int sub = lane & 3, ngrp = blockDim.x >> 2;
    for (int a0 = threadIdx.x >> 2; a0 - (int)(threadIdx.x >> 2) < nca; a0 += ngrp) {
      const int a = a0;
      double sv = 0.0;
      if (a < nca) {
        const int i0 = __ldg(cpt + a), i1 = __ldg(cpt + a + 1);
        for (int i = i0 + sub; i < i1; i += 4) sv += __ldcg(Rv + __ldg(cls + i));
      }
      sv += __shfl_xor_sync(FULLMASK, sv, 1);
      sv += __shfl_xor_sync(FULLMASK, sv, 2);
      if (a < nca && sub == 0) {
        const double ei = __ldg(Eiv + a);
        zr[a] = sv * ei;
        part += sv * sv * ei;
      }
    }
    part = wsum0(part);
    if (lane == 0) slots[4 * 32 + warp] = part;
    __syncthreads();
    for (int t = warp; t < nc; t += NW) {
      double sv = 0.0;
      for (int a = lane; a < nca; a += 32) sv += __ldg(CZm + (int64_t)t * A.ncmax + a) * zr[a];
      sv = wsum0(sv);
      if (lane == 0) csh[t] += sv;
    }
    __syncthreads();
  };
  auto coarse_v = [&](double s0) {  // vv = s0 zr - E^-1 (CZ)^T Ysh; one barrier
    for (int a = threadIdx.x; a < nca; a += blockDim.x) {
      double acc = 0.0;
      for (int t = 0; t < nc; t++) acc += __ldg(CZm + (int64_t)t * A.ncmax + a) * Ysh[t];
      vv[a] = (s0 != 0.0 ? s0 * zr[a] : 0.0) - __ldg(Eiv + a) * acc;
    }
    __syncthreads();
  };
  auto cz_at = [&](int k) -> double {
    if (!crs) return 0.0;
    const int a = __ldg(cmp + k);
    return (a >= 0) ? vv[a] : 0.0;
  };

  // ---- init: x0 = D^-1 C^T S^-1 t, r0 = A x0 - b, c = C D^-1 r0, yhat = S^-1 c; returns r0^T D^-1 r0
  auto init = [&](const double* tcol, const double* bb) -> double {
    for (int i = threadIdx.x; i < nc; i += blockDim.x) csh[i] = tcol[((int64_t)mp * nc + i) * A.n_rhs + rhs];
    __syncthreads();
    solve_y();
    __syncthreads();
    if (crs) coarse_v(0.0);
    rows([&] {
      if (lact)
        for (int z = 0; z < nz; z++) {
          const int k = nidx(z);
          const double x0 = dg[k] * ct_at(z, k) - cz_at(k);
          p_s[pidx(z)] = x0;
          Xv[k] = x0;
        }
    });
    __syncthreads();
    rows([&] {
      if (wact)
        sweep_stencil([&](int, int k, double Ap, double) {
          if (lact) Rv[k] = Ap - (bb ? bb[k] : 0.0);
        });
    });
    double rr = 0.0;
    rows([&] {
      if (wact)
        sweep_c([&](int, int k) -> double {
          if (!lact) return 0.0;
          const double rk = Rv[k];
          const double u = dg[k] * rk;
          rr += rk * u;
          return u;
        });
    });
    slot_put(2, rr);
    __syncthreads();
    reduce_c();
    __syncthreads();
    if (crs) coarse_c();
    solve_y();
    __syncthreads();
    const double rrt = slot_fin(2) + (crs ? slot_fin(4) : 0.0);
    if (crs) coarse_v(1.0);
    return rrt;
  };

  // reference scale: initial projected residual of the full (non-hierarchical) problem
  const double rr_ref = init(A.g0, nullptr);
  double rz_ref;
  {
    double v = 0.0;
    rows([&] {
      if (lact)
        for (int z = 0; z < nz; z++) {
          const int k = nidx(z);
          const double w = Rv[k] - ct_at(z, k);
          v += dg[k] * w * w;
        }
    });
    slot_put(0, v);
    __syncthreads();
    rz_ref = slot_fin(0);
    __syncthreads();
  }
  const double rr0 = init(gsrc, bvec);

  const double tol2 = A.rtol * A.rtol;
  const double floor2 = 1e-30 * fmax(rr0, rr_ref);
  double beta = 0.0, rz = 0.0, ref = 0.0, alpha = 0.0;
  int it = 0, breakdown = 0;
  for (;; it++) {
    // pass A: x += alpha_prev p_prev (deferred), r <- r - C^T yhat, z = D^-1 r, p <- -z + beta p
    double v = 0.0;
    rows([&] {
      if (!lact) return;
      const bool first = (it == 0);
      for (int z = 0; z < nz; z++) {
        const int k = nidx(z);
        const double rk = Rv[k] - ct_at(z, k);
        const double zz = dg[k] * rk + cz_at(k);
        double& pk = p_s[pidx(z)];
        const double pold = pk;
        if (!first) Xv[k] += alpha * pold;
        pk = first ? -zz : -zz + beta * pold;
        Rv[k] = rk;
        v += rk * zz;
      }
    });
    slot_put(0, v);
    __syncthreads();  // B1: p complete
    // pass B: q = A p, pq
    double w = 0.0;
    rows([&] {
      if (wact)
        sweep_stencil([&](int, int k, double Ap, double pk) {
          if (lact) {
            Qv[k] = Ap;
            w += pk * Ap;
          }
        });
    });
    slot_put(1, w);
    __syncthreads();  // B2
    rz = slot_fin(0);
    const double pq = slot_fin(1);
    if (it == 0) ref = fmax(rz, rz_ref);
    if (!(rz > fmax(tol2 * ref, floor2)) || it >= A.max_iter) break;
    if (!(pq > 0.0) || !isfinite(pq)) {
      breakdown = 1;
      break;
    }
    alpha = rz / pq;
    // pass C: r += alpha q, rr = r^T D^-1 r, c = C D^-1 r (per row)
    double rr = 0.0;
    rows([&] {
      if (wact)
        sweep_c([&](int, int k) -> double {
          if (!lact) return 0.0;
          const double rk = Rv[k] + alpha * Qv[k];
          Rv[k] = rk;
          const double u = dg[k] * rk;
          rr += rk * u;
          return u;
        });
    });
    slot_put(2, rr);
    __syncthreads();  // B3
    reduce_c();
    __syncthreads();  // B3b
    if (crs) coarse_c();
    solve_y();
    __syncthreads();  // B4
    const double cy = slot_fin(3);
    beta = (slot_fin(2) + (crs ? slot_fin(4) : 0.0) - cy) / rz;
    if (crs) coarse_v(1.0);
  }

  // feasibility restoration: x += D^-1 C^T S^-1 (g - C x)
  rows([&] {
    if (wact) sweep_c([&](int, int k) -> double { return lact ? Xv[k] : 0.0; });
  });
  __syncthreads();
  for (int i = threadIdx.x; i < nc; i += blockDim.x) {
    double s = 0.0;
    for (int yy = 0; yy < ny; yy++) s += bins[yy * NQ + i];
    csh[i] = gsrc[((int64_t)mp * nc + i) * A.n_rhs + rhs] - s;
  }
  __syncthreads();
  solve_y();
  __syncthreads();
  if (crs) coarse_v(0.0);
  rows([&] {
    if (lact)
      for (int z = 0; z < nz; z++) {
        const int k = nidx(z);
        Xv[k] += dg[k] * ct_at(z, k) - cz_at(k);
      }
  });
  if (threadIdx.x == 0) {
    A.iters[prob] = it;
    A.relres[prob] = (ref > 0.0) ? sqrt(fmax(rz, 0.0) / ref) : 0.0;
    double* dgo = A.diag + (int64_t)prob * 4;
    dgo[0] = rz;
    dgo[1] = ref;
    dgo[2] = floor2;
    dgo[3] = breakdown;
  }
}

// ------------------------------------------------------------------------------------------
// Level 1 (fine grid, windows of <= 49 nodes per side), same method and barriers as k_pcg3d.
// One CTA of NW = 14 or 7 warps per problem; task t = (node row y = t / 2, segment t % 2 of 32 nodes
// in x), 98 / NW tasks per warp.  p lives in global memory (its three active planes stay in L1); every thread
// walks its column in z with a sliding 3x3x3 window of p (9 loads per node) and a sliding 2x2x2
// window of the cells' kappa and ids (4 loads per node).  Operator: the Q1 element rows
// kappa h/12 (4 p_a - p_{a^3} - p_{a^5} - p_{a^6} - p_{a^7}) summed over the 8 cells;
// constraint weights m_{E,j,a} = [id_E = j] h^3/8.
//
// MODE 1 (transport, levels >= 2): the same walkers on the fine window of the problem compute
// Y = A_1 I_p (into FY) and g = g^0 - C_1 I_p from the transported field I_p (FI), replacing the
// generic per-node gather of k_transport (Eqs. 12-13; reading R9).
template <int N, int NW, int MODE = 0>
__global__ void __launch_bounds__(NW * 32, 448 / (NW * 32)) k_pcg3d_l1(LevelArgs A) {
  constexpr int NT = 98, RW = NT / NW;  // 98 row segments = 49 rows x 2
  constexpr int NQ = 27 * N;
  const int prob = blockIdx.x;
  const int mp = prob / A.n_rhs, rhs = prob - mp * A.n_rhs;
  const ProbDesc& P = A.probs[mp];
  const int* ncv = (MODE == 0) ? P.nc : P.ncf;  // fine cells of the window in both modes
  const int nx = ncv[0] + 1, ny = ncv[1] + 1, nz = ncv[2] + 1, nn = nx * ny * nz;
  const int ncx = nx - 1, ncy = ny - 1, ncz = nz - 1;
  const int nc = A.ncon;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t n = A.n;

  extern __shared__ __align__(16) double smem[];
  double* bins = smem;          // [NT task rows][NQ]
  double* Ysh = bins + NT * NQ;  // [NQ]
  double* csh = Ysh + NQ;        // [NQ]
  double* slots = csh + NQ;      // [5][32]
  double* zr = slots + 5 * 32;   // [256] coarse: E^-1 Z^T r
  double* vv = zr + 256;         // [256] coarse: coarse part of z
  int* zsm = reinterpret_cast<int*>(vv + 256);  // [49][3]
  for (int i = threadIdx.x; i < NT * NQ + 2 * NQ + 5 * 32; i += blockDim.x) bins[i] = 0.0;
  for (int z = threadIdx.x; z < nz; z += blockDim.x) {
    const Sides sd = sides_of(A, P, 2, z, ncz, 1);
    zsm[z * 3] = sd.pm;
    zsm[z * 3 + 1] = sd.k0;
    zsm[z * 3 + 2] = sd.k1;
  }
  __syncthreads();

  int t = 0, y = 0, seg = 0, x = 0, kxe = 1000;
  bool wact = false, lact = false;
  Sides sx{0, 0, 0}, sy{0, 0, 0};
  const int nxy = nx * ny;
  const int64_t n2 = (int64_t)A.n * A.n;
  unsigned pvm = 0;      // bit dy*3+dx: p neighbour (x+dx-1, y+dy-1) inside the window
  unsigned cvm = 0;      // bit oy*2+ox: cell (x-1+ox, y-1+oy) inside the window
  int64_t cbase = 0;     // global index of cell (x-1, y-1, -1) of the window
  auto tside = [](int pm, int ob) { return (pm == 3) ? ob : ((pm == 2) ? 1 : 0); };
  // subcell of the cell in xy-octant oxy = ox + 2 oy: ky * 3 + kx (per task)
  auto kxy = [&](int oxy) {
    const int ox = oxy & 1, oy = oxy >> 1;
    const int kx = ox ? ((sx.pm == 1) ? sx.k0 : sx.k1) : sx.k0;
    const int ky = oy ? ((sy.pm == 1) ? sy.k0 : sy.k1) : sy.k0;
    return ky * 3 + kx;
  };
  int kq[4];  // kxy per xy-octant of the current task (set by prep_keys)
  auto prep_keys = [&]() {
#pragma unroll
    for (int o = 0; o < 4; o++) kq[o] = kxy(o);
  };
  auto set_task = [&](int ri) {
    t = warp + ri * NW;
    y = t >> 1;
    seg = t & 1;
    x = seg * 32 + lane;
    wact = (y < ny) && (seg * 32 < nx);
    lact = wact && x < nx;
    sx = lact ? sides_of(A, P, 0, x, ncx, 1) : Sides{0, 0, 0};
    sy = wact ? sides_of(A, P, 1, y, ncy, 1) : Sides{0, 0, 0};
    kxe = (lact && x < ncx) ? slot3(A, P, 0, x, 1) : 1000;
    pvm = 0;
    cvm = 0;
    if (lact) {
#pragma unroll
      for (int dy = 0; dy < 3; dy++)
#pragma unroll
        for (int dx = 0; dx < 3; dx++) {
          const int xx = x + dx - 1, yy = y + dy - 1;
          if (xx >= 0 && xx < nx && yy >= 0 && yy < ny) pvm |= 1u << (dy * 3 + dx);
        }
#pragma unroll
      for (int o = 0; o < 4; o++) {
        const int ex = x - 1 + (o & 1), ey = y - 1 + (o >> 1);
        if (ex >= 0 && ex < ncx && ey >= 0 && ey < ncy) cvm |= 1u << o;
      }
    }
    cbase = ((int64_t)(P.lo[2] - 1) * A.n + (P.lo[1] + y - 1)) * A.n + (P.lo[0] + x - 1);
    prep_keys();
  };
  auto tasks = [&](auto&& f) {
    for (int ri = 0; ri < RW; ri++) {
      set_task(ri);
      f();
    }
  };

  const double* dg = A.dinv + P.node_off;
  double* pv = (MODE == 0) ? A.P + P.vec_off + (int64_t)rhs * nn : A.FI + P.fine_off + (int64_t)rhs * nn;
  double* Xv = A.X + P.vec_off + (int64_t)rhs * nn;
  double* Rv = A.R + P.vec_off + (int64_t)rhs * nn;
  double* Qv = A.Q + P.vec_off + (int64_t)rhs * nn;
  const double* Si = A.Sinv + (int64_t)mp * nc * nc;
  const double hq = 0.125 * A.h * A.h * A.h, kh = A.h * (1.0 / 12.0);
  auto nidx = [&](int z) { return (z * ny + y) * nx + x; };
  // fine cell (x-1+ox, y-1+oy, ez) of the window: kappa (0 outside) and id (0xFF outside)

  // column walkers over the cell ids: f(z, k, id[8]) with id[o] of cell octant o
  auto walk_ids = [&](auto&& f) {
    int idc[8];
    const uint8_t* ip = A.ids + cbase + n2;  // cell (x-1, y-1) of cell plane 0
    const int oxy[4] = {0, 1, (int)A.n, (int)A.n + 1};
#pragma unroll
    for (int o = 0; o < 4; o++) {
      idc[o] = 0xFF;
      idc[4 + o] = (((cvm >> o) & 1u) && ncz > 0) ? __ldg(ip + oxy[o]) : 0xFF;
    }
    int k = y * nx + x;
    for (int z = 0; z < nz; z++) {
      ip += n2;
      const bool nv = z + 1 < ncz;
      int nxt[4];
#pragma unroll
      for (int o = 0; o < 4; o++) nxt[o] = (((cvm >> o) & 1u) && nv) ? __ldg(ip + oxy[o]) : 0xFF;  // next plane
      f(z, k, idc);
      k += nxy;
#pragma unroll
      for (int o = 0; o < 4; o++) {
        idc[o] = idc[4 + o];
        idc[4 + o] = nxt[o];
      }
    }
  };
  auto ct_of = [&](int z, const int (&idc)[8]) -> double {
    const int pmz = zsm[z * 3];
    const int kz0 = zsm[z * 3 + 1] * 9, kz1 = ((pmz == 1) ? zsm[z * 3 + 1] : zsm[z * 3 + 2]) * 9;
    double ct = 0.0;
#pragma unroll
    for (int o = 0; o < 8; o++)
      if (idc[o] != 0xFF) ct += Ysh[(((o >> 2) ? kz1 : kz0) + kq[o & 3]) * N + idc[o]];
    return ct * hq;
  };

  // constraint accumulation for the current subcell layer in z, per xy-octant of the cells
  double acc[4][N];
  auto acc_zero = [&]() {
#pragma unroll
    for (int a = 0; a < 4; a++)
#pragma unroll
      for (int j = 0; j < N; j++) acc[a][j] = 0.0;
  };
  // add u h^3/8 for the cells whose z side is zsel
  auto acc_add = [&](int zsel, int z, const int (&idc)[8], double u) {
    const int pmz = zsm[z * 3];
    const double w = u * hq;
#pragma unroll
    for (int oz = 0; oz < 2; oz++) {
      if (tside(pmz, oz) != zsel) continue;  // uniform per plane
#pragma unroll
      for (int oxy = 0; oxy < 4; oxy++) {
        const int id = idc[oz * 4 + oxy];
#pragma unroll
        for (int j = 0; j < N; j++) acc[oxy][j] += (id == j) ? w : 0.0;
      }
    }
  };
  auto flush = [&](int kz) {
    double* B = bins + t * NQ;
#pragma unroll
    for (int ys = 0; ys < 2; ys++) {
      if (!((sy.pm >> ys) & 1)) continue;  // warp-uniform
      const int ky = ys ? sy.k1 : sy.k0;
      double g[2][N];  // side groups xs of this ys
#pragma unroll
      for (int xs = 0; xs < 2; xs++)
#pragma unroll
        for (int j = 0; j < N; j++) {
          double a = 0.0;
#pragma unroll
          for (int oxy = 0; oxy < 4; oxy++)
            if (tside(sy.pm, oxy >> 1) == ys && tside(sx.pm, oxy & 1) == xs) a += acc[oxy][j];
          g[xs][j] = a;
        }
      double v[N];
#pragma unroll
      for (int j = 0; j < N; j++) {
        const double tt = __shfl_down_sync(FULLMASK, g[0][j], 1);
        v[j] = g[1][j] + ((lane < 31) ? tt : 0.0);
      }
      const int kup = __shfl_up_sync(FULLMASK, kxe, 1);
      const unsigned hm = __ballot_sync(FULLMASK, lane == 0 || kxe != kup);
      const int head = 31 - __clz(hm & (0xffffffffu >> (31 - lane)));
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
        for (int j = 0; j < N; j++) {
          const double tt = __shfl_up_sync(FULLMASK, v[j], d);
          if (lane - d >= head) v[j] += tt;
        }
      }
      const bool tail = (lane == 31) || ((hm >> (lane + 1)) & 1u);
      if (tail && kxe < 1000) {
#pragma unroll
        for (int j = 0; j < N; j++) B[((kz * 3 + ky) * 3 + kxe) * N + j] += v[j];
      }
      __syncwarp();
      if (lane == 0 && lact && x >= 1) {  // element x-1 belongs to the previous segment's lane 31
#pragma unroll
        for (int j = 0; j < N; j++) B[((kz * 3 + ky) * 3 + sx.k0) * N + j] += g[0][j];
      }
      __syncwarp();
    }
    acc_zero();
  };
  auto sweep_c = [&](auto&& ufun) {
    for (int i = lane; i < NQ; i += 32) bins[t * NQ + i] = 0.0;
    __syncwarp();
    acc_zero();
    int layer = 0;
    walk_ids([&](int z, int k, const int (&idc)[8]) {
      const double u = ufun(z, k);
      const int pmz = zsm[z * 3];
      if (pmz == 3) {
        acc_add(0, z, idc, u);
        flush(zsm[z * 3 + 1]);
        acc_add(1, z, idc, u);
        layer = zsm[z * 3 + 2];
      } else {
        acc_add((pmz == 2) ? 1 : 0, z, idc, u);
        layer = (pmz == 2) ? zsm[z * 3 + 2] : zsm[z * 3 + 1];
      }
    });
    flush(layer);
  };
  // (A p)_k: f(z, k, Ap, p_k)
  auto sweep_stencil = [&](auto&& f) {
    const double* pz = pv + y * nx + x;               // node (x, y) of plane z
    const double* kp = A.kappa + cbase + n2;          // cell (x-1, y-1) of cell plane z
    const int oxy[4] = {0, 1, (int)A.n, (int)A.n + 1};
    int poff[9];
#pragma unroll
    for (int dy = 0; dy < 3; dy++)
#pragma unroll
      for (int dx = 0; dx < 3; dx++) poff[dy * 3 + dx] = (dy - 1) * nx + (dx - 1);
    double v[3][3][3];   // [dz][dy][dx]
    double kc[2][2][2];  // [oz][oy][ox]
#pragma unroll
    for (int dy = 0; dy < 3; dy++)
#pragma unroll
      for (int dx = 0; dx < 3; dx++) {
        v[0][dy][dx] = 0.0;
        v[1][dy][dx] = ((pvm >> (dy * 3 + dx)) & 1u) ? pz[poff[dy * 3 + dx]] : 0.0;
      }
#pragma unroll
    for (int o = 0; o < 4; o++) {
      kc[0][o >> 1][o & 1] = 0.0;
      kc[1][o >> 1][o & 1] = (((cvm >> o) & 1u) && ncz > 0) ? __ldg(kp + oxy[o]) : 0.0;
    }
    int k = y * nx + x;
    for (int z = 0; z < nz; z++) {
      pz += nxy;
      kp += n2;
      const bool pn = z + 1 < nz, cn = z + 1 < ncz;
#pragma unroll
      for (int dy = 0; dy < 3; dy++)
#pragma unroll
        for (int dx = 0; dx < 3; dx++)
          v[2][dy][dx] = (((pvm >> (dy * 3 + dx)) & 1u) && pn) ? pz[poff[dy * 3 + dx]] : 0.0;
      double kn[4];
#pragma unroll
      for (int o = 0; o < 4; o++) kn[o] = (((cvm >> o) & 1u) && cn) ? __ldg(kp + oxy[o]) : 0.0;  // next cells
      double Ap = 0.0;
#pragma unroll
      for (int o = 0; o < 8; o++) {
        const int ox = o & 1, oy = (o >> 1) & 1, oz = o >> 2;
        const int a = (~o) & 7;
        auto pv_b = [&](int b) {  // p at corner b of cell octant o
          return v[oz + ((b >> 2) & 1)][oy + ((b >> 1) & 1)][ox + (b & 1)];
        };
        Ap += kc[oz][oy][ox] * (4.0 * pv_b(a) - pv_b(a ^ 3) - pv_b(a ^ 5) - pv_b(a ^ 6) - pv_b(a ^ 7));
      }
      f(z, k, Ap * kh, v[1][1][1]);
      k += nxy;
#pragma unroll
      for (int dy = 0; dy < 3; dy++)
#pragma unroll
        for (int dx = 0; dx < 3; dx++) {
          v[0][dy][dx] = v[1][dy][dx];
          v[1][dy][dx] = v[2][dy][dx];
        }
#pragma unroll
      for (int o = 0; o < 4; o++) {
        kc[0][o >> 1][o & 1] = kc[1][o >> 1][o & 1];
        kc[1][o >> 1][o & 1] = kn[o];
      }
    }
  };

  auto slot_put = [&](int which, double v) {
    v = wsum0(v);
    if (lane == 0) slots[which * 32 + warp] = v;
  };
  auto slot_fin = [&](int which) { return wsum0((lane < NW) ? slots[which * 32 + lane] : 0.0); };
  auto reduce_c = [&](const double* sub) {  // csh = [sub -] sum of the task rows (one warp per row)
    for (int i = warp; i < nc; i += NW) {
      double s = 0.0;
      for (int tt = lane; tt < NT; tt += 32) s += bins[tt * NQ + i];
      s = wsum0(s);
      if (lane == 0) csh[i] = sub ? sub[((int64_t)mp * nc + i) * A.n_rhs + rhs] - s : s;
    }
  };
  auto solve_y = [&]() {
    double cyw = 0.0;
    for (int i = warp; i < nc; i += NW) {
      double s = 0.0;
      for (int j = lane; j < nc; j += 32) s += __ldg(Si + (int64_t)i * nc + j) * csh[j];
      s = wsum0(s);
      if (lane == 0) Ysh[i] = s;
      cyw += s * csh[i];
    }
    if (lane == 0) slots[3 * 32 + warp] = cyw;
  };

  // two-level preconditioner (level 1): M^-1 = D^-1 + Z E^-1 Z^T, M-metric projection
  const bool crs = (MODE == 0) && A.coarse && A.ncomp[mp] > 0;
  const int nca = crs ? A.ncomp[mp] : 0;
  const int* cmp = A.cmap + P.node_off;
  const int* cpt = A.cptr + (int64_t)mp * (A.ncmax + 1);
  const int* cls = A.clist + P.node_off;
  const double* Eiv = A.Einv + (int64_t)mp * A.ncmax;
  const double* CZm = A.CZ + (int64_t)mp * nc * A.ncmax;
  // zr = E^-1 Z^T R (4-lane groups over each component's node list), slot 4 = (Z^T r)^T E^-1 Z^T r,
  // then csh += (CZ) zr.  Two barriers.
  auto coarse_c = [&]() {
    double part = 0.0;
    const int sub = lane & 3, ngrp = blockDim.x >> 2;
    for (int a0 = threadIdx.x >> 2; a0 - (int)(threadIdx.x >> 2) < nca; a0 += ngrp) {
      const int a = a0;
      double sv = 0.0;
      if (a < nca) {
        const int i0 = __ldg(cpt + a), i1 = __ldg(cpt + a + 1);
        for (int i = i0 + sub; i < i1; i += 4) sv += __ldcg(Rv + __ldg(cls + i));
      }
      sv += __shfl_xor_sync(FULLMASK, sv, 1);
      sv += __shfl_xor_sync(FULLMASK, sv, 2);
      if (a < nca && sub == 0) {
        const double ei = __ldg(Eiv + a);
        zr[a] = sv * ei;
        part += sv * sv * ei;
      }
    }
    part = wsum0(part);
    if (lane == 0) slots[4 * 32 + warp] = part;
    __syncthreads();
    for (int t = warp; t < nc; t += NW) {
      double sv = 0.0;
      for (int a = lane; a < nca; a += 32) sv += __ldg(CZm + (int64_t)t * A.ncmax + a) * zr[a];
      sv = wsum0(sv);
      if (lane == 0) csh[t] += sv;
    }
    __syncthreads();
  };
  // vv = s0 zr - E^-1 (CZ)^T Ysh.  One barrier.
  auto coarse_v = [&](double s0) {
    for (int a = threadIdx.x; a < nca; a += blockDim.x) {
      double acc = 0.0;
      for (int t = 0; t < nc; t++) acc += __ldg(CZm + (int64_t)t * A.ncmax + a) * Ysh[t];
      vv[a] = (s0 != 0.0 ? s0 * zr[a] : 0.0) - __ldg(Eiv + a) * acc;
    }
    __syncthreads();
  };
  auto cz_at = [&](int k) -> double {
    if (!crs) return 0.0;
    const int a = __ldg(cmp + k);
    return (a >= 0) ? vv[a] : 0.0;
  };

  if (MODE == 1) {
    double* Yv = A.FY + P.fine_off + (int64_t)rhs * nn;
    tasks([&] {
      if (wact) sweep_stencil([&](int, int k, double Ap, double) { if (lact) Yv[k] = Ap; });
    });
    tasks([&] {
      if (wact) sweep_c([&](int, int k) -> double { return lact ? pv[k] : 0.0; });
    });
    __syncthreads();
    reduce_c(nullptr);
    __syncthreads();
    for (int i = threadIdx.x; i < nc; i += blockDim.x) {
      const int64_t gi = ((int64_t)mp * nc + i) * A.n_rhs + rhs;
      A.g[gi] = A.g0[gi] - csh[i];
    }
    return;
  }
  // init: x0 = D^-1 C^T S^-1 g0, r0 = A x0, c = C D^-1 r0, yhat = S^-1 c
  for (int i = threadIdx.x; i < nc; i += blockDim.x) csh[i] = A.g0[((int64_t)mp * nc + i) * A.n_rhs + rhs];
  __syncthreads();
  solve_y();
  __syncthreads();
  if (crs) coarse_v(0.0);
  tasks([&] {
    if (!wact) return;
    walk_ids([&](int z, int k, const int (&idc)[8]) {
      if (!lact) return;
      const double x0 = dg[k] * ct_of(z, idc) - cz_at(k);
      pv[k] = x0;
      Xv[k] = x0;
    });
  });
  __syncthreads();
  tasks([&] {
    if (wact) sweep_stencil([&](int, int k, double Ap, double) { if (lact) Rv[k] = Ap; });
  });
  double rr0 = 0.0;
  tasks([&] {
    if (wact)
      sweep_c([&](int, int k) -> double {
        if (!lact) return 0.0;
        const double rk = Rv[k];
        const double u = dg[k] * rk;
        rr0 += rk * u;
        return u;
      });
  });
  slot_put(2, rr0);
  __syncthreads();
  reduce_c(nullptr);
  __syncthreads();
  if (crs) coarse_c();
  solve_y();
  __syncthreads();
  rr0 = slot_fin(2) + (crs ? slot_fin(4) : 0.0);
  if (crs) coarse_v(1.0);

  const double tol2 = A.rtol * A.rtol;
  const double floor2 = 1e-30 * rr0;
  double beta = 0.0, rz = 0.0, ref = 0.0, alpha = 0.0;
  int it = 0, breakdown = 0;
  for (;; it++) {
    double v = 0.0;
    const bool first = (it == 0);
    tasks([&] {
      if (!wact) return;
      walk_ids([&](int z, int k, const int (&idc)[8]) {
        if (!lact) return;
        const double rk = Rv[k] - ct_of(z, idc);
        const double zz = dg[k] * rk + cz_at(k);
        const double pold = pv[k];
        if (!first) Xv[k] += alpha * pold;
        pv[k] = first ? -zz : -zz + beta * pold;
        Rv[k] = rk;
        v += rk * zz;
      });
    });
    slot_put(0, v);
    __syncthreads();  // B1
    double w = 0.0;
    tasks([&] {
      if (wact)
        sweep_stencil([&](int, int k, double Ap, double pk) {
          if (lact) {
            Qv[k] = Ap;
            w += pk * Ap;
          }
        });
    });
    slot_put(1, w);
    __syncthreads();  // B2
    rz = slot_fin(0);
    const double pq = slot_fin(1);
    if (it == 0) ref = rz;
    if (!(rz > fmax(tol2 * ref, floor2)) || it >= A.max_iter) break;
    if (!(pq > 0.0) || !isfinite(pq)) {
      breakdown = 1;
      break;
    }
    alpha = rz / pq;
    double rr = 0.0;
    tasks([&] {
      if (wact)
        sweep_c([&](int, int k) -> double {
          if (!lact) return 0.0;
          const double rk = Rv[k] + alpha * Qv[k];
          Rv[k] = rk;
          const double u = dg[k] * rk;
          rr += rk * u;
          return u;
        });
    });
    slot_put(2, rr);
    __syncthreads();  // B3
    reduce_c(nullptr);
    __syncthreads();
    if (crs) coarse_c();
    solve_y();
    __syncthreads();  // B4
    beta = (slot_fin(2) + (crs ? slot_fin(4) : 0.0) - slot_fin(3)) / rz;
    if (crs) coarse_v(1.0);
  }

  // feasibility restoration: x += D^-1 C^T S^-1 (g - C x); parents also into the pool
  tasks([&] {
    if (wact) sweep_c([&](int, int k) -> double { return lact ? Xv[k] : 0.0; });
  });
  __syncthreads();
  reduce_c(A.g0);
  __syncthreads();
  solve_y();
  __syncthreads();
  if (crs) coarse_v(0.0);
  double* po = (P.pool_off >= 0) ? A.pool + P.pool_off + (int64_t)rhs * nn : nullptr;
  tasks([&] {
    if (!wact) return;
    walk_ids([&](int z, int k, const int (&idc)[8]) {
      if (!lact) return;
      const double xf = Xv[k] + dg[k] * ct_of(z, idc) - cz_at(k);
      Xv[k] = xf;
      if (po) po[k] = xf;
    });
  });
  if (threadIdx.x == 0) {
    A.iters[prob] = it;
    A.relres[prob] = (ref > 0.0) ? sqrt(fmax(rz, 0.0) / ref) : 0.0;
    double* dgo = A.diag + (int64_t)prob * 4;
    dgo[0] = rz;
    dgo[1] = ref;
    dgo[2] = floor2;
    dgo[3] = breakdown;
  }
}

size_t pcg3d_l1_smem(int N) {
  return (size_t)(98 * 27 * N + 2 * 27 * N + 5 * 32 + 512) * sizeof(double) + 49 * 3 * sizeof(int);
}

// 14 warps (one CTA per SM) when the launch is at most a few waves, else 7 warps (two CTAs per SM:
// measured 12% faster on the 1000 problems of config 4, but 1.8x slower on the 216 of config 5)
cudaError_t launch_pcg3d_l1(const LevelArgs& A, cudaStream_t st) {
  const size_t smem = pcg3d_l1_smem(A.N);
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const int probs = A.nprob_mp * A.n_rhs;
  const bool wide = A.nprob_level * A.n_rhs >= 4 * sms;  // level-global: same kernel on every rank
  auto go = [&](auto k, int nw) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k<<<(unsigned)probs, nw * 32, smem, st>>>(A);
    return cudaGetLastError();
  };
  switch (A.N) {
    case 1: return wide ? go(k_pcg3d_l1<1, 7>, 7) : go(k_pcg3d_l1<1, 14>, 14);
    case 2: return wide ? go(k_pcg3d_l1<2, 7>, 7) : go(k_pcg3d_l1<2, 14>, 14);
    case 3: return wide ? go(k_pcg3d_l1<3, 7>, 7) : go(k_pcg3d_l1<3, 14>, 14);
    case 4: return wide ? go(k_pcg3d_l1<4, 7>, 7) : go(k_pcg3d_l1<4, 14>, 14);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_tapply3d(const LevelArgs& A, cudaStream_t st) {
  const size_t smem = pcg3d_l1_smem(A.N);
  const int probs = A.nprob_mp * A.n_rhs;
  auto go = [&](auto k) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k<<<(unsigned)probs, 7 * 32, smem, st>>>(A);
    return cudaGetLastError();
  };
  switch (A.N) {
    case 1: return go(k_pcg3d_l1<1, 7, 1>);
    case 2: return go(k_pcg3d_l1<2, 7, 1>);
    case 3: return go(k_pcg3d_l1<3, 7, 1>);
    case 4: return go(k_pcg3d_l1<4, 7, 1>);
  }
  return cudaErrorInvalidValue;
}

// ------------------------------------------------------------------------------------------
// Small 3D windows (<= 7 level nodes per side: config 5 level 4), block form of the same method:
// one CTA per macropoint carries all n_rhs = 4N right-hand sides together, one warp per
// right-hand side (north_star (c)).  The operator data the right-hand
// sides share — the 27-point stencil rows of A_n, the octant-merged constraint weights, D^-1 and
// the projector S^+ — are staged once in shared memory; each warp keeps its x, r, p, q in
// registers (lane owns nodes lane + 32 i) and its p (zero halo) in shared memory.  Every sum
// is a warp reduction in a fixed order and no block barrier is taken after the staging, so the
// right-hand sides iterate independently (each to its own convergence) and the results are
// bitwise reproducible.  Same iteration as k_pcg3d (init from the full problem's scale, pass A
// with the re-projection, q = A p, r update, c = C D^-1 r, yhat = S^+ c, restoration).
constexpr int kW7 = 7;                      // nodes per side
constexpr int kW7P = kW7 + 2;               // padded p pitch
constexpr int kW7NN = kW7 * kW7 * kW7;      // 343
constexpr int kW7KPL = (kW7NN + 31) / 32;   // nodes per lane (11)

template <int N, bool LOCK>
__global__ void __launch_bounds__(128 * N, 1) k_pcg3d_w7(LevelArgs A) {
  constexpr int NR = 4 * N;   // right-hand sides = warps
  constexpr int NQ = 27 * N;  // constraint rows
  constexpr int PP = kW7P * kW7P * kW7P;
  const int mp = blockIdx.x;
  const ProbDesc& P = A.probs[mp];
  const int nx = P.nc[0] + 1, ny = P.nc[1] + 1, nz = P.nc[2] + 1, nn = nx * ny * nz;
  const int lane = threadIdx.x & 31, rhs = threadIdx.x >> 5;

  constexpr int EC = 729 * N;  // constraint entries: sum_nodes prod_d (element sides of the node) <= 9^3, x N
  extern __shared__ __align__(16) double smem[];
  double* st_s = smem;                  // [27][nn] stencil rows
  double* rw_s = st_s + 27 * kW7NN;     // [EC] row-major constraint entries: weight
  double* nw_s = rw_s + EC;             // [EC] node-major constraint entries: weight
  double* dg_s = nw_s + EC;             // [nn] D^-1
  double* si_s = dg_s + kW7NN;          // [NQ][NQ] S^+ transposed: si_s[j*NQ + i] = S^+_ij
  double* p_all = si_s + ((NQ * NQ + 1) & ~1);  // [NR][PP] p with zero halo (also D^-1 r / x for C u);
                                        // 16-byte aligned (double2 accesses of the lockstep form)
  double* c_all = p_all + (NR + 2) * PP;  // [NR][NQ] (lockstep form: [NQ][NR + 2], p_all [PP][NR + 2])
  double* y_all = c_all + (NR + 2) * NQ;  // as c_all
  int* sd_s = reinterpret_cast<int*>(y_all + (NR + 2) * NQ);  // [3][7] sides packed pm | k0 << 4 | k1 << 8
  int* rg_s = sd_s + 3 * kW7;                             // [3][3] node range of subcell coordinate: lo | hi << 8
  int* rs_s = rg_s + 9;                                   // [NQ + 1] row starts
  int* ns_s = rs_s + NQ + 1;                              // [nn + 1] node starts
  int* ri_s = ns_s + kW7NN + 1;                           // [EC] padded p index of a row entry
  int* nr_s = ri_s + EC;                                  // [EC] constraint row of a node entry
  int* pm_s = nr_s + EC;                                  // [nn] node of slot s (slots sorted by entry count)

  {
    const double* S27 = A.STC + P.node_off * 27;
    const double* Si = A.Sinv + (int64_t)mp * NQ * NQ;
    for (int i = threadIdx.x; i < NQ * NQ; i += blockDim.x) {
      const int r = i / NQ, c = i - r * NQ;
      si_s[c * NQ + r] = __ldg(Si + i);
    }
    for (int i = threadIdx.x; i < (NR + 2) * PP; i += blockDim.x) p_all[i] = 0.0;  // zero halo (either layout)
    if (threadIdx.x < 3 * kW7) {
      const int d = threadIdx.x / kW7, X = threadIdx.x - d * kW7;
      const int ncd = P.nc[d];
      if (X <= ncd) {
        const Sides s = sides_of(A, P, d, X, ncd);
        sd_s[threadIdx.x] = s.pm | (s.k0 << 4) | (s.k1 << 8);
      } else {
        sd_s[threadIdx.x] = 0;
      }
    }
    __syncthreads();
    if (threadIdx.x < 9) {
      const int d = threadIdx.x / 3, q = threadIdx.x - d * 3;
      int lo = 99, hi = -1;
      for (int X = 0; X <= P.nc[d]; X++) {
        const int v = sd_s[d * kW7 + X], pm = v & 15, k0 = (v >> 4) & 15, k1 = (v >> 8) & 15;
        if (((pm & 1) && k0 == q) || ((pm & 2) && k1 == q)) {
          lo = min(lo, X);
          hi = max(hi, X);
        }
      }
      rg_s[threadIdx.x] = (hi >= lo) ? (lo | (hi << 8)) : (1 | (0 << 8));  // empty: lo > hi
    }
    __syncthreads();
    // constraint weights as sparse lists, both ways: per row (q, j) its (node, weight) entries for
    // c = C u, per node its (row, weight) entries for C^T yhat (octant-merged weights of k_node_ops3d)
    const double* MW = A.MLR + P.node_off * 8 * N;
    auto rng_n = [&](int r) { return max(0, (r >> 8) - (r & 255) + 1); };
    // entries per node (N x the subcells around it: 1 to 8); nodes are dealt to the lanes in slots
    // sorted by that count (s = lane + 32 i, node pm_s[s]), so the 32 lanes of a slot walk lists of
    // (nearly) equal length in C^T yhat: in node order a warp's 32 nodes mixed 2- to 16-entry lists
    // and every lane waited for the longest (the loop was over half of the kernel's instructions)
    int* cnt_s = nr_s;  // temporary, overwritten by the node entries below
    for (int k = threadIdx.x; k < nn; k += blockDim.x) {
      const int z = k / (nx * ny), t = k - z * nx * ny, y = t / nx, x = t - y * nx;
      const int px = __popc(sd_s[x] & 3), py = __popc(sd_s[kW7 + y] & 3), pz = __popc(sd_s[2 * kW7 + z] & 3);
      cnt_s[k] = px * py * pz;
    }
    if (threadIdx.x < NQ) {
      const int q = threadIdx.x / N, qz = q / 9, qy = (q / 3) % 3, qx = q % 3;
      rs_s[threadIdx.x + 1] = rng_n(rg_s[qx]) * rng_n(rg_s[3 + qy]) * rng_n(rg_s[6 + qz]);
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // stable counting sort by ballots, classes 1, 2, 4, 8 subcells
      int pos = 0;
      for (int cls = 1; cls <= 8; cls <<= 1)
        for (int k0 = 0; k0 < nn; k0 += 32) {
          const int k = k0 + lane;
          const bool hit = k < nn && cnt_s[k] == cls;
          const unsigned b = __ballot_sync(FULLMASK, hit);
          if (hit) pm_s[pos + __popc(b & ((1u << lane) - 1u))] = k;
          pos += __popc(b);
        }
    }
    __syncthreads();
    for (int sl = threadIdx.x; sl < nn; sl += blockDim.x) ns_s[sl + 1] = N * cnt_s[pm_s[sl]];
    // stencil rows and D^-1 in slot order (lane-contiguous reads in the solve)
    for (int i = threadIdx.x; i < 27 * nn; i += blockDim.x) {
      const int c = i / nn, sl = i - c * nn;
      st_s[i] = __ldg(S27 + c * nn + pm_s[sl]);
    }
    for (int sl = threadIdx.x; sl < nn; sl += blockDim.x) dg_s[sl] = __ldg(A.dinv + P.node_off + pm_s[sl]);
    __syncthreads();
    if (threadIdx.x == 0) {
      ns_s[0] = 0;
      for (int k = 0; k < nn; k++) ns_s[k + 1] += ns_s[k];
    } else if (threadIdx.x == 32) {
      rs_s[0] = 0;
      for (int r = 0; r < NQ; r++) rs_s[r + 1] += rs_s[r];
    }
    __syncthreads();
    if (ns_s[nn] > EC || rs_s[NQ] > EC) __trap();  // >= 2 level cells per subcell (reading R22) bounds both
    for (int sl = threadIdx.x; sl < nn; sl += blockDim.x) {
      const int k = pm_s[sl];
      const int z = k / (nx * ny), t = k - z * nx * ny, y = t / nx, x = t - y * nx;
      const int sx = sd_s[x], sy = sd_s[kW7 + y], sz = sd_s[2 * kW7 + z];
      int e = ns_s[sl];
      for (int zs = 0; zs < 2; zs++) {
        if (!((sz >> zs) & 1)) continue;
        const int kz = (sz >> (4 + 4 * zs)) & 15;
        for (int ys = 0; ys < 2; ys++) {
          if (!((sy >> ys) & 1)) continue;
          const int ky = (sy >> (4 + 4 * ys)) & 15;
          for (int xs = 0; xs < 2; xs++) {
            if (!((sx >> xs) & 1)) continue;
            const int kx = (sx >> (4 + 4 * xs)) & 15;
            const int o = xs + 2 * ys + 4 * zs;
            for (int j = 0; j < N; j++, e++) {
              nr_s[e] = ((kz * 3 + ky) * 3 + kx) * N + j;
              nw_s[e] = __ldg(MW + (int64_t)(o * N + j) * nn + k);
            }
          }
        }
      }
    }
    if (threadIdx.x < NQ) {
      const int row = threadIdx.x, q = row / N, j = row - q * N;
      const int qz = q / 9, qy = (q / 3) % 3, qx = q % 3;
      const int rx = rg_s[qx], ry = rg_s[3 + qy], rz = rg_s[6 + qz];
      int e = rs_s[row];
      for (int Z = rz & 255; Z <= (rz >> 8); Z++) {
        const int vz = sd_s[2 * kW7 + Z];
        const int bz = (((vz & 1) && ((vz >> 4) & 15) == qz) ? 0 : 1);
        for (int Y = ry & 255; Y <= (ry >> 8); Y++) {
          const int vy = sd_s[kW7 + Y];
          const int by = (((vy & 1) && ((vy >> 4) & 15) == qy) ? 0 : 1);
          for (int X = rx & 255; X <= (rx >> 8); X++, e++) {
            const int vx = sd_s[X];
            const int bx = (((vx & 1) && ((vx >> 4) & 15) == qx) ? 0 : 1);
            const int o = bx + 2 * by + 4 * bz;
            const int k = (Z * ny + Y) * nx + X;
            ri_s[e] = ((Z + 1) * kW7P + (Y + 1)) * kW7P + (X + 1);
            rw_s[e] = __ldg(MW + (int64_t)(o * N + j) * nn + k);
          }
        }
      }
    }
    __syncthreads();
  }
  if constexpr (LOCK) {
    // ---- lockstep form: the n_rhs = 4N right-hand sides iterate together.  A task is (node slot s,
    // half h of four right-hand sides); thread t owns tasks t + 128N i (i < 3), all of half t & 1, and
    // keeps x, r, p, q of its tasks' four right-hand sides in registers.  The vectors the operator
    // reads are interleaved by rhs in shared memory (p_all[padded node][NR], c_all / y_all[row][NR]),
    // so each stencil coefficient, constraint weight and S^+ entry is read once for four right-hand
    // sides (the warp-per-rhs form re-read them per rhs and was shared-memory bound).  Per-rhs
    // scalars come from fixed-order block reductions; a right-hand side that meets its stopping
    // test is frozen (x, r, p no longer updated) while the others continue, so every rhs takes
    // the same iterates as in the per-rhs form (up to the reduction order).
    constexpr int HV = NR / 4;        // halves
    constexpr int NRP = NR + 2;       // padded node / row stride of the interleaved vectors: 80 B for
                                      // NR = 8 spreads the scattered slots' 16-byte loads over the banks
                                      // (a 64 B stride put every other slot on the same 16 banks)
    constexpr int TPT = 3;            // HV * nn <= 3 * 128 N for nn <= 343
    const int tid = threadIdx.x, nt = blockDim.x, nwp = nt >> 5;
    const int h = (HV == 2) ? (tid & 1) : 0, r0 = 4 * h;
    __shared__ double redw[4 * N][2 * NR];
    __shared__ double tot_s[2 * NR];
    __shared__ double sc_alpha[NR], sc_beta[NR], sc_rz[NR], sc_ref[NR], sc_fl[NR], sc_rzref[NR];
    __shared__ int sc_act[NR], sc_it[NR], sc_bd[NR], sc_any;
    int tpx[TPT], tsl[TPT];  // padded p index (-1: no task) and slot of each task
#pragma unroll
    for (int i = 0; i < TPT; i++) {
      const int tau = tid + nt * i, sl = tau / HV;
      tsl[i] = sl;
      tpx[i] = -1;
      if (sl < nn) {
        const int k = pm_s[sl];
        const int z = k / (nx * ny), t = k - z * nx * ny, y = t / nx, x = t - y * nx;
        tpx[i] = ((z + 1) * kW7P + (y + 1)) * kW7P + (x + 1);
      }
    }
    auto ld4 = [](const double* a, double (&v)[4]) {
      const double2 u0 = *reinterpret_cast<const double2*>(a), u1 = *reinterpret_cast<const double2*>(a + 2);
      v[0] = u0.x; v[1] = u0.y; v[2] = u1.x; v[3] = u1.y;
    };
    auto st4 = [](double* a, const double (&v)[4]) {
      *reinterpret_cast<double2*>(a) = make_double2(v[0], v[1]);
      *reinterpret_cast<double2*>(a + 2) = make_double2(v[2], v[3]);
    };
    // block sums of two per-rhs quantities (this thread's four) into tot_s[0..NR), tot_s[NR..2NR)
    auto bsum2 = [&](const double (&a)[4], const double (&b)[4]) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 4; u++) { v[u] = a[u]; v[4 + u] = b[u]; }
#pragma unroll
      for (int o = 16; o >= HV; o >>= 1)
#pragma unroll
        for (int u = 0; u < 8; u++) v[u] += __shfl_xor_sync(FULLMASK, v[u], o);
      if ((tid & 31) < HV) {
#pragma unroll
        for (int u = 0; u < 4; u++) {
          redw[tid >> 5][r0 + u] = v[u];
          redw[tid >> 5][NR + r0 + u] = v[4 + u];
        }
      }
      __syncthreads();
      if (tid < 2 * NR) {
        double sacc = 0.0;
        for (int w = 0; w < nwp; w++) sacc += redw[w][tid];
        tot_s[tid] = sacc;
      }
      __syncthreads();
    };
    // (C^T yhat) of task i for its four right-hand sides
    auto ct4 = [&](int i, double (&ct)[4]) {
#pragma unroll
      for (int u = 0; u < 4; u++) ct[u] = 0.0;
      const int sl = tsl[i];
      for (int e = ns_s[sl], e1 = ns_s[sl + 1]; e < e1; e++) {
        const double w = nw_s[e];
        double yv[4];
        ld4(y_all + nr_s[e] * NRP + r0, yv);
#pragma unroll
        for (int u = 0; u < 4; u++) ct[u] += w * yv[u];
      }
    };
    // (A p) of task i from p_all
    auto apply4 = [&](int i, double (&a)[4]) {
#pragma unroll
      for (int u = 0; u < 4; u++) a[u] = 0.0;
      const int sl = tsl[i];
      const double* pb = p_all + tpx[i] * NRP + r0;
#pragma unroll
      for (int dz = -1; dz <= 1; dz++)
#pragma unroll
        for (int dy = -1; dy <= 1; dy++)
#pragma unroll
          for (int dx = -1; dx <= 1; dx++) {
            const int c = (dx + 1) + 3 * (dy + 1) + 9 * (dz + 1);
            const double cf = st_s[c * nn + sl];
            double pv[4];
            ld4(pb + ((dz * kW7P + dy) * kW7P + dx) * NRP, pv);
#pragma unroll
            for (int u = 0; u < 4; u++) a[u] += cf * pv[u];
          }
    };
    // c = C u (u in p_all): tasks (row, half, part) = tid < 2 NQ HV, each part half of the row's
    // entries, the two parts summed through the partner lane (tid ^ 1); ends with a barrier
    auto cmul4 = [&]() {
      if (tid < 2 * NQ * HV) {
        const int q = tid & 1, hh = (tid >> 1) % HV, row = (tid >> 1) / HV;
        const int e0 = rs_s[row], e1 = rs_s[row + 1], em = (e0 + e1) >> 1;
        double cv[4] = {0.0, 0.0, 0.0, 0.0};
        for (int e = q ? em : e0, ee = q ? e1 : em; e < ee; e++) {
          const double w = rw_s[e];
          double uv[4];
          ld4(p_all + ri_s[e] * NRP + 4 * hh, uv);
#pragma unroll
          for (int u = 0; u < 4; u++) cv[u] += w * uv[u];
        }
#pragma unroll
        for (int u = 0; u < 4; u++) cv[u] += __shfl_xor_sync(0xffffffffu >> (32 - min(32, 2 * NQ * HV - (tid & ~31))), cv[u], 1);
        if (q == 0) st4(c_all + row * NRP + 4 * hh, cv);
      }
      __syncthreads();
    };
    // y = S^+ c, tasks as cmul4 (parts: j < NQ/2, j >= NQ/2); ends with a barrier.  cy partials
    // (this thread's half, rows tid / HV) into cy[] after that barrier
    auto smul4 = [&](double (&cy)[4]) {
      if (tid < 2 * NQ * HV) {
        const int q = tid & 1, hh = (tid >> 1) % HV, row = (tid >> 1) / HV;
        double yv[4] = {0.0, 0.0, 0.0, 0.0};
        for (int j = q ? NQ / 2 : 0, je = q ? NQ : NQ / 2; j < je; j++) {
          const double sv = si_s[j * NQ + row];
          double cv[4];
          ld4(c_all + j * NRP + 4 * hh, cv);
#pragma unroll
          for (int u = 0; u < 4; u++) yv[u] += sv * cv[u];
        }
#pragma unroll
        for (int u = 0; u < 4; u++) yv[u] += __shfl_xor_sync(0xffffffffu >> (32 - min(32, 2 * NQ * HV - (tid & ~31))), yv[u], 1);
        if (q == 0) st4(y_all + row * NRP + 4 * hh, yv);
      }
      __syncthreads();
#pragma unroll
      for (int u = 0; u < 4; u++) cy[u] = 0.0;
      if (tid < NQ * HV) {
        const int row = tid / HV;
        double yv[4], cr[4];
        ld4(y_all + row * NRP + r0, yv);
        ld4(c_all + row * NRP + r0, cr);
#pragma unroll
        for (int u = 0; u < 4; u++) cy[u] = yv[u] * cr[u];
      }
    };

    double xr[TPT][4], rv[TPT][4], pr[TPT][4], qr[TPT][4];
#pragma unroll
    for (int i = 0; i < TPT; i++)
#pragma unroll
      for (int u = 0; u < 4; u++) xr[i][u] = rv[i][u] = pr[i][u] = qr[i][u] = 0.0;
    const double* bbase = A.B + P.vec_off;
    const double zero4[4] = {0.0, 0.0, 0.0, 0.0};
    // init: x0 = D^-1 C^T S^+ t, r0 = A x0 - b, c = C D^-1 r0, yhat = S^+ c; tot_s[0..NR) = r0^T D^-1 r0
    auto init = [&](const double* tcol, bool withb) {
      for (int idx = tid; idx < NQ * NR; idx += nt) {
        const int row = idx / NR, rr = idx - row * NR;
        c_all[row * NRP + rr] = tcol[((int64_t)mp * NQ + row) * A.n_rhs + rr];
      }
      __syncthreads();
      double cyd[4];
      smul4(cyd);
#pragma unroll
      for (int i = 0; i < TPT; i++)
        if (tpx[i] >= 0) {
          double ct[4];
          ct4(i, ct);
          const double dgv = dg_s[tsl[i]];
#pragma unroll
          for (int u = 0; u < 4; u++) xr[i][u] = dgv * ct[u];
          st4(p_all + tpx[i] * NRP + r0, xr[i]);
        }
      __syncthreads();
#pragma unroll
      for (int i = 0; i < TPT; i++)
        if (tpx[i] >= 0) {
          double ap[4];
          apply4(i, ap);
          const int k = pm_s[tsl[i]];
#pragma unroll
          for (int u = 0; u < 4; u++) rv[i][u] = ap[u] - (withb ? bbase[(int64_t)(r0 + u) * nn + k] : 0.0);
        }
      __syncthreads();
      double rr[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int i = 0; i < TPT; i++)
        if (tpx[i] >= 0) {
          const double dgv = dg_s[tsl[i]];
          double uv[4];
#pragma unroll
          for (int u = 0; u < 4; u++) {
            uv[u] = dgv * rv[i][u];
            rr[u] += rv[i][u] * uv[u];
          }
          st4(p_all + tpx[i] * NRP + r0, uv);
        }
      __syncthreads();
      cmul4();
      smul4(cyd);
      bsum2(rr, zero4);
    };

    init(A.g0, false);
    {
      double rz[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int i = 0; i < TPT; i++)
        if (tpx[i] >= 0) {
          double ct[4];
          ct4(i, ct);
          const double dgv = dg_s[tsl[i]];
#pragma unroll
          for (int u = 0; u < 4; u++) {
            const double w = rv[i][u] - ct[u];
            rz[u] += dgv * w * w;
          }
        }
      if (tid < NR) sc_fl[tid] = tot_s[tid];  // rr_ref (stash)
      __syncthreads();
      bsum2(rz, zero4);
      if (tid < NR) sc_rzref[tid] = tot_s[tid];
      __syncthreads();
    }
    init(A.g, true);
    const double tol2 = A.rtol * A.rtol;
    if (tid < NR) {
      sc_fl[tid] = 1e-30 * fmax(tot_s[tid], sc_fl[tid]);  // floor2 = 1e-30 max(rr0, rr_ref)
      sc_act[tid] = 1;
      sc_it[tid] = 0;
      sc_bd[tid] = 0;
      sc_alpha[tid] = 0.0;
      sc_beta[tid] = 0.0;
    }
    __syncthreads();
    for (int it = 0;; it++) {
      // pass A: x += alpha_prev p_prev (deferred), r <- r - C^T yhat, z = D^-1 r, p <- -z + beta p
      double v[4] = {0.0, 0.0, 0.0, 0.0};
      bool act[4];
      double al[4], be[4];
#pragma unroll
      for (int u = 0; u < 4; u++) {
        act[u] = sc_act[r0 + u] != 0;
        al[u] = sc_alpha[r0 + u];
        be[u] = sc_beta[r0 + u];
      }
#pragma unroll
      for (int i = 0; i < TPT; i++)
        if (tpx[i] >= 0) {
          double ct[4];
          ct4(i, ct);
          const double dgv = dg_s[tsl[i]];
#pragma unroll
          for (int u = 0; u < 4; u++) {
            if (!act[u]) continue;
            const double rk = rv[i][u] - ct[u];
            const double zz = dgv * rk;
            const double pold = pr[i][u];
            if (it > 0) xr[i][u] += al[u] * pold;
            pr[i][u] = (it == 0) ? -zz : -zz + be[u] * pold;
            rv[i][u] = rk;
            v[u] += rk * zz;
          }
          st4(p_all + tpx[i] * NRP + r0, pr[i]);
        }
      __syncthreads();
      // pass B: q = A p, pq
      double w[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int i = 0; i < TPT; i++)
        if (tpx[i] >= 0) {
          apply4(i, qr[i]);
#pragma unroll
          for (int u = 0; u < 4; u++) w[u] += pr[i][u] * qr[i][u];
        }
      bsum2(v, w);
      if (tid < NR && sc_act[tid]) {
        const double rz = tot_s[tid], pq = tot_s[NR + tid];
        if (it == 0) sc_ref[tid] = fmax(rz, sc_rzref[tid]);
        sc_rz[tid] = rz;
        if (!(rz > fmax(tol2 * sc_ref[tid], sc_fl[tid])) || it >= A.max_iter) {
          sc_act[tid] = 0;
          sc_it[tid] = it;
        } else if (!(pq > 0.0) || !isfinite(pq)) {
          sc_act[tid] = 0;
          sc_it[tid] = it;
          sc_bd[tid] = 1;
        } else {
          sc_alpha[tid] = rz / pq;
        }
      }
      __syncthreads();
      if (tid == 0) {
        int any = 0;
        for (int q = 0; q < NR; q++) any |= sc_act[q];
        sc_any = any;
      }
#pragma unroll
      for (int u = 0; u < 4; u++) {
        act[u] = sc_act[r0 + u] != 0;
        al[u] = sc_alpha[r0 + u];
      }
      __syncthreads();
      if (!sc_any) break;
      // pass C: r += alpha q, rr = r^T D^-1 r, u = D^-1 r -> p_all (p stays in registers)
      double rr[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int i = 0; i < TPT; i++)
        if (tpx[i] >= 0) {
          const double dgv = dg_s[tsl[i]];
          double uv[4];
#pragma unroll
          for (int u = 0; u < 4; u++) {
            if (act[u]) rv[i][u] += al[u] * qr[i][u];
            uv[u] = dgv * rv[i][u];
            rr[u] += rv[i][u] * uv[u];
          }
          st4(p_all + tpx[i] * NRP + r0, uv);
        }
      __syncthreads();
      cmul4();
      double cy[4];
      smul4(cy);
      bsum2(rr, cy);
      if (tid < NR && sc_act[tid]) sc_beta[tid] = (tot_s[tid] - tot_s[NR + tid]) / sc_rz[tid];
      __syncthreads();
    }
    // feasibility restoration: x += D^-1 C^T S^+ (g - C x)
#pragma unroll
    for (int i = 0; i < TPT; i++)
      if (tpx[i] >= 0) st4(p_all + tpx[i] * NRP + r0, xr[i]);
    __syncthreads();
    cmul4();
    for (int idx = tid; idx < NQ * NR; idx += nt) {
      const int row = idx / NR, rr = idx - row * NR;
      c_all[row * NRP + rr] = A.g[((int64_t)mp * NQ + row) * A.n_rhs + rr] - c_all[row * NRP + rr];
    }
    __syncthreads();
    double cyd[4];
    smul4(cyd);
    double* Xb = A.X + P.vec_off;
#pragma unroll
    for (int i = 0; i < TPT; i++)
      if (tpx[i] >= 0) {
        double ct[4];
        ct4(i, ct);
        const double dgv = dg_s[tsl[i]];
        const int k = pm_s[tsl[i]];
#pragma unroll
        for (int u = 0; u < 4; u++) Xb[(int64_t)(r0 + u) * nn + k] = xr[i][u] + dgv * ct[u];
      }
    if (tid < NR) {
      const int prob = mp * A.n_rhs + tid;
      A.iters[prob] = sc_it[tid];
      const double ref = sc_ref[tid], rz = sc_rz[tid];
      A.relres[prob] = (ref > 0.0) ? sqrt(fmax(rz, 0.0) / ref) : 0.0;
      double* dgo = A.diag + (int64_t)prob * 4;
      dgo[0] = rz;
      dgo[1] = ref;
      dgo[2] = sc_fl[tid];
      dgo[3] = sc_bd[tid];
    }
    return;
  }
  double* p_s = p_all + rhs * PP;
  double* c_s = c_all + rhs * NQ;
  double* y_s = y_all + rhs * NQ;

  // owned nodes: slot lane + 32 i, node pm_s[slot]
  int pix[kW7KPL];  // padded index of the node, -1 if absent
#pragma unroll
  for (int i = 0; i < kW7KPL; i++) {
    const int sl = lane + 32 * i;
    if (sl < nn) {
      const int k = pm_s[sl];
      const int z = k / (nx * ny), t = k - z * nx * ny, y = t / nx, x = t - y * nx;
      pix[i] = ((z + 1) * kW7P + (y + 1)) * kW7P + (x + 1);
    } else {
      pix[i] = -1;
    }
  }
  auto wsum = [](double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULLMASK, v, o);
    return v;
  };
  // (C^T yhat)_k from the node's constraint entries
  auto ct_at = [&](int i) -> double {
    const int k = lane + 32 * i;
    double ct = 0.0;
#pragma unroll 2
    for (int e = ns_s[k], e1 = ns_s[k + 1]; e < e1; e++) ct += nw_s[e] * y_s[nr_s[e]];
    return ct;
  };
  // c = C u with u in p_s (interior), rows over lanes, from the row entries; ends with __syncwarp
  auto cmul = [&]() {
    for (int row = lane; row < NQ; row += 32) {
      double sacc = 0.0;
      for (int e = rs_s[row], e1 = rs_s[row + 1]; e < e1; e++) sacc += rw_s[e] * p_s[ri_s[e]];
      c_s[row] = sacc;
    }
    __syncwarp();
  };
  // y = S^+ c (rows over lanes); returns c . y (all lanes); ends with __syncwarp
  auto smul = [&]() -> double {
    double cy = 0.0;
    for (int row = lane; row < NQ; row += 32) {
      double s = 0.0;
      for (int j = 0; j < NQ; j++) s += si_s[j * NQ + row] * c_s[j];
      y_s[row] = s;
      cy += s * c_s[row];
    }
    __syncwarp();
    return wsum(cy);
  };
  // q = A p at the owned nodes (p from p_s)
  auto apply = [&](int i) -> double {
    const int k = lane + 32 * i;
    const double* pb = p_s + pix[i];
    double a[3] = {0.0, 0.0, 0.0};  // one chain per plane dz (three independent FMA chains)
#pragma unroll
    for (int dz = -1; dz <= 1; dz++)
#pragma unroll
      for (int dy = -1; dy <= 1; dy++)
#pragma unroll
        for (int dx = -1; dx <= 1; dx++) {
          const int c = (dx + 1) + 3 * (dy + 1) + 9 * (dz + 1);
          a[dz + 1] += st_s[c * nn + k] * pb[(dz * kW7P + dy) * kW7P + dx];
        }
    return (a[0] + a[1]) + a[2];
  };

  double xr[kW7KPL], rr_[kW7KPL], pr[kW7KPL], qr[kW7KPL];
#pragma unroll
  for (int i = 0; i < kW7KPL; i++) xr[i] = rr_[i] = pr[i] = qr[i] = 0.0;
  const double* bvec = A.B + P.vec_off + (int64_t)rhs * nn;
  // init: x0 = D^-1 C^T S^+ t, r0 = A x0 - b, c = C D^-1 r0, yhat = S^+ c; returns r0^T D^-1 r0
  auto init = [&](const double* tcol, const double* bb) -> double {
    for (int i = lane; i < NQ; i += 32) c_s[i] = tcol[((int64_t)mp * NQ + i) * A.n_rhs + rhs];
    __syncwarp();
    smul();
#pragma unroll
    for (int i = 0; i < kW7KPL; i++)
      if (pix[i] >= 0) {
        const double x0 = dg_s[lane + 32 * i] * ct_at(i);
        xr[i] = x0;
        p_s[pix[i]] = x0;
      }
    __syncwarp();
    double rr = 0.0;
#pragma unroll
    for (int i = 0; i < kW7KPL; i++)
      if (pix[i] >= 0) rr_[i] = apply(i) - (bb ? bb[pm_s[lane + 32 * i]] : 0.0);
    __syncwarp();
#pragma unroll
    for (int i = 0; i < kW7KPL; i++)
      if (pix[i] >= 0) {
        const double u = dg_s[lane + 32 * i] * rr_[i];
        rr += rr_[i] * u;
        p_s[pix[i]] = u;
      }
    __syncwarp();
    cmul();
    smul();
    return wsum(rr);
  };

  const double rr_ref = init(A.g0, nullptr);
  double rz_ref = 0.0;
#pragma unroll
  for (int i = 0; i < kW7KPL; i++)
    if (pix[i] >= 0) {
      const double w = rr_[i] - ct_at(i);
      rz_ref += dg_s[lane + 32 * i] * w * w;
    }
  rz_ref = wsum(rz_ref);
  const double rr0 = init(A.g, bvec);

  const double tol2 = A.rtol * A.rtol;
  const double floor2 = 1e-30 * fmax(rr0, rr_ref);
  double beta = 0.0, rz = 0.0, ref = 0.0, alpha = 0.0;
  int it = 0, breakdown = 0;
  for (;; it++) {
    // pass A: x += alpha_prev p_prev (deferred), r <- r - C^T yhat, z = D^-1 r, p <- -z + beta p
    double v = 0.0;
    const bool first = (it == 0);
#pragma unroll
    for (int i = 0; i < kW7KPL; i++)
      if (pix[i] >= 0) {
        const double rk = rr_[i] - ct_at(i);
        const double zz = dg_s[lane + 32 * i] * rk;
        const double pold = pr[i];
        if (!first) xr[i] += alpha * pold;
        const double pn = first ? -zz : -zz + beta * pold;
        pr[i] = pn;
        p_s[pix[i]] = pn;
        rr_[i] = rk;
        v += rk * zz;
      }
    __syncwarp();
    // pass B: q = A p, pq
    double w = 0.0;
#pragma unroll
    for (int i = 0; i < kW7KPL; i++)
      if (pix[i] >= 0) {
        qr[i] = apply(i);
        w += pr[i] * qr[i];
      }
    rz = wsum(v);
    const double pq = wsum(w);
    if (it == 0) ref = fmax(rz, rz_ref);
    if (!(rz > fmax(tol2 * ref, floor2)) || it >= A.max_iter) break;
    if (!(pq > 0.0) || !isfinite(pq)) {
      breakdown = 1;
      break;
    }
    alpha = rz / pq;
    // pass C: r += alpha q, rr = r^T D^-1 r, u = D^-1 r -> p_s (p itself stays in registers)
    double rr = 0.0;
    __syncwarp();
#pragma unroll
    for (int i = 0; i < kW7KPL; i++)
      if (pix[i] >= 0) {
        const double rk = rr_[i] + alpha * qr[i];
        rr_[i] = rk;
        const double u = dg_s[lane + 32 * i] * rk;
        rr += rk * u;
        p_s[pix[i]] = u;
      }
    __syncwarp();
    cmul();
    const double cy = smul();
    beta = (wsum(rr) - cy) / rz;
  }

  // feasibility restoration: x += D^-1 C^T S^+ (g - C x)
  __syncwarp();
#pragma unroll
  for (int i = 0; i < kW7KPL; i++)
    if (pix[i] >= 0) p_s[pix[i]] = xr[i];
  __syncwarp();
  cmul();
  for (int i = lane; i < NQ; i += 32) c_s[i] = A.g[((int64_t)mp * NQ + i) * A.n_rhs + rhs] - c_s[i];
  __syncwarp();
  smul();
  double* Xv = A.X + P.vec_off + (int64_t)rhs * nn;
#pragma unroll
  for (int i = 0; i < kW7KPL; i++)
    if (pix[i] >= 0) Xv[pm_s[lane + 32 * i]] = xr[i] + dg_s[lane + 32 * i] * ct_at(i);
  if (lane == 0) {
    const int prob = mp * A.n_rhs + rhs;
    A.iters[prob] = it;
    A.relres[prob] = (ref > 0.0) ? sqrt(fmax(rz, 0.0) / ref) : 0.0;
    double* dgo = A.diag + (int64_t)prob * 4;
    dgo[0] = rz;
    dgo[1] = ref;
    dgo[2] = floor2;
    dgo[3] = breakdown;
  }
}

size_t pcg3d_w7_smem(int N) {
  const size_t NQ = 27 * (size_t)N, NR = 4 * (size_t)N;
  const size_t EC = 729 * (size_t)N;
  const size_t d = 27 * kW7NN + 2 * EC + kW7NN + ((NQ * NQ + 1) & ~(size_t)1) + (NR + 2) * kW7P * kW7P * kW7P + 2 * (NR + 2) * NQ;
  return d * sizeof(double) + (3 * kW7 + 9 + NQ + 1 + kW7NN + 1 + 2 * EC + kW7NN) * sizeof(int);
}

cudaError_t launch_pcg3d_w7(const LevelArgs& A, cudaStream_t st) {
  const size_t smem = pcg3d_w7_smem(A.N);
  // lockstep form by default; MCH_PCG3D_W7_WARP=1: one warp per rhs (A/B and path cross-check)
  const char* we = getenv("MCH_PCG3D_W7_WARP");
  const bool lock = !(we && atoi(we) != 0);
  auto go = [&](auto k, int N) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k<<<(unsigned)A.nprob_mp, 128 * N, smem, st>>>(A);
    return cudaGetLastError();
  };
  if (A.n_rhs != 4 * A.N) return cudaErrorInvalidValue;
  switch (A.N) {
    case 1: return lock ? go(k_pcg3d_w7<1, true>, 1) : go(k_pcg3d_w7<1, false>, 1);
    case 2: return lock ? go(k_pcg3d_w7<2, true>, 2) : go(k_pcg3d_w7<2, false>, 2);
  }
  return cudaErrorInvalidValue;
}



// ------------------------------------------------------------------------------------------
size_t pcg3d_smem(int N, int nxm) {
  const size_t d = (size_t)(nxm + 2) * (nxm + 2) * nxm + (size_t)nxm * 27 * N + 2 * 27 * N + 5 * 32 + 512;
  return d * sizeof(double) + (size_t)nxm * 3 * sizeof(int);
}

cudaError_t launch_node_ops3d(const LevelArgs& A, int max_nodes, cudaStream_t st) {
  dim3 grid((unsigned)((max_nodes + 127) / 128), (unsigned)A.nprob_mp);
  switch (A.N) {
    case 1: k_node_ops3d<1><<<grid, 128, 0, st>>>(A); break;
    case 2: k_node_ops3d<2><<<grid, 128, 0, st>>>(A); break;
    case 3: k_node_ops3d<3><<<grid, 128, 0, st>>>(A); break;
    case 4: k_node_ops3d<4><<<grid, 128, 0, st>>>(A); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

template <int N, int NXM, int RW, int MINB>
static cudaError_t launch3(const LevelArgs& A, cudaStream_t st) {
  auto k = k_pcg3d<N, NXM, RW, MINB>;
  const size_t smem = pcg3d_smem(N, NXM);
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  constexpr int LPR = (NXM > 16) ? 32 : ((NXM > 8) ? 16 : 8), RPW = 32 / LPR;
  constexpr int NW = (NXM + RPW * RW - 1) / (RPW * RW);
  k<<<(unsigned)A.nprob_mp * A.n_rhs, 32 * NW, smem, st>>>(A);
  return cudaGetLastError();
}

template <int N>
static cudaError_t launch3n(const LevelArgs& A, int nxm, cudaStream_t st) {
  switch (nxm) {
    case 7: return launch3<N, 7, 1, 8>(A, st);
    case 13: return launch3<N, 13, 1, MCH_P13_MINB>(A, st);
    case 25: return launch3<N, 25, 2, 1>(A, st);
  }
  return cudaErrorInvalidValue;
}

// smallest compiled window width >= nodes per side (0: none)
int pcg3d_nxm(int max_nodes_per_side) {
  if (max_nodes_per_side <= 7) return 7;
  if (max_nodes_per_side <= 13) return 13;
  if (max_nodes_per_side <= 25) return 25;
  return 0;
}

cudaError_t launch_pcg3d(const LevelArgs& A, int nxm, cudaStream_t st) {
  switch (A.N) {
    case 1: return launch3n<1>(A, nxm, st);
    case 2: return launch3n<2>(A, nxm, st);
    case 3: return launch3n<3>(A, nxm, st);
    case 4: return launch3n<4>(A, nxm, st);
  }
  return cudaErrorInvalidValue;
}
