// Hot-path kernels of hierarchical multicontinuum homogenization (sm_100a).
//
//  k_level_ops   exact Galerkin level-n element data from fine kappa/psi (PAPER.md:369-371,
//                reading R11): operator weights W and constraint weights m_{E,j,a}.
//  k_targets     c_mj and the targets of Eqs. (3)/(4).
//  k_transport   I_p = sum_t c_t phi_t(x_t + .) (Eq. 11, readings R9/R10),
//                b = -P^T A_1 I_p and g = g0 - C_1 I_p (Eqs. 12/13, R5).
//  k_proj_setup  Jacobi D^-1 and the projector's S^-1 = (C D^-1 C^T)^-1 per macropoint.
//  k_pcg         projected preconditioned CG per (macropoint, rhs) for
//                min 1/2 x^T A x - b^T x  s.t. C x = g  (Eqs. 3/4 at n = 1, 12/13 at n >= 2).
//  k_combine     phi_p = P_n xi + I_p at fine resolution (Eq. 11).
//  k_gram        G_p[a][b] = int_{K_p} kappa grad Phi_a . grad Phi_b (Eq. 7).
#include <cuda_runtime.h>
#include "device_common.cuh"
#include "kernels.h"

// ---------------------------------------------------------------------------------------
// level-n element data (levels >= 2), one thread per global level-n cell
__device__ __forceinline__ double int_pair(int t, double t0, double t1) {
  // int_{t0}^{t1} lhat_a lhat_b, lhat_0 = 1-t, lhat_1 = t; type t = a+b
  if (t == 0) return ((1 - t0) * (1 - t0) * (1 - t0) - (1 - t1) * (1 - t1) * (1 - t1)) / 3.0;
  if (t == 1) return (t1 * t1 / 2 - t1 * t1 * t1 / 3) - (t0 * t0 / 2 - t0 * t0 * t0 / 3);
  return (t1 * t1 * t1 - t0 * t0 * t0) / 3.0;
}

template <int D>
__global__ void k_level_ops(LevelArgs A) {
  const int64_t ncell = (D == 2) ? (int64_t)A.gn * A.gn : (int64_t)A.gn * A.gn * A.gn;
  const int64_t gc = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gc >= ncell) return;
  int cc[3] = {(int)(gc % A.gn), (int)((gc / A.gn) % A.gn), (D == 3) ? (int)(gc / ((int64_t)A.gn * A.gn)) : 0};
  const int s = A.s;
  const double Hc = A.h * s;
  double W[DimC<D>::NW];
  double Mc[4 * (1 << D)];
  for (int i = 0; i < DimC<D>::NW; i++) W[i] = 0.0;
  for (int i = 0; i < 4 * (1 << D); i++) Mc[i] = 0.0;
  const double hd = (D == 2) ? A.h * A.h : A.h * A.h * A.h;
  const double wscale = A.h * ((D == 2) ? 1.0 / Hc : 1.0);  // h Hc^(D-3)
  const int sz = (D == 3) ? s : 1;
  for (int iz = 0; iz < sz; iz++)
    for (int iy = 0; iy < s; iy++)
      for (int ix = 0; ix < s; ix++) {
        const int ii[3] = {ix, iy, iz};
        int64_t f = 0;
        for (int i = D - 1; i >= 0; i--) f = f * A.n + (cc[i] * s + ii[i]);
        const double kap = A.kappa[f];
        const int id = A.ids[f];
        double I[3][3];  // I[dim][type]
        double Lc[3][2]; // lhat at cell centre
        for (int i = 0; i < D; i++) {
          const double t0 = (double)ii[i] / s, t1 = (double)(ii[i] + 1) / s, tc = (ii[i] + 0.5) / s;
          for (int t = 0; t < 3; t++) I[i][t] = int_pair(t, t0, t1);
          Lc[i][0] = 1.0 - tc;
          Lc[i][1] = tc;
        }
        for (int k = 0; k < D; k++) {
          if (D == 2) {
            const int o = 1 - k;
            for (int t = 0; t < 3; t++) W[k * 3 + t] += kap * I[o][t];
          } else {
            const int o1 = (k == 0) ? 1 : 0, o2 = (k == 2) ? 1 : 2;
            for (int t2 = 0; t2 < 3; t2++)
              for (int t1 = 0; t1 < 3; t1++) W[k * 9 + t1 + 3 * t2] += kap * I[o1][t1] * I[o2][t2];
          }
        }
        for (int a = 0; a < (1 << D); a++) {
          double v = 1.0;
          for (int i = 0; i < D; i++) v *= Lc[i][(a >> i) & 1];
          Mc[id * (1 << D) + a] += v;
        }
      }
  double* wo = const_cast<double*>(A.W) + gc * DimC<D>::NW;
  for (int i = 0; i < DimC<D>::NW; i++) wo[i] = W[i] * wscale;
  double* mo = const_cast<double*>(A.Mc) + gc * (A.N << D);
  for (int i = 0; i < (A.N << D); i++) mo[i] = Mc[i] * hd;
}

// ---------------------------------------------------------------------------------------
// targets: one CTA per macropoint.  K_p first (the whole CTA: its centroids c_mj enter every
// subcell's targets), then one warp per subcell with warp reductions (r02 reduced every subcell
// over the CTA: two barriers and a serial thread-0 section per subcell)
template <int D>
__global__ void k_targets(LevelArgs A) {
  const int mp = blockIdx.x;
  const ProbDesc& P = A.probs[mp];
  __shared__ double scratch[32 * 16];
  __shared__ double tot[16];
  __shared__ double cm[3][4];
  const int N = A.N;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwp = blockDim.x >> 5;
  const double hd = (D == 2) ? A.h * A.h : A.h * A.h * A.h;
  // fine-cell box of subcell q
  auto box = [&](int q, int (&lo)[3], int (&ext)[3]) -> bool {
    bool present = true;
    int rem = q;
    for (int i = 0; i < 3; i++) { lo[i] = 0; ext[i] = 1; }
    for (int i = 0; i < D; i++) {
      const int slot = rem % A.w;
      rem /= A.w;
      const int v = P.k[i] - A.l + slot;
      int flo = v * A.c - A.coff, fhi = flo + A.c;
      flo = flo < 0 ? 0 : flo;
      fhi = fhi > A.n ? A.n : fhi;
      if (fhi <= flo) present = false;
      lo[i] = flo;
      ext[i] = fhi - flo;
    }
    return present;
  };
  // v[j*4] = count, v[j*4+1+m] = sum (f_m + 1/2) over the box's cells of continuum j (N <= 4 x 4
  // entries: per thread, cells t0, t0 + stride, ... of the box plane by plane, 32-bit index
  // arithmetic with the float-reciprocal division of fdiv, exact below 2^22)
  auto accum = [&](const int (&lo)[3], const int (&ext)[3], int t0, int stride, double (&v)[16]) {
    const int pc = ext[0] * ext[1];
    const float inv0 = 1.0f / (float)ext[0];
    for (int zz = 0; zz < ext[2]; zz++)
      for (int t = t0; t < pc; t += stride) {
        const int yy = fdiv(t, inv0);
        const int f[3] = {lo[0] + t - yy * ext[0], lo[1] + yy, lo[2] + zz};
        int64_t fi = 0;
        for (int i = D - 1; i >= 0; i--) fi = fi * A.n + f[i];
        const int id = A.ids[fi];
#pragma unroll
        for (int j = 0; j < 4; j++) {
          if (j == id) {
            v[j * 4] += 1.0;
#pragma unroll
            for (int m = 0; m < D; m++) v[j * 4 + 1 + m] += f[m] + 0.5;
          }
        }
      }
  };
  {  // K_p (subcell index of slot l in every dim): centroids c_mj
    int qc = 0;
    for (int i = D - 1; i >= 0; i--) qc = qc * A.w + A.l;
    int lo[3], ext[3];
    const bool present = box(qc, lo, ext);
    double v[16];
#pragma unroll
    for (int i = 0; i < 16; i++) v[i] = 0.0;
    if (present) accum(lo, ext, threadIdx.x, blockDim.x, v);
    if (N <= 2) {
      double v8[8];
#pragma unroll
      for (int i = 0; i < 8; i++) v8[i] = v[i];
      block_sum<8>(v8, scratch, tot);
    } else {
      block_sum<16>(v, scratch, tot);
    }
    const int ts = (N <= 2) ? 4 : 4;
    if (threadIdx.x == 0) {
      for (int j = 0; j < N; j++) {
        const double cnt = tot[j * ts];
        if (cnt == 0.0) atomicOr(&A.flags[mp], 1);
        for (int m = 0; m < D; m++) cm[m][j] = (cnt > 0) ? (tot[j * ts + 1 + m] * A.h) / cnt : 0.0;
      }
      for (int m = 0; m < D; m++)
        for (int j = 0; j < N; j++) A.cm[(mp * 3 + m) * 4 + j] = cm[m][j];
    }
    __syncthreads();
  }
  for (int q = wid; q < A.nsub; q += nwp) {
    int lo[3], ext[3];
    const bool present = box(q, lo, ext);
    double v[16];
#pragma unroll
    for (int i = 0; i < 16; i++) v[i] = 0.0;
    if (present) accum(lo, ext, lane, 32, v);
#pragma unroll
    for (int i = 0; i < 16; i++)
      if (i < 4 * N)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_xor_sync(FULLMASK, v[i], o);
#pragma unroll
    for (int j = 0; j < 4; j++) {  // lane j writes continuum j's rows
      if (j >= N || lane != j) continue;
      const int row = q * N + j;
      const double cnt = present ? v[j * 4] : 0.0;
      A.meas[(int64_t)mp * A.ncon + row] = cnt * hd;
      double* gr = A.g0 + ((int64_t)mp * A.ncon + row) * A.n_rhs;
      for (int a = 0; a < A.n_rhs; a++) gr[a] = 0.0;
      gr[j] = cnt * hd;
      for (int m = 0; m < D; m++)
        gr[N + j * D + m] = (cnt > 0) ? hd * (v[j * 4 + 1 + m] * A.h - cm[m][j] * cnt) : 0.0;
    }
  }
}

// ---------------------------------------------------------------------------------------
// transport (levels >= 2): one CTA per problem (macropoint, rhs)
template <int D>
__global__ void k_transport(LevelArgs A) {
  const int prob = blockIdx.x;
  const int mp = prob / A.n_rhs, r = prob % A.n_rhs;
  const ProbDesc& P = A.probs[mp];
  extern __shared__ double smem[];
  const Geo<D> gf = fine_geo<D>(P);
  const Geo<D> gl = level_geo<D>(A, P);
  double* I = A.FI + P.fine_off + (int64_t)r * gf.nnodes;
  double* Y = A.FY + P.fine_off + (int64_t)r * gf.nnodes;
  if (A.tphase != 2) {
  // phase 1: I_p at fine nodes (local-coordinate transport, reading R9)
  for (int k = threadIdx.x; k < gf.nnodes; k += blockDim.x) {
    int x[3];
    node_xyz<D>(gf, k, x);
    double s = 0.0;
    for (int t = 0; t < P.npar; t++) {
      int64_t idx = 0;
      for (int i = D - 1; i >= 0; i--) {
        const int xt = P.lo[i] + x[i] + (A.phys ? 0 : (P.par_k[t][i] - P.k[i]) * A.c) - P.par_lo[t][i];
        idx = idx * (P.par_ncf[t][i] + 1) + xt;
      }
      int64_t pn = 1;
      for (int i = 0; i < D; i++) pn *= (P.par_ncf[t][i] + 1);
      s += P.par_w[t] * A.pool[P.par_pool[t] + (int64_t)r * pn + idx];
    }
    I[k] = s;
  }
  if (A.tphase == 1) return;
  __syncthreads();
  // phase 2: Y = A_1 I (fine operator on the window, natural BC)
  for (int k = threadIdx.x; k < gf.nnodes; k += blockDim.x) Y[k] = apply_node<D>(A, P, gf, I, k);
  // C_1 I -> g = g0 - C_1 I
  int* eb = reinterpret_cast<int*>(smem);
  double* bins = smem + (A.nsub * 7 + 2 + 1) / 2;  // after the subcell-box int area (nsub*7+2 ints)
  double* cI = bins + (A.band > 0 ? 0 : 32 * A.ncon);
  __shared__ int ntask;
  subcell_boxes<D>(A, P, gf, eb, &ntask);
  if (A.band > 0) constraint_apply_owned<D>(A, P, gf, eb, [&](int k) { return I[k]; }, cI);
  else constraint_apply<D>(A, P, gf, eb, ntask, [&](int k) { return I[k]; }, bins, cI);
  for (int i = threadIdx.x; i < A.ncon; i += blockDim.x) {
    const int64_t gi = ((int64_t)mp * A.ncon + i) * A.n_rhs + r;
    A.g[gi] = A.g0[gi] - cI[i];
  }
  }  // tphase != 2
  __syncthreads();
  // phase 3: b = -P_n^T Y at level-n nodes.  P_n^T is the tensor product of the 1D restrictions
  // (weights 1 - |d|/s, |d| < s), applied dimension by dimension in place in Y: one thread per
  // fine row writes its restricted values over the row's head in increasing order (output X only
  // reads positions >= (X-1)s+1 >= X, so nothing is overwritten before it is read).
  const int s = A.s;
  const double inv_s = 1.0 / (double)s;
  const int nfx = gf.nn[0], nfy = gf.nn[1], nfz = gf.nn[2];
  const int nlx = gl.nn[0], nly = gl.nn[1], nlz = gl.nn[2];
  auto restrict1 = [&](double* v, int64_t stride, int nf, int nl, auto&& put) {
    for (int X = 0; X < nl; X++) {
      const int c0 = X * s;
      double acc = v[(int64_t)c0 * stride];
      for (int d = 1; d < s; d++) {
        const double w = 1.0 - d * inv_s;
        if (c0 - d >= 0) acc += w * v[(int64_t)(c0 - d) * stride];
        if (c0 + d < nf) acc += w * v[(int64_t)(c0 + d) * stride];
      }
      put(X, acc);
    }
  };
  __syncthreads();
  for (int row = threadIdx.x; row < nfy * nfz; row += blockDim.x) {
    double* v = Y + (int64_t)row * nfx;
    restrict1(v, 1, nfx, nlx, [&](int X, double a) { v[X] = a; });
  }
  __syncthreads();
  for (int col = threadIdx.x; col < nfz * nlx; col += blockDim.x) {
    const int fz = col / nlx, X = col - fz * nlx;
    double* v = Y + (int64_t)fz * nfy * nfx + X;
    restrict1(v, nfx, nfy, nly, [&](int Yc, double a) { v[(int64_t)Yc * nfx] = a; });
  }
  __syncthreads();
  double* bvec = A.B + P.vec_off + (int64_t)r * gl.nnodes;
  for (int col = threadIdx.x; col < nly * nlx; col += blockDim.x) {
    const int Yc = col / nlx, X = col - Yc * nlx;
    double* v = Y + (int64_t)Yc * nfx + X;
    restrict1(v, (int64_t)nfy * nfx, nfz, nlz, [&](int Z, double a) { bvec[((int64_t)Z * nly + Yc) * nlx + X] = -a; });
  }
}

// ---------------------------------------------------------------------------------------
// 2D transport of all right-hand sides of a macropoint in one CTA (levels >= 2, dense projector):
// the geometry of each fine node (parent indices, element kappa, element ids) is formed once and
// applied to the NR vectors, and the restriction passes run over (rhs, row) pairs.  Every value is
// summed in the order k_transport uses except the constraint sums, whose 32-element tasks are
// dealt to 8 warps instead of blockDim/32 (config 2 coefficients agree to 5e-13;
// MCH_TRANSPORT_GENERIC=1 selects k_transport; tools/env_ab.py).
template <int NR>
__global__ void __launch_bounds__(256) k_transport2d_mr(LevelArgs A) {
  const int mp = blockIdx.x;
  const ProbDesc& P = A.probs[mp];
  extern __shared__ double smem[];
  const Geo<2> gf = fine_geo<2>(P);
  const Geo<2> gl = level_geo<2>(A, P);
  const int nnf = gf.nnodes, nfx = gf.nn[0], nfy = gf.nn[1];
  double* I = A.FI + P.fine_off;  // rhs r at r * nnf
  double* Y = A.FY + P.fine_off;
  // phase 1: I_p at fine nodes (local-coordinate transport, reading R9)
  for (int k = threadIdx.x; k < nnf; k += blockDim.x) {
    int x[3];
    node_xyz<2>(gf, k, x);
    double sr[NR];
#pragma unroll
    for (int r = 0; r < NR; r++) sr[r] = 0.0;
    for (int t = 0; t < P.npar; t++) {
      int64_t idx = 0;
      for (int i = 1; i >= 0; i--) {
        const int xt = P.lo[i] + x[i] + (A.phys ? 0 : (P.par_k[t][i] - P.k[i]) * A.c) - P.par_lo[t][i];
        idx = idx * (P.par_ncf[t][i] + 1) + xt;
      }
      const int64_t pn = (int64_t)(P.par_ncf[t][0] + 1) * (P.par_ncf[t][1] + 1);
      const double* src = A.pool + P.par_pool[t] + idx;
      const double w = P.par_w[t];
#pragma unroll
      for (int r = 0; r < NR; r++) sr[r] += w * src[(int64_t)r * pn];
    }
#pragma unroll
    for (int r = 0; r < NR; r++) I[(int64_t)r * nnf + k] = sr[r];
  }
  __syncthreads();
  // phase 2: Y = A_1 I (fine operator on the window, natural BC), as apply_xyz
  for (int k = threadIdx.x; k < nnf; k += blockDim.x) {
    int xx[3];
    node_xyz<2>(gf, k, xx);
    bool okn[9];
#pragma unroll
    for (int c = 0; c < 9; c++) {
      const int dx = c % 3 - 1, dy = c / 3 - 1;
      okn[c] = (xx[0] + dx >= 0) && (xx[0] + dx < nfx) && (xx[1] + dy >= 0) && (xx[1] + dy < nfy);
    }
    double kap[4];
    bool oke[4];
#pragma unroll
    for (int o = 0; o < 4; o++) {
      int e[3] = {xx[0] - 1 + (o & 1), xx[1] - 1 + ((o >> 1) & 1), 0};
      oke[o] = e[0] >= 0 && e[0] < gf.nc[0] && e[1] >= 0 && e[1] < gf.nc[1];
      kap[o] = oke[o] ? A.kappa[fine_cell_index<2>(A, P, gf, e, nullptr)] : 0.0;
    }
#pragma unroll 1
    for (int r = 0; r < NR; r++) {
      const double* v = I + (int64_t)r * nnf;
      double nb[9];
#pragma unroll
      for (int c = 0; c < 9; c++) nb[c] = okn[c] ? v[k + (c % 3 - 1) + (c / 3 - 1) * nfx] : 0.0;
      double out = 0.0;
#pragma unroll
      for (int o = 0; o < 4; o++) {
        if (!oke[o]) continue;
        const int a = (~o) & 3;
        auto nbv = [&](int b) {
          const int dx = (b & 1) - (a & 1), dy = ((b >> 1) & 1) - ((a >> 1) & 1);
          return nb[(dx + 1) + 3 * (dy + 1)];
        };
        out += kap[o] * (1.0 / 6.0) * (4.0 * nbv(a) - nbv(a ^ 1) - nbv(a ^ 2) - 2.0 * nbv(a ^ 3));
      }
      Y[(int64_t)r * nnf + k] = out;
    }
  }
  // C_1 I -> g = g0 - C_1 I (as constraint_apply: 32-element tasks per subcell, warp sums, bins
  // per warp summed in warp order)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  const int nc = A.ncon, N = A.N;
  int* eb = reinterpret_cast<int*>(smem);
  double* bins = smem + (A.nsub * 7 + 2 + 1) / 2;  // [nw][ncon][NR]
  for (int i = threadIdx.x; i < nw * nc * NR; i += blockDim.x) bins[i] = 0.0;
  __shared__ int ntask;
  subcell_boxes<2>(A, P, gf, eb, &ntask);  // syncs
  const int* pref = eb + A.nsub * 6;
  const double hh = 0.25 * A.h * A.h;
  for (int t = wid; t < ntask; t += nw) {
    int q = 0;
    while (pref[q + 1] <= t) q++;
    const int* bx = eb + q * 6;
    const int idx = (t - pref[q]) * 32 + lane;
    const int cnt = bx[3] * bx[4] * bx[5];
    double sv[NR];
    int id = -1;
#pragma unroll
    for (int r = 0; r < NR; r++) sv[r] = 0.0;
    if (idx < cnt) {
      const int i1 = fdiv(idx, 1.0f / (float)bx[3]);
      int e[3] = {bx[0] + idx - i1 * bx[3], bx[1] + i1, 0};
      int kb[4];
#pragma unroll
      for (int b = 0; b < 4; b++) {
        int xb[3] = {e[0] + (b & 1), e[1] + ((b >> 1) & 1), 0};
        kb[b] = node_id<2>(gf, xb);
      }
      id = A.ids[fine_cell_index<2>(A, P, gf, e, nullptr)];
#pragma unroll
      for (int r = 0; r < NR; r++) {
        const double* v = I + (int64_t)r * nnf;
        double s = 0.0;
#pragma unroll
        for (int b = 0; b < 4; b++) s += v[kb[b]];
        sv[r] = s * hh;
      }
    }
    for (int j = 0; j < N; j++) {
#pragma unroll
      for (int r = 0; r < NR; r++) {
        double v = (j == id) ? sv[r] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(FULLMASK, v, o);
        if (lane == 0) bins[(wid * nc + q * N + j) * NR + r] += v;
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nc * NR; i += blockDim.x) {
    const int row = i / NR, r = i - row * NR;
    double s = 0.0;
    for (int w = 0; w < nw; w++) s += bins[(w * nc + row) * NR + r];
    const int64_t gi = ((int64_t)mp * nc + row) * A.n_rhs + r;
    A.g[gi] = A.g0[gi] - s;
  }
  __syncthreads();
  // phase 3: b = -P_n^T Y at level-n nodes, the separable in-place restriction of k_transport
  const int s = A.s;
  const double inv_s = 1.0 / (double)s;
  const int nlx = gl.nn[0], nly = gl.nn[1];
  auto restrict1 = [&](double* v, int64_t stride, int nf, int nl, auto&& put) {
    for (int X = 0; X < nl; X++) {
      const int c0 = X * s;
      double acc = v[(int64_t)c0 * stride];
      for (int d = 1; d < s; d++) {
        const double w = 1.0 - d * inv_s;
        if (c0 - d >= 0) acc += w * v[(int64_t)(c0 - d) * stride];
        if (c0 + d < nf) acc += w * v[(int64_t)(c0 + d) * stride];
      }
      put(X, acc);
    }
  };
  for (int u = threadIdx.x; u < NR * nfy; u += blockDim.x) {
    const int r = u / nfy, row = u - r * nfy;
    double* v = Y + (int64_t)r * nnf + (int64_t)row * nfx;
    restrict1(v, 1, nfx, nlx, [&](int X, double a) { v[X] = a; });
  }
  __syncthreads();
  for (int u = threadIdx.x; u < NR * nlx; u += blockDim.x) {
    const int r = u / nlx, X = u - r * nlx;
    double* v = Y + (int64_t)r * nnf + X;
    double* bvec = A.B + P.vec_off + (int64_t)r * gl.nnodes;
    // the z pass of k_transport is the identity in 2D (one plane): write -value directly
    restrict1(v, nfx, nfy, nly, [&](int Yc, double a) { bvec[(int64_t)Yc * nlx + X] = -a; });
  }
}

// 3D split transport, phases 1 (I_p) and 2 (b = -P_n^T Y) of k_transport for all right-hand
// sides of a macropoint in one CTA (up to kMaxR): parent indices formed once per fine node, the
// restriction passes over (rhs, line) pairs; per rhs the arithmetic is k_transport's.
constexpr int kMaxR = 12;
__global__ void __launch_bounds__(256) k_transport3d_mr(LevelArgs A) {
  const int mp = blockIdx.x;
  const ProbDesc& P = A.probs[mp];
  const Geo<3> gf = fine_geo<3>(P);
  const Geo<3> gl = level_geo<3>(A, P);
  const int nr = A.n_rhs;
  const int64_t nnf = gf.nnodes;
  double* I = A.FI + P.fine_off;
  double* Y = A.FY + P.fine_off;
  if (A.tphase == 1) {
    for (int k = threadIdx.x; k < gf.nnodes; k += blockDim.x) {
      int x[3];
      node_xyz<3>(gf, k, x);
      double sr[kMaxR];
#pragma unroll
      for (int r = 0; r < kMaxR; r++) sr[r] = 0.0;
      for (int t = 0; t < P.npar; t++) {
        int64_t idx = 0;
        for (int i = 2; i >= 0; i--) {
          const int xt = P.lo[i] + x[i] + (A.phys ? 0 : (P.par_k[t][i] - P.k[i]) * A.c) - P.par_lo[t][i];
          idx = idx * (P.par_ncf[t][i] + 1) + xt;
        }
        int64_t pn = 1;
        for (int i = 0; i < 3; i++) pn *= (P.par_ncf[t][i] + 1);
        const double* src = A.pool + P.par_pool[t] + idx;
        const double w = P.par_w[t];
#pragma unroll
        for (int r = 0; r < kMaxR; r++)
          if (r < nr) sr[r] += w * src[(int64_t)r * pn];
      }
#pragma unroll
      for (int r = 0; r < kMaxR; r++)
        if (r < nr) I[(int64_t)r * nnf + k] = sr[r];
    }
    return;
  }
  // phase 2: the separable in-place restriction of k_transport, per rhs
  const int s = A.s;
  const double inv_s = 1.0 / (double)s;
  const int nfx = gf.nn[0], nfy = gf.nn[1], nfz = gf.nn[2];
  const int nlx = gl.nn[0], nly = gl.nn[1], nlz = gl.nn[2];
  auto restrict1 = [&](double* v, int64_t stride, int nf, int nl, auto&& put) {
    for (int X = 0; X < nl; X++) {
      const int c0 = X * s;
      double acc = v[(int64_t)c0 * stride];
      for (int d = 1; d < s; d++) {
        const double w = 1.0 - d * inv_s;
        if (c0 - d >= 0) acc += w * v[(int64_t)(c0 - d) * stride];
        if (c0 + d < nf) acc += w * v[(int64_t)(c0 + d) * stride];
      }
      put(X, acc);
    }
  };
  const int rows = nfy * nfz;
  for (int u = threadIdx.x; u < nr * rows; u += blockDim.x) {
    const int r = u / rows, row = u - r * rows;
    double* v = Y + (int64_t)r * nnf + (int64_t)row * nfx;
    restrict1(v, 1, nfx, nlx, [&](int X, double a) { v[X] = a; });
  }
  __syncthreads();
  const int cols = nfz * nlx;
  for (int u = threadIdx.x; u < nr * cols; u += blockDim.x) {
    const int r = u / cols, col = u - r * cols;
    const int fz = col / nlx, X = col - fz * nlx;
    double* v = Y + (int64_t)r * nnf + (int64_t)fz * nfy * nfx + X;
    restrict1(v, nfx, nfy, nly, [&](int Yc, double a) { v[(int64_t)Yc * nfx] = a; });
  }
  __syncthreads();
  const int lines = nly * nlx;
  for (int u = threadIdx.x; u < nr * lines; u += blockDim.x) {
    const int r = u / lines, col = u - r * lines;
    const int Yc = col / nlx, X = col - Yc * nlx;
    double* v = Y + (int64_t)r * nnf + (int64_t)Yc * nfx + X;
    double* bvec = A.B + P.vec_off + (int64_t)r * gl.nnodes;
    restrict1(v, (int64_t)nfy * nfx, nfz, nlz, [&](int Z, double a) { bvec[((int64_t)Z * nly + Yc) * nlx + X] = -a; });
  }
}

// ---------------------------------------------------------------------------------------
// projector setup: one CTA per macropoint
template <int D>
__global__ void k_proj_setup(LevelArgs A) {
  const int mp = blockIdx.x;
  const ProbDesc& P = A.probs[mp];
  const Geo<D> g = level_geo<D>(A, P);
  extern __shared__ double smem[];
  const int nc = A.ncon;
  double* S = smem;                 // nc*nc
  double* scratch = S + nc * nc;    // 32*16
  double* tot = scratch + 32 * 16;  // 16
  int* eb = reinterpret_cast<int*>(tot + 16);
  double* eb_end = tot + 16 + (A.nsub * 7 + 2 + 1) / 2 + 1;  // V (nc*nc) after the int area
  double* dinv = A.dinv + P.node_off;
  if (A.psplit == 2) {  // second half: S = C D^-1 C^T as the first half left it in Sinv
    const double* si = A.Sinv + (int64_t)mp * nc * nc;
    for (int i = threadIdx.x; i < nc * nc; i += blockDim.x) S[i] = si[i];
    __syncthreads();
  } else {
  // D^-1 rounded to fp32 in 2D: the on-chip PCG (pcg2d.cu) keeps it in fp32 shared memory, and S
  // below must be formed with the identical values for the projection to be exact
  for (int k = threadIdx.x; k < g.nnodes; k += blockDim.x) {
    const double dv = 1.0 / diag_node<D>(A, P, g, k);
    dinv[k] = (D == 2) ? (double)(float)dv : dv;
  }
  // nw[j][k] = sum over the elements around node k of m_{E,j,a} (used for subcell-interior nodes by
  // the generic k_pcg only: the specialised solvers form their own constraint weights)
  double* nwt = A.NWt + P.node_off * A.N;
  for (int k = threadIdx.x; A.need_nwt && k < g.nnodes; k += blockDim.x) {
    int x[3];
    node_xyz<D>(g, k, x);
    double w[4] = {0.0, 0.0, 0.0, 0.0};
    for (int ep = 0; ep < (1 << D); ep++) {
      int e[3] = {0, 0, 0};
      bool ok = true;
      for (int i = 0; i < D; i++) {
        e[i] = x[i] - 1 + ((ep >> i) & 1);
        ok = ok && e[i] >= 0 && e[i] < g.nc[i];
      }
      if (!ok) continue;
      const int a = (~ep) & ((1 << D) - 1);
      for (int j = 0; j < A.N; j++) w[j] += elem_m<D>(A, P, g, e, j, a);
    }
    for (int j = 0; j < A.N; j++) nwt[(int64_t)j * g.nnodes + k] = w[j];
  }
  for (int i = threadIdx.x; i < nc * nc; i += blockDim.x) S[i] = 0.0;
  __shared__ int ntask;
  subcell_boxes<D>(A, P, g, eb, &ntask);  // also syncs (dinv visible to block)
  const int N = A.N;
  // S = C D^-1 C^T over pairs of subcells that share nodes: one warp per pair (q1 <= q2), lanes over
  // the nodes of the two subcells' common node box, warp reduction in a fixed order.  No block
  // barrier per pair (r01/r02 reduced every pair over the CTA: two barriers each, ~190 pairs per
  // 3x3x3 window)
  {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwp = blockDim.x >> 5;
    const int nsub = A.nsub, npairs = nsub * (nsub + 1) / 2;
    for (int pi = wid; pi < npairs; pi += nwp) {
      int q1 = 0, rem = pi;
      while (rem >= nsub - q1) {
        rem -= nsub - q1;
        q1++;
      }
      const int q2 = q1 + rem;
      const int* b1 = eb + q1 * 6;
      const int* b2 = eb + q2 * 6;
      int lo[3], hi[3];
      bool empty = false;
      for (int i = 0; i < 3; i++) {
        if (i >= D) { lo[i] = 0; hi[i] = 0; continue; }
        if (b1[3 + i] == 0 || b2[3 + i] == 0) { empty = true; break; }
        lo[i] = max(b1[i], b2[i]);
        hi[i] = min(b1[i] + b1[3 + i], b2[i] + b2[3 + i]);  // node ranges are [lo, lo+ext] inclusive
        if (hi[i] < lo[i]) { empty = true; break; }
      }
      if (empty) continue;  // uniform across the warp
      const int ex = hi[0] - lo[0] + 1, ey = hi[1] - lo[1] + 1, ez = hi[2] - lo[2] + 1;
      const int cnt = ex * ey * ez;
      double v[16];
      for (int i = 0; i < 16; i++) v[i] = 0.0;
      for (int idx = lane; idx < cnt; idx += 32) {
        const int x[3] = {lo[0] + idx % ex, lo[1] + (idx / ex) % ey, lo[2] + idx / (ex * ey)};
        const int k = node_id<D>(g, x);
        double w1[4] = {0, 0, 0, 0}, w2[4] = {0, 0, 0, 0};
        for (int ep = 0; ep < (1 << D); ep++) {
          int e[3] = {0, 0, 0};
          bool ok = true;
          for (int i = 0; i < D; i++) {
            e[i] = x[i] - 1 + ((ep >> i) & 1);
            ok = ok && e[i] >= 0 && e[i] < g.nc[i];
          }
          if (!ok) continue;
          const int q = elem_subcell<D>(A, P, g, e);
          if (q != q1 && q != q2) continue;
          const int a = (~ep) & ((1 << D) - 1);
          for (int j = 0; j < N; j++) {
            const double m = elem_m<D>(A, P, g, e, j, a);
            if (q == q1) w1[j] += m;
            if (q == q2) w2[j] += m;
          }
        }
        const double di = dinv[k];
        for (int j1 = 0; j1 < N; j1++)
          for (int j2 = 0; j2 < N; j2++) v[j1 * 4 + j2] += w1[j1] * w2[j2] * di;
      }
      for (int j1 = 0; j1 < N; j1++)
        for (int j2 = 0; j2 < N; j2++) {
          double t = v[j1 * 4 + j2];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(FULLMASK, t, o);
          if (lane == 0) {
            const int r1 = q1 * N + j1, r2 = q2 * N + j2;
            S[r1 * nc + r2] = t;
            S[r2 * nc + r1] = t;
          }
        }
    }
    __syncthreads();
  }
  if (A.psplit == 1) {  // first half (beside k_coarse_setup): hand S over in Sinv
    double* so = A.Sinv + (int64_t)mp * nc * nc;
    for (int i = threadIdx.x; i < nc * nc; i += blockDim.x) so[i] = S[i];
    return;
  }
  }  // psplit != 2
  // two-level preconditioner: S_M = C M^-1 C^T = C D^-1 C^T + (CZ) E^-1 (CZ)^T
  if (A.coarse) {
    const int nca = A.ncomp[mp];
    const double* CZ = A.CZ + (int64_t)mp * nc * A.ncmax;
    const double* Ei = A.Einv + (int64_t)mp * A.ncmax;
    // staged in shared memory (after V's area) so the nc^2 dot products read no L2
    double* czs = eb_end + nc * nc;  // [nc][nca]
    double* eis = czs + nc * nca;    // [nca]
    for (int idx = threadIdx.x; idx < nc * nca; idx += blockDim.x) {
      const int i = idx / nca, a = idx - i * nca;
      czs[idx] = CZ[(int64_t)i * A.ncmax + a];
    }
    for (int a = threadIdx.x; a < nca; a += blockDim.x) eis[a] = Ei[a];
    __syncthreads();
    for (int idx = threadIdx.x; idx < nc * nc; idx += blockDim.x) {
      const int i = idx / nc, j = idx % nc;
      double acc = 0.0;
      for (int a = 0; a < nca; a++) acc += czs[i * nca + a] * eis[a] * czs[j * nca + a];
      S[idx] += acc;
    }
    __syncthreads();
  }
  // equilibrate, mark inactive rows, Gauss-Jordan inverse (SPD, no pivoting)
  __shared__ double ds[128];
  const double* meas = A.meas + (int64_t)mp * nc;
  for (int i = threadIdx.x; i < nc; i += blockDim.x) {
    const bool act = meas[i] > 0.0 && S[i * nc + i] > 0.0;
    ds[i] = act ? 1.0 / sqrt(S[i * nc + i]) : 0.0;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < nc * nc; idx += blockDim.x) {
    const int i = idx / nc, j = idx % nc;
    if (ds[i] == 0.0 || ds[j] == 0.0)
      S[idx] = (i == j) ? 1.0 : 0.0;
    else
      S[idx] = S[idx] * ds[i] * ds[j];
  }
  __syncthreads();
  // backup S~ in V, then in-place Gauss-Jordan: S <- S~^-1, tracking the smallest pivot
  double* V = eb_end;
  for (int idx = threadIdx.x; idx < nc * nc; idx += blockDim.x) V[idx] = S[idx];
  __shared__ double minpiv;
  if (threadIdx.x == 0) minpiv = 1e300;
  __syncthreads();
  for (int p = 0; p < nc; p++) {
    const double piv = S[p * nc + p];
    const double ip = 1.0 / piv;  // one division per pivot (r01 divided per element)
    __syncthreads();
    if (threadIdx.x == 0) minpiv = fmin(minpiv, piv);
    // rank-1 update of the entries off row and column p (element (i, j) stepped without div/mod)
    {
      int i = threadIdx.x / nc, j = threadIdx.x - (threadIdx.x / nc) * nc;
      const int di = blockDim.x / nc, dj = blockDim.x - di * nc;
      for (int idx = threadIdx.x; idx < nc * nc; idx += blockDim.x) {
        if (i != p && j != p) S[idx] -= S[i * nc + p] * ip * S[p * nc + j];
        i += di;
        j += dj;
        if (j >= nc) {
          j -= nc;
          i++;
        }
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nc; i += blockDim.x) {
      if (i != p) {
        S[i * nc + p] = -S[i * nc + p] * ip;
        S[p * nc + i] = S[p * nc + i] * ip;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) S[p * nc + p] = ip;
    __syncthreads();
  }
  double* out = A.Sinv + (int64_t)mp * nc * nc;
  // a small pivot only flags possible dependence: k_pinv then decides by the eigenvalues with
  // exactly the oracle's criterion (lambda < 1e-11 lambda_max dropped, reading R20)
  if (minpiv > 1e-6) {
    for (int idx = threadIdx.x; idx < nc * nc; idx += blockDim.x) {
      const int i = idx / nc, j = idx % nc;
      out[idx] = S[idx] * ds[i] * ds[j];
    }
    return;
  }
  // Reading R20: dependent level-n constraint rows.  The pseudo-inverse of S~ is formed by
  // k_pinv (parallel Jacobi, one warp per window): hand over S~ and the row scales.
  if (threadIdx.x == 0) atomicOr(&A.flags[mp], 2);
  double* so = A.Sinv + (int64_t)mp * nc * nc;  // S~ in place of S^-1 until k_pinv replaces it
  for (int idx = threadIdx.x; idx < nc * nc; idx += blockDim.x) so[idx] = V[idx];
  for (int i = threadIdx.x; i < nc; i += blockDim.x) A.pinv_ds[(int64_t)mp * nc + i] = ds[i];
}

// ---------------------------------------------------------------------------------------
// Two-level preconditioner setup (level 1, generic k_pcg): one CTA per macropoint.
// High-contrast inclusions make the near-constant value of each inclusion the slowest mode of
// Jacobi-PCG.  If the window's contrast kappa_max / kappa_min >= 100, every node touching a cell
// with kappa > sqrt(kappa_min kappa_max) is "high"; the 3^D-connected components of high nodes
// are the coarse basis Z (indicators).  Two nodes of different components never share a cell,
// so E = Z^T A Z is diagonal.  Components are labelled by minimum-label propagation with
// pointer jumping (the result is the smallest node index of each component, independent of
// the order of updates) and numbered in node order.  Per component: bounding box, E_aa = z_a^T
// A z_a, and C z_a (constraint rows of the indicator).  Everything summed in a fixed order.
// exclusive prefix sum over the CTA of one int per thread (blockDim a multiple of 32): returns
// this thread's prefix; *tot = the sum, valid after the call (two barriers inside)
__device__ __forceinline__ int block_excl_scan(int v, int* wtot, int* tot) {
  const int ln = threadIdx.x & 31, wd = threadIdx.x >> 5, nwp = blockDim.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(FULLMASK, incl, o);
    if (ln >= o) incl += t;
  }
  if (ln == 31) wtot[wd] = incl;
  __syncthreads();
  if (wd == 0) {
    int w = (ln < nwp) ? wtot[ln] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(FULLMASK, w, o);
      if (ln >= o) w += t;
    }
    if (ln < nwp) wtot[ln] = w;
    if (ln == nwp - 1) *tot = w;
  }
  __syncthreads();
  return incl - v + (wd > 0 ? wtot[wd - 1] : 0);
}

#ifndef MCH_PINV_TOL
#define MCH_PINV_TOL 1e-34  // Jacobi stops when sum(offdiag^2) <= tol * sum(diag^2)
#endif
#ifndef MCH_COARSE_CONTRAST
#define MCH_COARSE_CONTRAST 20.0  // window contrast kappa_max / kappa_min that turns the coarse space on
#endif
#ifndef MCH_COMP_NODES
#define MCH_COMP_NODES 400
#endif
constexpr int kCompNodes = MCH_COMP_NODES;  // largest component kept in the coarse space

template <int D>
__global__ void k_coarse_setup(LevelArgs A) {
  const int mp = blockIdx.x;
  const ProbDesc& P = A.probs[mp];
  const Geo<D> g = level_geo<D>(A, P);
  int* cm = A.cmap + P.node_off;
  const int nn = g.nnodes, nc = A.ncon;
  __shared__ double red[64];
  __shared__ int flag, total;
  extern __shared__ double smem[];
  double* cvals = smem;                               // ncon
  int* cnt = reinterpret_cast<int*>(cvals + nc);       // blockDim.x
  // kappa of a level-n cell: the fine value (level 1) or the mean over its s^D fine cells
  auto kcell = [&](const int* e) -> double {
    if (g.fineop) return A.kappa[fine_cell_index<D>(A, P, g, e, nullptr)];
    double sum = 0.0;
    const int s = g.s;
    for (int iz = 0; iz < (D == 3 ? s : 1); iz++)
      for (int iy = 0; iy < s; iy++)
        for (int ix = 0; ix < s; ix++) {
          const int sub[3] = {ix, iy, iz};
          sum += A.kappa[fine_cell_index<D>(A, P, g, e, sub)];
        }
    return sum / (double)((D == 3) ? s * s * s : s * s);
  };
  // 1. contrast of the window
  double kmin = 1e300, kmax = 0.0;
  const int ncell = g.nc[0] * g.nc[1] * (D == 3 ? g.nc[2] : 1);
  for (int idx = threadIdx.x; idx < ncell; idx += blockDim.x) {
    int e[3] = {idx % g.nc[0], (idx / g.nc[0]) % g.nc[1], (D == 3) ? idx / (g.nc[0] * g.nc[1]) : 0};
    const double kv = kcell(e);
    kmin = fmin(kmin, kv);
    kmax = fmax(kmax, kv);
  }
  for (int o = 16; o > 0; o >>= 1) {
    kmin = fmin(kmin, __shfl_xor_sync(FULLMASK, kmin, o));
    kmax = fmax(kmax, __shfl_xor_sync(FULLMASK, kmax, o));
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (lane == 0) { red[wid] = kmin; red[32 + wid] = kmax; }
  __syncthreads();
  kmin = 1e300; kmax = 0.0;
  for (int w = 0; w < nw; w++) { kmin = fmin(kmin, red[w]); kmax = fmax(kmax, red[32 + w]); }
  const bool use = kmax >= MCH_COARSE_CONTRAST * kmin;
  const double thr = sqrt(kmin * kmax);
  const double thr1 = 0.5 * (kmin + kmax);  // pass 1: cells mostly made of the high phase
  __shared__ int csize[1024];
  __shared__ int cnew[1024];
  __shared__ int redo;
  __shared__ int wtot[32];
  int nall = 0;
  // Two passes at most.  Pass 0: high nodes = nodes touching a cell with kappa > thr.  On a coarse
  // level mesh the cell means widen every inclusion by up to a cell, so close inclusions fuse into
  // one component above kCompNodes, which the selection below would drop (config 5, level 2: the
  // four windows around the largest spheres then iterate on Jacobi alone, 220-286 iterations
  // instead of ~45).  Pass 1 (MCH_COARSE_ERODE=0 turns it off) relabels the nodes of such
  // components only: a node stays high when it touches a cell whose mean is above the midpoint
  // thr1, i.e. a cell mostly made of the high phase, which separates the fused inclusions again.
  // The kept nodes are a subset of one pass-0 component, and two of them sharing a cell are
  // neighbours, so nodes of different components still never share a cell and E stays diagonal.
  for (int pass = 0; pass < 2; pass++) {
  // 2. high nodes: label = own index
  for (int k = threadIdx.x; k < nn; k += blockDim.x) {
    int lab = -1;
    const int prev = (pass == 0) ? 0 : cm[k];  // pass 1: component id of pass 0 (or -1)
    const bool big = pass == 1 && prev >= 0 && prev < nall && csize[prev] > kCompNodes;
    if (pass == 1 && prev >= 0 && !big) lab = k;
    if (use && (pass == 0 || big)) {
      int x[3];
      node_xyz<D>(g, k, x);
      bool any = false, maj = false;
      for (int o = 0; o < (1 << D); o++) {
        int e[3] = {0, 0, 0};
        bool ok = true;
        for (int i = 0; i < D; i++) {
          e[i] = x[i] - 1 + ((o >> i) & 1);
          ok = ok && e[i] >= 0 && e[i] < g.nc[i];
        }
        if (ok) {
          const double kc = kcell(e);
          any = any || kc > thr;
          maj = maj || kc > thr1;
        }
      }
      if (pass == 0 ? any : maj) lab = k;
    }
    cm[k] = lab;
  }
  __syncthreads();
  // 3. minimum-label propagation over the 3^D neighbourhood, with pointer jumping
  if (use) {
    for (;;) {
      if (threadIdx.x == 0) flag = 0;
      __syncthreads();
      for (int k = threadIdx.x; k < nn; k += blockDim.x) {
        const int lk = cm[k];
        if (lk < 0) continue;
        int x[3];
        node_xyz<D>(g, k, x);
        int m = lk;
        for (int c = 0; c < DimC<D>::NB; c++) {
          const int dx = c % 3 - 1, dy = (c / 3) % 3 - 1, dz = (D == 3) ? c / 9 - 1 : 0;
          const int xx[3] = {x[0] + dx, x[1] + dy, x[2] + dz};
          bool ok = xx[0] >= 0 && xx[0] < g.nn[0] && xx[1] >= 0 && xx[1] < g.nn[1];
          if (D == 3) ok = ok && xx[2] >= 0 && xx[2] < g.nn[2];
          if (!ok) continue;
          const int ln = cm[node_id<D>(g, xx)];
          if (ln >= 0 && ln < m) m = ln;
        }
        if (m < lk) {
          atomicMin(&cm[k], m);
          flag = 1;
        }
      }
      __syncthreads();
      for (int k = threadIdx.x; k < nn; k += blockDim.x) {
        int lk = cm[k];
        if (lk < 0) continue;
        int r = cm[lk];
        while (r >= 0 && r < lk) { lk = r; r = cm[lk]; }
        atomicMin(&cm[k], lk);
      }
      __syncthreads();
      if (!flag) break;
      __syncthreads();
    }
  }
  // 4. number the roots (cm[k] == k) in node order: per-thread contiguous chunks + scan
  const int chunk = (nn + blockDim.x - 1) / blockDim.x;
  const int k0 = threadIdx.x * chunk, k1 = min(nn, k0 + chunk);
  int mine = 0;
  for (int k = k0; k < k1; k++) mine += (cm[k] == k);
  cnt[threadIdx.x] = block_excl_scan(mine, wtot, &total);
  __syncthreads();
  {
    int id = cnt[threadIdx.x];
    for (int k = k0; k < k1; k++)
      if (cm[k] == k) cm[k] = -(id++) - 2;  // roots: encoded id
  }
  __syncthreads();
  for (int k = threadIdx.x; k < nn; k += blockDim.x) {
    const int lk = cm[k];
    if (lk >= 0) cm[k] = -cm[lk] - 2;  // member: the root's id
  }
  __syncthreads();
  for (int k = threadIdx.x; k < nn; k += blockDim.x) {
    const int lk = cm[k];
    if (lk <= -2) cm[k] = -lk - 2;  // root: decode
  }
  __syncthreads();
  // keep components of at most kCompNodes nodes (long ones, e.g. channels across the window,
  // would make the per-component sums of every iteration a long serial chain), renumbered in
  // order; at most ncmax of them
  nall = min(total, 1024);
  if (threadIdx.x == 0) redo = 0;
  for (int a = threadIdx.x; a < nall; a += blockDim.x) csize[a] = 0;
  __syncthreads();
  for (int k = threadIdx.x; k < nn; k += blockDim.x)
    if (cm[k] >= 0 && cm[k] < nall) atomicAdd(&csize[cm[k]], 1);
  __syncthreads();
  if (pass == 0 && (A.coarse & 2) && total <= 1024)
    for (int a = threadIdx.x; a < nall; a += blockDim.x)
      if (csize[a] > kCompNodes) redo = 1;
  __syncthreads();
  if (!redo) break;
  }  // pass
  if (threadIdx.x == 0) {
    int next = 0;
    for (int a = 0; a < nall; a++) cnew[a] = (csize[a] <= kCompNodes && next < A.ncmax) ? next++ : -1;
    total = (total > 1024) ? 0 : next;
  }
  __syncthreads();
  const int ncomp = total;
  for (int k = threadIdx.x; k < nn; k += blockDim.x) {
    const int lk = cm[k];
    cm[k] = (lk >= 0 && lk < nall && ncomp > 0) ? cnew[lk] : -1;
  }
  if (threadIdx.x == 0) A.ncomp[mp] = ncomp;
  int* box = A.cbox + (int64_t)mp * A.ncmax * 6;
  for (int a = threadIdx.x; a < ncomp; a += blockDim.x) {
    box[a * 6 + 0] = box[a * 6 + 1] = box[a * 6 + 2] = 1 << 30;
    box[a * 6 + 3] = box[a * 6 + 4] = box[a * 6 + 5] = -1;
  }
  __syncthreads();
  if (ncomp == 0) return;
  // 5. bounding boxes
  for (int k = threadIdx.x; k < nn; k += blockDim.x) {
    const int a = cm[k];
    if (a < 0) continue;
    int x[3];
    node_xyz<D>(g, k, x);
    for (int i = 0; i < 3; i++) {
      atomicMin(&box[a * 6 + i], x[i]);
      atomicMax(&box[a * 6 + 3 + i], x[i]);
    }
  }
  __syncthreads();
  // 5b. node lists per component (CSR, node order): counts, prefix, fill (thread per component)
  int* cp = A.cptr + (int64_t)mp * (A.ncmax + 1);
  int* cl = A.clist + P.node_off;
  for (int a = threadIdx.x; a < ncomp; a += blockDim.x) {
    const int* bx = box + a * 6;
    int c = 0;
    for (int z = bx[2]; z <= bx[5]; z++)
      for (int y = bx[1]; y <= bx[4]; y++)
        for (int x = bx[0]; x <= bx[3]; x++) {
          const int xx[3] = {x, y, z};
          c += (cm[node_id<D>(g, xx)] == a);
        }
    cp[a + 1] = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    cp[0] = 0;
    for (int a = 0; a < ncomp; a++) cp[a + 1] += cp[a];
  }
  __syncthreads();
  for (int a = threadIdx.x; a < ncomp; a += blockDim.x) {
    const int* bx = box + a * 6;
    int o = cp[a];
    for (int z = bx[2]; z <= bx[5]; z++)
      for (int y = bx[1]; y <= bx[4]; y++)
        for (int x = bx[0]; x <= bx[3]; x++) {
          const int xx[3] = {x, y, z};
          const int k = node_id<D>(g, xx);
          if (cm[k] == a) cl[o++] = k;
        }
  }
  __syncthreads();
  // 6. per component: E_aa = z_a^T A z_a (fine Q1 element rows) and C z_a
  double* Ei = A.Einv + (int64_t)mp * A.ncmax;
  double* CZ = A.CZ + (int64_t)mp * nc * A.ncmax;
  __shared__ int ebs[125 * 7 + 2];
  __shared__ int ntask;
  subcell_boxes<D>(A, P, g, ebs, &ntask);
  // one warp per component (lanes over its bounding box, fixed-order warp sum): no block-wide
  // reduction per component
  const int lane_ = threadIdx.x & 31, nwarp_ = blockDim.x >> 5;
  for (int a = threadIdx.x >> 5; a < ncomp; a += nwarp_) {
    const int* bx = box + a * 6;
    const int ex = bx[3] - bx[0] + 1, ey = bx[4] - bx[1] + 1, ez = (D == 3) ? bx[5] - bx[2] + 1 : 1;
    double v[1] = {0.0};
    for (int idx = lane_; idx < ex * ey * ez; idx += 32) {
      const int x[3] = {bx[0] + idx % ex, bx[1] + (idx / ex) % ey, (D == 3) ? bx[2] + idx / (ex * ey) : 0};
      const int k = node_id<D>(g, x);
      if (cm[k] != a) continue;
      double az = 0.0;  // (A z_a)_k
      for (int o = 0; o < (1 << D); o++) {
        int e[3] = {0, 0, 0};
        bool ok = true;
        for (int i = 0; i < D; i++) {
          e[i] = x[i] - 1 + ((o >> i) & 1);
          ok = ok && e[i] >= 0 && e[i] < g.nc[i];
        }
        if (!ok) continue;
        const int ac = (~o) & ((1 << D) - 1);  // corner of node k in cell e
        double zc[1 << D];
        for (int b = 0; b < (1 << D); b++) {
          int xb[3] = {e[0] + (b & 1), e[1] + ((b >> 1) & 1), (D == 3) ? e[2] + ((b >> 2) & 1) : 0};
          zc[b] = (cm[node_id<D>(g, xb)] == a) ? 1.0 : 0.0;
        }
        double W[DimC<D>::NW];
        elem_W<D>(A, P, g, e, W);  // level 1: kappa times the Q1 weights; n >= 2: exact Galerkin
        az += elem_row<D>(W, zc, ac);
      }
      v[0] += az;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[0] += __shfl_down_sync(FULLMASK, v[0], o);
    if (lane_ == 0) Ei[a] = (v[0] > 0.0) ? 1.0 / v[0] : 0.0;
  }
  __syncthreads();
  // (A z_a) lists for the recurrence Z^T r_{k+1} = Z^T r~_k + alpha (A Z)^T p_k of the on-chip 2D
  // kernels: thread per component over its bounding box grown by one node, nonzeros in node
  // order; a window whose lists exceed kAzCap entries per node runs without the coarse space
  if (A.azp != nullptr && D == 2) {
    int* ap = A.azp + (int64_t)mp * (A.ncmax + 1);
    int* ai = A.azi + (int64_t)kAzCap * P.node_off;
    double* aw = A.azw + (int64_t)kAzCap * P.node_off;
    auto azval = [&](int a, const int* x) -> double {  // (A z_a) at node x
      double az = 0.0;
      for (int o = 0; o < (1 << D); o++) {
        int e[3] = {0, 0, 0};
        bool ok = true;
        for (int i = 0; i < D; i++) {
          e[i] = x[i] - 1 + ((o >> i) & 1);
          ok = ok && e[i] >= 0 && e[i] < g.nc[i];
        }
        if (!ok) continue;
        const int ac = (~o) & ((1 << D) - 1);
        double zc[1 << D];
        bool any = false;
        for (int b = 0; b < (1 << D); b++) {
          int xb[3] = {e[0] + (b & 1), e[1] + ((b >> 1) & 1), 0};
          zc[b] = (cm[node_id<D>(g, xb)] == a) ? 1.0 : 0.0;
          any = any || zc[b] != 0.0;
        }
        if (!any) continue;
        double W[DimC<D>::NW];
        elem_W<D>(A, P, g, e, W);
        az += elem_row<D>(W, zc, ac);
      }
      return az;
    };
    // one warp per component over its grown bounding box in row-major chunks of 32 nodes
    // (ballots keep the node order), counts then one block scan (ncomp <= ncmax < blockDim)
    const int wl = threadIdx.x & 31, wn = blockDim.x >> 5;
    auto gbox = [&](int a, int& x0, int& y0, int& ex, int& ey) {
      const int* bx = box + a * 6;
      x0 = max(bx[0] - 1, 0);
      y0 = max(bx[1] - 1, 0);
      ex = min(bx[3] + 1, g.nn[0] - 1) - x0 + 1;
      ey = min(bx[4] + 1, g.nn[1] - 1) - y0 + 1;
    };
    __shared__ int azc[256];
    for (int a = threadIdx.x >> 5; a < ncomp; a += wn) {
      int x0, y0, ex, ey;
      gbox(a, x0, y0, ex, ey);
      int c = 0;
      for (int base = 0; base < ex * ey; base += 32) {
        const int idx = base + wl;
        bool nz = false;
        if (idx < ex * ey) {
          const int xx[3] = {x0 + idx % ex, y0 + idx / ex, 0};
          nz = azval(a, xx) != 0.0;
        }
        c += __popc(__ballot_sync(FULLMASK, nz));
      }
      if (wl == 0) azc[a] = c;
    }
    __syncthreads();
    const int myc = ((int)threadIdx.x < ncomp) ? azc[threadIdx.x] : 0;
    __shared__ int aztot;
    const int aexcl = block_excl_scan(myc, wtot, &aztot);
    if ((int)threadIdx.x < ncomp) ap[threadIdx.x] = aexcl;
    if (threadIdx.x == 0) ap[ncomp] = aztot;
    __syncthreads();
    if (aztot > kAzCap * nn) {  // overflow: no coarse space for this window
      for (int k = threadIdx.x; k < nn; k += blockDim.x) cm[k] = -1;
      if (threadIdx.x == 0) A.ncomp[mp] = 0;
      return;
    }
    for (int a = threadIdx.x >> 5; a < ncomp; a += wn) {
      int x0, y0, ex, ey;
      gbox(a, x0, y0, ex, ey);
      int o = ap[a];
      for (int base = 0; base < ex * ey; base += 32) {
        const int idx = base + wl;
        double w = 0.0;
        int x = 0, y = 0;
        if (idx < ex * ey) {
          x = x0 + idx % ex;
          y = y0 + idx / ex;
          const int xx[3] = {x, y, 0};
          w = azval(a, xx);
        }
        const unsigned m = __ballot_sync(FULLMASK, w != 0.0);
        if (w != 0.0) {
          const int at = o + __popc(m & ((1u << wl) - 1u));
          ai[at] = x | (y << 16);
          aw[at] = w;
        }
        o += __popc(m);
      }
    }
    __syncthreads();
  }
  // C z_a: thread per component over the cells touching it (its bounding box grown by one cell
  // on the lower sides), contributions m_{E,j,a} = [id_E = j] h^D / 2^D per corner in the
  // component, accumulated per constraint row in cell order (fixed order)
  (void)ebs;
  for (int a = threadIdx.x; a < ncomp; a += blockDim.x) {
    for (int r = 0; r < nc; r++) CZ[(int64_t)r * A.ncmax + a] = 0.0;
    const int* bx = box + a * 6;
    int lo[3], hi[3];
    for (int i = 0; i < 3; i++) {
      lo[i] = (i < D) ? max(bx[i] - 1, 0) : 0;
      hi[i] = (i < D) ? min(bx[3 + i], g.nc[i] - 1) : 0;
    }
    for (int ez = lo[2]; ez <= hi[2]; ez++)
      for (int ey = lo[1]; ey <= hi[1]; ey++)
        for (int ex = lo[0]; ex <= hi[0]; ex++) {
          const int e[3] = {ex, ey, ez};
          unsigned in = 0;
          for (int b = 0; b < (1 << D); b++) {
            const int xb[3] = {ex + (b & 1), ey + ((b >> 1) & 1), (D == 3) ? ez + ((b >> 2) & 1) : 0};
            if (cm[node_id<D>(g, xb)] == a) in |= 1u << b;
          }
          if (!in) continue;
          const int q = elem_subcell<D>(A, P, g, e);
          for (int j = 0; j < A.N; j++) {
            double m = 0.0;
            for (int b = 0; b < (1 << D); b++)
              if ((in >> b) & 1u) m += elem_m<D>(A, P, g, e, j, b);
            CZ[(int64_t)(q * A.N + j) * A.ncmax + a] += m;
          }
        }
  }
}

cudaError_t launch_coarse_setup(const LevelArgs& A, cudaStream_t st) {
  const size_t sm = sizeof(double) * A.ncon + sizeof(int) * 512;
  if (A.D == 2) k_coarse_setup<2><<<A.nprob_mp, 512, sm, st>>>(A);
  else k_coarse_setup<3><<<A.nprob_mp, 512, sm, st>>>(A);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// Large oversampling (2D windows with more constraint rows than the dense path holds, l >= 4):
// S = C D^-1 C^T couples only subcells that share nodes, |q1 - q2| <= w + 1 in the lexicographic
// subcell order, so with rows r = q N + j its half-bandwidth is (w + 2) N - 1.  The equilibrated
// S~ = Lambda S Lambda (Lambda = diag(S)^-1/2, inactive rows -> identity, as in k_proj_setup) is
// factored by banded Cholesky in shared memory (one warp, left-looking by columns); k_pcg applies
// S^-1 = Lambda S~^-1 Lambda by two banded triangular solves.  A pivot below 1e-12 means
// dependent rows (reading R20), which this path does not handle: flag 8, reported by the host.
template <int D>
__global__ void k_proj_setup_band(LevelArgs A) {
  const int mp = blockIdx.x;
  const ProbDesc& P = A.probs[mp];
  const Geo<D> g = level_geo<D>(A, P);
  extern __shared__ double smem[];
  const int nc = A.ncon, bw = A.band, B1 = bw + 1;
  double* Lb = smem;                // nc*B1: Lb[r*B1 + k] = S(r, r-k), then L(r, r-k)
  double* ds = Lb + nc * B1;        // nc
  double* scratch = ds + nc;        // 32*16
  double* tot = scratch + 32 * 16;  // 16
  int* eb = reinterpret_cast<int*>(tot + 16);
  double* dinv = A.dinv + P.node_off;
  for (int k = threadIdx.x; k < g.nnodes; k += blockDim.x) {
    const double dv = 1.0 / diag_node<D>(A, P, g, k);
    dinv[k] = (D == 2) ? (double)(float)dv : dv;
  }
  double* nwt = A.NWt + P.node_off * A.N;
  for (int k = threadIdx.x; k < g.nnodes; k += blockDim.x) {
    int x[3];
    node_xyz<D>(g, k, x);
    double w[4] = {0.0, 0.0, 0.0, 0.0};
    for (int ep = 0; ep < (1 << D); ep++) {
      int e[3] = {0, 0, 0};
      bool ok = true;
      for (int i = 0; i < D; i++) {
        e[i] = x[i] - 1 + ((ep >> i) & 1);
        ok = ok && e[i] >= 0 && e[i] < g.nc[i];
      }
      if (!ok) continue;
      const int a = (~ep) & ((1 << D) - 1);
      for (int j = 0; j < A.N; j++) w[j] += elem_m<D>(A, P, g, e, j, a);
    }
    for (int j = 0; j < A.N; j++) nwt[(int64_t)j * g.nnodes + k] = w[j];
  }
  for (int i = threadIdx.x; i < nc * B1; i += blockDim.x) Lb[i] = 0.0;
  __shared__ int ntask;
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  subcell_boxes<D>(A, P, g, eb, &ntask);  // also syncs
  const int N = A.N;
  for (int q1 = 0; q1 < A.nsub; q1++) {
    for (int q2 = q1; q2 < A.nsub; q2++) {
      const int* b1 = eb + q1 * 6;
      const int* b2 = eb + q2 * 6;
      int lo[3], hi[3];
      bool empty = false;
      for (int i = 0; i < 3; i++) {
        if (i >= D) { lo[i] = 0; hi[i] = 0; continue; }
        if (b1[3 + i] == 0 || b2[3 + i] == 0) { empty = true; break; }
        lo[i] = max(b1[i], b2[i]);
        hi[i] = min(b1[i] + b1[3 + i], b2[i] + b2[3 + i]);
        if (hi[i] < lo[i]) { empty = true; break; }
      }
      if (empty) continue;
      const int ex = hi[0] - lo[0] + 1, ey = hi[1] - lo[1] + 1, ez = hi[2] - lo[2] + 1;
      const int cnt = ex * ey * ez;
      double v[16];
      for (int i = 0; i < 16; i++) v[i] = 0.0;
      for (int idx = threadIdx.x; idx < cnt; idx += blockDim.x) {
        const int x[3] = {lo[0] + idx % ex, lo[1] + (idx / ex) % ey, lo[2] + idx / (ex * ey)};
        const int k = node_id<D>(g, x);
        double w1[4] = {0, 0, 0, 0}, w2[4] = {0, 0, 0, 0};
        for (int ep = 0; ep < (1 << D); ep++) {
          int e[3] = {0, 0, 0};
          bool ok = true;
          for (int i = 0; i < D; i++) {
            e[i] = x[i] - 1 + ((ep >> i) & 1);
            ok = ok && e[i] >= 0 && e[i] < g.nc[i];
          }
          if (!ok) continue;
          const int q = elem_subcell<D>(A, P, g, e);
          if (q != q1 && q != q2) continue;
          const int a = (~ep) & ((1 << D) - 1);
          for (int j = 0; j < N; j++) {
            const double m = elem_m<D>(A, P, g, e, j, a);
            if (q == q1) w1[j] += m;
            if (q == q2) w2[j] += m;
          }
        }
        const double di = dinv[k];
        for (int j1 = 0; j1 < N; j1++)
          for (int j2 = 0; j2 < N; j2++) v[j1 * 4 + j2] += w1[j1] * w2[j2] * di;
      }
      block_sum<16>(v, scratch, tot);
      if (threadIdx.x == 0) {
        for (int j1 = 0; j1 < N; j1++)
          for (int j2 = 0; j2 < N; j2++) {
            const int r1 = q1 * N + j1, r2 = q2 * N + j2;
            const int r = max(r1, r2), c = min(r1, r2);
            if (r - c > bw) {
              if (tot[j1 * 4 + j2] != 0.0) bad = 1;
            } else {
              Lb[r * B1 + (r - c)] = tot[j1 * 4 + j2];
            }
          }
      }
      __syncthreads();
    }
  }
  const double* meas = A.meas + (int64_t)mp * nc;
  for (int i = threadIdx.x; i < nc; i += blockDim.x) {
    const bool act = meas[i] > 0.0 && Lb[i * B1] > 0.0;
    ds[i] = act ? 1.0 / sqrt(Lb[i * B1]) : 0.0;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < nc * B1; idx += blockDim.x) {
    const int r = idx / B1, k = idx - r * B1, c = r - k;
    if (c < 0) Lb[idx] = 0.0;
    else if (ds[r] == 0.0 || ds[c] == 0.0) Lb[idx] = (k == 0) ? 1.0 : 0.0;
    else Lb[idx] *= ds[r] * ds[c];
  }
  __syncthreads();
  if (threadIdx.x < 32) {  // banded Cholesky, left-looking by columns
    const int lane = threadIdx.x;
    for (int j = 0; j < nc; j++) {
      double sq = 0.0;
      for (int k = 1 + lane; k <= min(bw, j); k += 32) sq += Lb[j * B1 + k] * Lb[j * B1 + k];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(FULLMASK, sq, o);
      const double d = Lb[j * B1] - sq;
      if (!(d > 1e-12) && lane == 0) bad = 2;
      const double ljj = sqrt(fmax(d, 1e-300));
      __syncwarp();
      if (lane == 0) Lb[j * B1] = ljj;
      for (int i = j + 1 + lane; i <= min(j + bw, nc - 1); i += 32) {
        double sv = Lb[i * B1 + (i - j)];
        for (int m = max(i - bw, 0); m < j; m++) sv -= Lb[i * B1 + (i - m)] * Lb[j * B1 + (j - m)];
        Lb[i * B1 + (i - j)] = sv / ljj;
      }
      __syncwarp();
    }
  }
  __syncthreads();
  if (bad && threadIdx.x == 0) atomicOr(&A.flags[mp], 8);
  double* out = A.Sinv + (int64_t)mp * nc * B1;
  for (int idx = threadIdx.x; idx < nc * B1; idx += blockDim.x) out[idx] = Lb[idx];
  for (int i = threadIdx.x; i < nc; i += blockDim.x) A.pinv_ds[(int64_t)mp * nc + i] = ds[i];
}

// ---------------------------------------------------------------------------------------
// Reading R20, direct form.  S~ (unit diagonal on active rows) is factored by
// Cholesky with diagonal pivoting, S~ = L L^T + T, stopping at rank r when every remaining pivot is
// <= 1e-11 (T: the trailing Schur complement).  Then S~^+ = L G^-2 L^T with G = L^T L (r x r; its
// eigenvalues are the r nonzero eigenvalues of L L^T), i.e. W W^T with W = L G^-1.  This equals
// the eigen-truncated pseudo-inverse of the oracle (eigenvalues <= 1e-11 lambda_max dropped) when
// both decide the same rank, which two bounds certify:
//   (a) trace(T) <= 1e-12: by Weyl, the n - r smallest eigenvalues of S~ are <= lambda_max(T) <=
//       trace(T) < 1e-11 <= 1e-11 lambda_max (lambda_max >= max diag = 1): all dropped by the oracle;
//   (b) 1 / trace(G^-1) >= 1e-9 n: the r largest eigenvalues of S~ are >= those of L L^T (T is
//       PSD) >= lambda_min(G) >= 1 / trace(G^-1) > 1e-11 n >= 1e-11 lambda_max: all kept.
// A window that fails either bound is left to the Jacobi eigen-solver (k_pinv, flag 16).
// Per window n pivot steps with three barriers each plus one Gauss-Jordan inverse of G, against the
// ~10 Jacobi sweeps x (n - 1) rounds x 3 barriers of k_pinv.
__global__ void k_pinv_all_jacobi(LevelArgs A) {  // dev switch MCH_PINV_JACOBI: skip the direct form
  const int mp = blockIdx.x * blockDim.x + threadIdx.x;
  if (mp < A.nprob_mp && (A.flags[mp] & 2)) A.flags[mp] |= 16;
}

__global__ void __launch_bounds__(256) k_pinv_chol(LevelArgs A) {
  const int mp = blockIdx.x;
  if (!(A.flags[mp] & 2)) return;
  const int n = A.ncon, tid = threadIdx.x, lane = tid & 31, nt = blockDim.x;
  extern __shared__ double sm[];
  double* Sw = sm;           // n*n working Schur complement, later W = L G^-1 (n x r)
  double* Lc = Sw + n * n;   // column k of L at Lc[k*n + i] (i: original row index)
  double* Gm = Lc + n * n;   // G = L^T L, inverted in place (r x r, stride n)
  int* done = reinterpret_cast<int*>(Gm + n * n);  // n
  __shared__ int piv_s, amb_s;
  __shared__ double dp_s;
  double* Sg = A.Sinv + (int64_t)mp * n * n;
  for (int idx = tid; idx < n * n; idx += nt) Sw[idx] = Sg[idx];
  for (int i = tid; i < n; i += nt) done[i] = 0;
  __syncthreads();
  int r = 0;
  for (int k = 0; k < n; k++) {
    if (tid < 32) {  // largest remaining pivot, ties to the smaller index
      double best = -1.0;
      int bi = n;
      for (int i = lane; i < n; i += 32) {
        const double d = Sw[i * n + i];
        if (!done[i] && d > best) { best = d; bi = i; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(FULLMASK, best, o);
        const int oi = __shfl_xor_sync(FULLMASK, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (lane == 0) { piv_s = bi; dp_s = best; }
    }
    __syncthreads();
    if (!(dp_s > 1e-11)) break;  // uniform
    const int p = piv_s;
    const double lp = sqrt(dp_s), ilp = 1.0 / lp;
    for (int i = tid; i < n; i += nt) Lc[k * n + i] = done[i] ? 0.0 : ((i == p) ? lp : Sw[i * n + p] * ilp);
    __syncthreads();
    if (tid == 0) done[p] = 1;
    const double* lk = Lc + k * n;
    for (int idx = tid; idx < n * n; idx += nt) {
      const int i = idx / n, j = idx - (idx / n) * n;
      if (!done[i] && !done[j] && i != p && j != p) Sw[idx] -= lk[i] * lk[j];
    }
    r = k + 1;
    __syncthreads();
  }
  // (a) trace of the trailing Schur complement
  if (tid < 32) {
    double tr = 0.0;
    for (int i = lane; i < n; i += 32)
      if (!done[i]) tr += fmax(Sw[i * n + i], 0.0);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tr += __shfl_xor_sync(FULLMASK, tr, o);
    if (lane == 0) amb_s = !(tr <= 1e-12);
  }
  __syncthreads();
  if (amb_s) {
    if (tid == 0) atomicOr(&A.flags[mp], 16);
    return;
  }
  // G = L^T L
  for (int idx = tid; idx < r * r; idx += nt) {
    const int a = idx / r, b = idx - (idx / r) * r;
    if (a > b) continue;
    double acc = 0.0;
    for (int i = 0; i < n; i++) acc += Lc[a * n + i] * Lc[b * n + i];
    Gm[a * n + b] = acc;
    Gm[b * n + a] = acc;
  }
  __syncthreads();
  // G^-1 in place (Gauss-Jordan, SPD: no pivoting)
  for (int q = 0; q < r; q++) {
    const double ip = 1.0 / Gm[q * n + q];
    __syncthreads();
    for (int idx = tid; idx < r * r; idx += nt) {
      const int i = idx / r, j = idx - (idx / r) * r;
      if (i != q && j != q) Gm[i * n + j] -= Gm[i * n + q] * ip * Gm[q * n + j];
    }
    __syncthreads();
    for (int i = tid; i < r; i += nt) {
      if (i != q) {
        Gm[i * n + q] = -Gm[i * n + q] * ip;
        Gm[q * n + i] = Gm[q * n + i] * ip;
      }
    }
    __syncthreads();
    if (tid == 0) Gm[q * n + q] = ip;
    __syncthreads();
  }
  // (b) trace(G^-1)
  if (tid < 32) {
    double tr = 0.0;
    for (int a = lane; a < r; a += 32) tr += Gm[a * n + a];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tr += __shfl_xor_sync(FULLMASK, tr, o);
    if (lane == 0) amb_s = !(tr > 0.0 && tr * 1e-9 * n <= 1.0);
  }
  __syncthreads();
  if (amb_s) {
    if (tid == 0) atomicOr(&A.flags[mp], 16);
    return;
  }
  if (tid == 0 && r < n) atomicOr(&A.flags[mp], 4);  // rows were dependent
  // W = L G^-1 (n x r) into Sw
  for (int idx = tid; idx < n * r; idx += nt) {
    const int i = idx / r, a = idx - (idx / r) * r;
    double acc = 0.0;
    for (int b = 0; b < r; b++) acc += Lc[b * n + i] * Gm[b * n + a];
    Sw[i * n + a] = acc;
  }
  __syncthreads();
  // S^+ = Lambda W W^T Lambda, symmetric
  const double* ds = A.pinv_ds + (int64_t)mp * n;
  for (int idx = tid; idx < n * n; idx += nt) {
    const int i = idx / n, j = idx - (idx / n) * n;
    if (i > j) continue;
    double acc = 0.0;
    for (int a = 0; a < r; a++) acc += Sw[i * n + a] * Sw[j * n + a];
    const double v = acc * ds[i] * ds[j];
    Sg[i * n + j] = v;
    Sg[j * n + i] = v;
  }
}

// ---------------------------------------------------------------------------------------
// Reading R20: S^+ = Lambda S~^+ Lambda with S~ = V diag(lambda) V^T, eigenvalues
// below 1e-11 lambda_max dropped.  One CTA per flagged window: parallel cyclic Jacobi with the
// round-robin ordering (each round rotates nc/2 disjoint pairs at once; the row and column updates
// of all pairs are spread over the CTA), sweeps until the off-diagonal mass is below 1e-34 of the
// diagonal's (at most 40 sweeps).
__global__ void __launch_bounds__(256) k_pinv(LevelArgs A) {
  const int mp = blockIdx.x;
  if (!(A.flags[mp] & 16)) return;  // only the windows k_pinv_chol could not certify
  const int nc = A.ncon, tid = threadIdx.x, lane = tid & 31, nt = blockDim.x;
  extern __shared__ double sm[];
  double* S = sm;            // nc*nc (padded to even m)
  const int m = (nc + 1) & ~1;
  double* V = S + m * m;     // m*m
  double* rc = V + m * m;    // [64] cos, [64] sin of this round's rotations (m <= 128)
  double* rs = rc + 64;
  int* pos = reinterpret_cast<int*>(rs + 64);  // m
  int* rp = pos + m;         // [64] p, [64] q of this round's pairs (q = -1: no rotation)
  int* rq = rp + 64;
  __shared__ int done;
  double* Sg = A.Sinv + (int64_t)mp * nc * nc;
  for (int idx = tid; idx < m * m; idx += nt) {
    const int i = idx / m, j = idx % m;
    S[idx] = (i < nc && j < nc) ? Sg[i * nc + j] : 0.0;  // padded row/column: decoupled zero
    V[idx] = (i == j) ? 1.0 : 0.0;
  }
  for (int i = tid; i < m; i += nt) pos[i] = i;
  __syncthreads();
  const int np = m / 2;
  for (int sweep = 0; sweep < 40; sweep++) {
    if (tid < 32) {  // convergence test by warp 0 (one fixed summation order)
      double off = 0.0, dia = 0.0;
      for (int idx = lane; idx < m * m; idx += 32) {
        const int i = idx / m, j = idx % m;
        const double a = S[idx];
        if (i < j) off += a * a;
        else if (i == j) dia += a * a;
      }
      for (int o = 16; o > 0; o >>= 1) {
        off += __shfl_xor_sync(FULLMASK, off, o);
        dia += __shfl_xor_sync(FULLMASK, dia, o);
      }
      if (lane == 0) done = (off <= MCH_PINV_TOL * dia);
    }
    __syncthreads();
#ifdef MCH_PINV_STATS
    if (tid == 0 && (done || sweep == 39)) atomicAdd(&A.flags[mp], (sweep + 1) << 8);
#endif
    if (done) break;
    for (int round = 0; round < m - 1; round++) {
      // pairs of this round: (pos(k), pos(m-1-k)), k < m/2, circle method (index 0 fixed, the
      // others rotated by `round`)
      const int m1 = m - 1;
      auto posr = [&](int i) { return (i == 0) ? 0 : ((i - 1 - round) % m1 + m1) % m1 + 1; };
      if (tid < np) {
        int p = posr(tid), q = posr(m - 1 - tid);
        if (p > q) { const int tt = p; p = q; q = tt; }
        const double apq = S[p * m + q];
        double c = 1.0, sn = 0.0;
        if (fabs(apq) >= 1e-300) {
          const double th = (S[q * m + q] - S[p * m + p]) / (2.0 * apq);
          const double t = (th >= 0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
          c = 1.0 / sqrt(t * t + 1.0);
          sn = t * c;
        } else {
          q = -1;  // no rotation
        }
        rp[tid] = p;
        rq[tid] = q;
        rc[tid] = c;
        rs[tid] = sn;
      }
      __syncthreads();
      // rows p, q (all columns), then columns p, q (all rows): S <- J^T S J, V <- V J; the pairs
      // are disjoint, so every element is updated once per phase (as the one-warp form)
      for (int idx = tid; idx < np * m; idx += nt) {
        const int k2 = idx / m, k = idx - k2 * m;
        const int p = rp[k2], q = rq[k2];
        if (q < 0) continue;
        const double c = rc[k2], sn = rs[k2];
        const double skp = S[p * m + k], skq = S[q * m + k];
        S[p * m + k] = c * skp - sn * skq;
        S[q * m + k] = sn * skp + c * skq;
      }
      __syncthreads();
      for (int idx = tid; idx < np * m; idx += nt) {
        const int k2 = idx / m, k = idx - k2 * m;
        const int p = rp[k2], q = rq[k2];
        if (q < 0) continue;
        const double c = rc[k2], sn = rs[k2];
        const double skp = S[k * m + p], skq = S[k * m + q];
        S[k * m + p] = (k == q) ? 0.0 : c * skp - sn * skq;  // the rotated-out pair entries are set to 0
        S[k * m + q] = (k == p) ? 0.0 : sn * skp + c * skq;
        const double vkp = V[k * m + p], vkq = V[k * m + q];
        V[k * m + p] = c * vkp - sn * vkq;
        V[k * m + q] = sn * vkp + c * vkq;
      }
      __syncthreads();
    }
  }
  __shared__ double lmax_s;
  __shared__ int trunc_s;
  if (tid < 32) {
    double lmax = 0.0;
    for (int i = lane; i < nc; i += 32) lmax = fmax(lmax, S[i * m + i]);
    for (int o = 16; o > 0; o >>= 1) lmax = fmax(lmax, __shfl_xor_sync(FULLMASK, lmax, o));
    bool trunc = false;
    for (int k = lane; k < nc; k += 32) trunc = trunc || !(S[k * m + k] > 1e-11 * lmax);
    const bool any = __any_sync(FULLMASK, trunc);
    if (lane == 0) {
      lmax_s = lmax;
      trunc_s = any;
      if (any) atomicOr(&A.flags[mp], 4);  // rows were dependent
    }
  }
  __syncthreads();
  const double lmax = lmax_s;
  const double* ds = A.pinv_ds + (int64_t)mp * nc;
  // 1/lambda_k of the kept eigenvalues (0 for the truncated ones), once per window: the assembly
  // below then has no division (r01 divided in its innermost loop, nc^3 divisions per window)
  double* il = rc;  // rc/rs (128 doubles) are free now
  for (int k = tid; k < nc; k += nt) {
    const double lk = S[k * m + k];
    il[k] = (lk > 1e-11 * lmax) ? 1.0 / lk : 0.0;
  }
  __syncthreads();
  // S+ = V diag(il) V^T, symmetric: entries i <= j formed once and mirrored
  for (int idx = tid; idx < nc * nc; idx += nt) {
    const int i = idx / nc, j = idx % nc;
    if (i > j) continue;
    double acc = 0.0;
    for (int k = 0; k < nc; k++) acc += V[i * m + k] * V[j * m + k] * il[k];
    const double v = acc * ds[i] * ds[j];
    Sg[i * nc + j] = v;
    Sg[j * nc + i] = v;
  }
}

// ---------------------------------------------------------------------------------------
// projected PCG: one CTA per problem (macropoint, rhs)
template <int D>
__global__ void __launch_bounds__(512, (D == 2) ? 2 : 1) k_pcg(LevelArgs A) {
  const int prob = blockIdx.x;
  const int mp = prob / A.n_rhs, r = prob % A.n_rhs;
  const ProbDesc& P = A.probs[mp];
  const Geo<D> g = level_geo<D>(A, P);
  const int nc = A.ncon;
  const bool band = A.band > 0;
  const int B1 = A.band + 1;
  extern __shared__ double smem[];
  // dense: S^-1 (nc*nc) and per-warp constraint bins (32*nc); band: the banded Cholesky factor
  // (nc*B1) and its row scales, constraint sums owned per subcell (no bins)
  double* Si = smem;
  double* ds = Si + (band ? nc * B1 : nc * nc);  // band only: nc
  double* yhat = ds + (band ? nc : 0);           // nc
  double* cvec = yhat + nc;                       // nc
  double* tg = cvec + nc;                         // nc
  double* gcol = tg + nc;                         // nc
  double* g0col = gcol + nc;                      // nc
  const bool crs = A.coarse && !band && A.ncomp[mp] > 0;  // two-level preconditioner
  double* zr = g0col + nc;                        // coarse: ncmax (E^-1 Z^T r)
  double* vv = zr + (A.coarse ? A.ncmax : 0);     // coarse: ncmax (coarse part of z)
  double* bins = vv + (A.coarse ? A.ncmax : 0);   // dense: 32*nc
  double* scratch = bins + (band ? 0 : 32 * nc);  // 32*4
  double* tot = scratch + 32 * 4;                 // 4
  int* eb = reinterpret_cast<int*>(tot + 4);
  __shared__ int ntask;

  const int nn = g.nnodes;
  double* x = A.X + P.vec_off + (int64_t)r * nn;
  double* rv = A.R + P.vec_off + (int64_t)r * nn;
  double* p = A.P + P.vec_off + (int64_t)r * nn;
  double* q = A.Q + P.vec_off + (int64_t)r * nn;
  const double* b = (A.level >= 2) ? A.B + P.vec_off + (int64_t)r * nn : nullptr;
  const double* dinv = A.dinv + P.node_off;
  const double* nwt = A.NWt + P.node_off * A.N;
  if (band) {
    for (int i = threadIdx.x; i < nc * B1; i += blockDim.x) Si[i] = A.Sinv[(int64_t)mp * nc * B1 + i];
    for (int i = threadIdx.x; i < nc; i += blockDim.x) ds[i] = A.pinv_ds[(int64_t)mp * nc + i];
  } else {
    for (int i = threadIdx.x; i < nc * nc; i += blockDim.x) Si[i] = A.Sinv[(int64_t)mp * nc * nc + i];
  }
  subcell_boxes<D>(A, P, g, eb, &ntask);

  auto sinv_apply = [&](const double* in, double* out) {
    if (band) {  // out = Lambda L^-T L^-1 Lambda in (warp 0; in != out)
      if (threadIdx.x < 32) {
        const int lane = threadIdx.x, bw = A.band;
        for (int i = lane; i < nc; i += 32) out[i] = ds[i] * in[i];
        __syncwarp();
        for (int r = 0; r < nc; r++) {
          double sv = 0.0;
          for (int k = 1 + lane; k <= min(bw, r); k += 32) sv += Si[r * B1 + k] * out[r - k];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) sv += __shfl_xor_sync(FULLMASK, sv, o);
          if (lane == 0) out[r] = (out[r] - sv) / Si[r * B1];
          __syncwarp();
        }
        for (int r = nc - 1; r >= 0; r--) {
          double sv = 0.0;
          for (int k = 1 + lane; k <= bw && r + k < nc; k += 32) sv += Si[(r + k) * B1 + k] * out[r + k];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) sv += __shfl_xor_sync(FULLMASK, sv, o);
          if (lane == 0) out[r] = (out[r] - sv) / Si[r * B1];
          __syncwarp();
        }
        for (int i = lane; i < nc; i += 32) out[i] *= ds[i];
      }
    } else {
      for (int i = threadIdx.x; i < nc; i += blockDim.x) {
        double s = 0.0;
        for (int j = 0; j < nc; j++) s += Si[i * nc + j] * in[j];
        out[i] = s;
      }
    }
    __syncthreads();
  };
  auto capply = [&](auto&& uf, double* out) {
    if (band) constraint_apply_owned<D>(A, P, g, eb, uf, out);
    else constraint_apply<D>(A, P, g, eb, ntask, uf, bins, out);
  };
  const int nca = crs ? A.ncomp[mp] : 0;
  const int* cmp = A.cmap + P.node_off;
  const int* cbx = A.cbox + (int64_t)mp * A.ncmax * 6;
  const double* Ei = A.Einv + (int64_t)mp * A.ncmax;
  const double* CZm = A.CZ + (int64_t)mp * nc * A.ncmax;
  // zr = E^-1 Z^T rvec (one warp per component over its bounding box, fixed order), c += (CZ) zr;
  // returns (Z^T r)^T E^-1 (Z^T r)
  auto coarse_c = [&](const double* rvec, double* c) -> double {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    double part[1] = {0.0};
    for (int a = wid; a < nca; a += nw) {
      const int* bx = cbx + a * 6;
      const int ex = bx[3] - bx[0] + 1, ey = bx[4] - bx[1] + 1, ez = (D == 3) ? bx[5] - bx[2] + 1 : 1;
      double sv = 0.0;
      for (int idx = lane; idx < ex * ey * ez; idx += 32) {
        const int xx[3] = {bx[0] + idx % ex, bx[1] + (idx / ex) % ey, (D == 3) ? bx[2] + idx / (ex * ey) : 0};
        const int k = node_id<D>(g, xx);
        if (cmp[k] == a) sv += rvec[k];
      }
      for (int o = 16; o > 0; o >>= 1) sv += __shfl_xor_sync(FULLMASK, sv, o);
      if (lane == 0) {
        zr[a] = sv * Ei[a];
        part[0] += sv * sv * Ei[a];
      }
    }
    block_sum<1>(part, scratch, tot);
    const double zw = tot[0];
    for (int i = threadIdx.x; i < nc; i += blockDim.x) {
      double acc = 0.0;
      for (int a = 0; a < nca; a++) acc += CZm[(int64_t)i * A.ncmax + a] * zr[a];
      c[i] += acc;
    }
    __syncthreads();
    return zw;
  };
  // vv = s0 * zr - E^-1 (CZ)^T yh   (s0 = 0: the coarse part of M^-1 C^T yh, negated)
  auto coarse_v = [&](const double* yh, double s0) {
    for (int a = threadIdx.x; a < nca; a += blockDim.x) {
      double acc = 0.0;
      for (int i = 0; i < nc; i++) acc += CZm[(int64_t)i * A.ncmax + a] * yh[i];
      vv[a] = (s0 != 0.0 ? s0 * zr[a] : 0.0) - Ei[a] * acc;  // zr is not yet set when s0 == 0
    }
    __syncthreads();
  };
  auto cz_at = [&](int k) -> double {  // coarse part of the preconditioned vector at node k
    if (!crs) return 0.0;
    const int a = cmp[k];
    return (a >= 0) ? vv[a] : 0.0;
  };

  // init: x = D^-1 C^T S^-1 t, r = A x - b (unprojected), c = C D^-1 r, yhat = S^-1 c.
  // returns r^T D^-1 r of the unprojected residual
  auto init = [&](const double* targets, const double* bb) -> double {
    for (int i = threadIdx.x; i < nc; i += blockDim.x) tg[i] = targets[i];
    __syncthreads();
    sinv_apply(tg, yhat);
    if (crs) coarse_v(yhat, 0.0);  // x0 = M^-1 C^T S^-1 t: coarse part = -vv
    for (int k = threadIdx.x; k < nn; k += blockDim.x) x[k] = dinv[k] * ct_node<D>(A, P, g, yhat, k) - cz_at(k);
    __syncthreads();
    double v[1] = {0.0};
    for (int k = threadIdx.x; k < nn; k += blockDim.x) {
      const double rk = apply_node<D>(A, P, g, x, k) - (bb ? bb[k] : 0.0);
      rv[k] = rk;
      v[0] += dinv[k] * rk * rk;
    }
    block_sum<1>(v, scratch, tot);
    double rr = tot[0];
    capply([&](int k) { return dinv[k] * rv[k]; }, cvec);
    if (crs) rr += coarse_c(rv, cvec);  // r^T M^-1 r and C M^-1 r
    sinv_apply(cvec, yhat);
    if (crs) coarse_v(yhat, 1.0);  // z = M^-1 (r - C^T yhat): coarse part vv
    return rr;
  };

  // targets of this rhs: column r of g (or g0 at level 1)
  const double* gsrc = (A.level >= 2) ? A.g : A.g0;
  for (int i = threadIdx.x; i < nc; i += blockDim.x) {
    gcol[i] = gsrc[((int64_t)mp * nc + i) * A.n_rhs + r];
    g0col[i] = A.g0[((int64_t)mp * nc + i) * A.n_rhs + r];
  }
  __syncthreads();
  double rz_ref = 0.0, rr_ref = 0.0;
  if (A.level >= 2) {
    // reference scale: initial projected residual of the full (non-hierarchical) problem,
    // projected explicitly (no cancellation formula)
    rr_ref = init(g0col, nullptr);
    double v[1] = {0.0};
    for (int k = threadIdx.x; k < nn; k += blockDim.x) {
      const double rk = rv[k] - ct_node<D>(A, P, g, yhat, k);
      v[0] += dinv[k] * rk * rk;
    }
    block_sum<1>(v, scratch, tot);
    rz_ref = tot[0];
  }
  const double rr0 = init(gcol, b);
  for (int k = threadIdx.x; k < nn; k += blockDim.x) p[k] = 0.0;
  __syncthreads();

  const double tol2 = A.rtol * A.rtol;
  // attainable-accuracy floor: the first projection leaves roundoff of ~eps*|r_unprojected|
  const double floor2 = 1e-30 * fmax(rr0, rr_ref);
  double beta = 0.0, rz = 0.0, ref = 0.0;
  int it = 0, breakdown = 0;
  for (;; it++) {
    // pass 1: r <- r - C^T yhat (re-projection), z = D^-1 r, p <- -z + beta p, rz = r.z
    double v[1] = {0.0};
    for (int k = threadIdx.x; k < nn; k += blockDim.x) {
      const double rk = rv[k] - ct_fast<D>(A, P, g, nwt, yhat, k);
      const double zk = dinv[k] * rk + cz_at(k);
      rv[k] = rk;
      p[k] = -zk + beta * p[k];
      v[0] += rk * zk;
    }
    block_sum<1>(v, scratch, tot);
    rz = tot[0];
    if (it == 0) ref = fmax(rz, rz_ref);
    if (!(rz > fmax(tol2 * ref, floor2)) || it >= A.max_iter) break;
    // pass 1b: q = A p, pq
    double w[1] = {0.0};
    for (int k = threadIdx.x; k < nn; k += blockDim.x) {
      const double qk = apply_node<D>(A, P, g, p, k);
      q[k] = qk;
      w[0] += p[k] * qk;
    }
    block_sum<1>(w, scratch, tot);
    if (!(tot[0] > 0.0) || !isfinite(tot[0])) {  // loss of definiteness: report, do not loop
      breakdown = 1;
      break;
    }
    const double alpha = rz / tot[0];
    // pass 2: x += alpha p, r += alpha q, rr = r^T D^-1 r
    double u[1] = {0.0};
    for (int k = threadIdx.x; k < nn; k += blockDim.x) {
      x[k] += alpha * p[k];
      const double rk = rv[k] + alpha * q[k];
      rv[k] = rk;
      u[0] += dinv[k] * rk * rk;
    }
    block_sum<1>(u, scratch, tot);
    double rr = tot[0];
    capply([&](int k) { return dinv[k] * rv[k]; }, cvec);
    if (crs) rr += coarse_c(rv, cvec);
    sinv_apply(cvec, yhat);
    double cy = 0.0;
    for (int j = 0; j < nc; j++) cy += cvec[j] * yhat[j];
    beta = (rr - cy) / rz;
    if (crs) coarse_v(yhat, 1.0);
  }
  // feasibility restoration: x += D^-1 C^T S^-1 (g - C x)
  capply([&](int k) { return x[k]; }, cvec);
  for (int i = threadIdx.x; i < nc; i += blockDim.x) tg[i] = gcol[i] - cvec[i];
  __syncthreads();
  sinv_apply(tg, yhat);
  if (crs) coarse_v(yhat, 0.0);
  for (int k = threadIdx.x; k < nn; k += blockDim.x) x[k] += dinv[k] * ct_node<D>(A, P, g, yhat, k) - cz_at(k);
  __syncthreads();
  if (A.level == 1 && P.pool_off >= 0) {
    double* dst = A.pool + P.pool_off + (int64_t)r * nn;
    for (int k = threadIdx.x; k < nn; k += blockDim.x) dst[k] = x[k];
  }
  if (threadIdx.x == 0) {
    A.iters[prob] = it;
    A.relres[prob] = (ref > 0.0) ? sqrt(fmax(rz, 0.0) / ref) : 0.0;
    double* dg = A.diag + (int64_t)prob * 4;
    dg[0] = rz;
    dg[1] = ref;
    dg[2] = floor2;
    dg[3] = breakdown;
  }
}

// ---------------------------------------------------------------------------------------
// combine (levels >= 2): phi = P_n xi + I_p, one CTA per problem
template <int D>
__global__ void k_combine(LevelArgs A) {
  const int prob = blockIdx.x;
  const int mp = prob / A.n_rhs, r = prob % A.n_rhs;
  const ProbDesc& P = A.probs[mp];
  const Geo<D> gf = fine_geo<D>(P);
  const Geo<D> gl = level_geo<D>(A, P);
  double* I = A.FI + P.fine_off + (int64_t)r * gf.nnodes;
  const double* xi = A.X + P.vec_off + (int64_t)r * gl.nnodes;
  double* dst = (P.pool_off >= 0) ? A.pool + P.pool_off + (int64_t)r * gf.nnodes : nullptr;
  const int s = A.s;
  for (int k = threadIdx.x; k < gf.nnodes; k += blockDim.x) {
    int x[3];
    node_xyz<D>(gf, k, x);
    int c0[3];
    double t[3];
    for (int i = 0; i < 3; i++) {
      if (i < D) {
        c0[i] = x[i] / s;
        t[i] = (double)(x[i] - c0[i] * s) / s;
        if (c0[i] == gl.nc[i]) { c0[i] -= 1; t[i] = 1.0; }
      } else {
        c0[i] = 0;
        t[i] = 0.0;
      }
    }
    double v = 0.0;
    for (int a = 0; a < (1 << D); a++) {
      double wgt = 1.0;
      int xc[3] = {0, 0, 0};
      for (int i = 0; i < D; i++) {
        const int ai = (a >> i) & 1;
        wgt *= ai ? t[i] : 1.0 - t[i];
        xc[i] = c0[i] + ai;
      }
      if (wgt != 0.0) v += wgt * xi[node_id<D>(gl, xc)];
    }
    const double phi = I[k] + v;
    I[k] = phi;
    if (dst) dst[k] = phi;
  }
}

// all right-hand sides of a macropoint in one CTA: the interpolation weights and level-n node
// ids of each fine node are formed once; per rhs the arithmetic is k_combine's (bitwise equal)
template <int D>
__global__ void __launch_bounds__(256) k_combine_mr(LevelArgs A) {
  const int mp = blockIdx.x;
  const ProbDesc& P = A.probs[mp];
  const Geo<D> gf = fine_geo<D>(P);
  const Geo<D> gl = level_geo<D>(A, P);
  const int s = A.s, nr = A.n_rhs;
  const int64_t nnf = gf.nnodes, nnl = gl.nnodes;
  for (int k = threadIdx.x; k < gf.nnodes; k += blockDim.x) {
    int x[3];
    node_xyz<D>(gf, k, x);
    int c0[3];
    double t[3];
    for (int i = 0; i < 3; i++) {
      if (i < D) {
        c0[i] = x[i] / s;
        t[i] = (double)(x[i] - c0[i] * s) / s;
        if (c0[i] == gl.nc[i]) { c0[i] -= 1; t[i] = 1.0; }
      } else {
        c0[i] = 0;
        t[i] = 0.0;
      }
    }
    double wgt[1 << D];
    int nid[1 << D];
#pragma unroll
    for (int a = 0; a < (1 << D); a++) {
      double w = 1.0;
      int xc[3] = {0, 0, 0};
      for (int i = 0; i < D; i++) {
        const int ai = (a >> i) & 1;
        w *= ai ? t[i] : 1.0 - t[i];
        xc[i] = c0[i] + ai;
      }
      wgt[a] = w;
      nid[a] = node_id<D>(gl, xc);
    }
    for (int r = 0; r < nr; r++) {
      const double* xi = A.X + P.vec_off + (int64_t)r * nnl;
      double v = 0.0;
#pragma unroll
      for (int a = 0; a < (1 << D); a++)
        if (wgt[a] != 0.0) v += wgt[a] * xi[nid[a]];
      double* I = A.FI + P.fine_off + (int64_t)r * nnf;
      const double phi = I[k] + v;
      I[k] = phi;
      if (P.pool_off >= 0) A.pool[P.pool_off + (int64_t)r * nnf + k] = phi;
    }
  }
}

// ---------------------------------------------------------------------------------------
// Gram / Eq. (7): one CTA per macropoint
template <int D>
__global__ void k_gram(LevelArgs A) {
  const int mp = blockIdx.x;
  const ProbDesc& P = A.probs[mp];
  const Geo<D> gf = fine_geo<D>(P);
  __shared__ double scratch[32 * 16];
  __shared__ double tot[16];
  const int nr = A.n_rhs;
  int ext[3] = {1, 1, 1}, lo[3] = {0, 0, 0};
  for (int i = 0; i < D; i++) {
    lo[i] = P.kp_lo[i] - P.lo[i];
    ext[i] = P.kp_hi[i] - P.kp_lo[i];
  }
  const int cnt = ext[0] * ext[1] * ext[2];
  // fused 3D path (fine3d.cu): phi on the K_p node box in FK
  const bool kpl = (D == 3) && A.level >= 2 && A.FK != nullptr;
  const int kn0 = ext[0] + 1, kn1 = ext[1] + 1;
  auto field = [&](int rr) -> const double* {
    if (A.level == 1) return A.X + P.vec_off + (int64_t)rr * gf.nnodes;
    if (kpl) return A.FK + ((int64_t)mp * nr + rr) * A.nkp_max;
    return A.FI + P.fine_off + (int64_t)rr * gf.nnodes;
  };
  auto nodeid = [&](const int* xb) {
    return kpl ? ((xb[2] - lo[2]) * kn1 + (xb[1] - lo[1])) * kn0 + (xb[0] - lo[0]) : node_id<D>(gf, xb);
  };
  double* Gout = A.G + P.lin * nr * nr;
  for (int a = 0; a < nr; a++) {
    double v[16];
    for (int i = 0; i < 16; i++) v[i] = 0.0;
    const double* fa = field(a);
    for (int idx = threadIdx.x; idx < cnt; idx += blockDim.x) {
      int e[3] = {lo[0] + idx % ext[0], lo[1] + (idx / ext[0]) % ext[1], lo[2] + idx / (ext[0] * ext[1])};
      double W[DimC<D>::NW];
      elem_W<D>(A, P, gf, e, W);
      int nid[1 << D];
      double ca[1 << D];
      for (int bb = 0; bb < (1 << D); bb++) {
        int xb[3] = {e[0] + (bb & 1), e[1] + ((bb >> 1) & 1), (D == 3) ? e[2] + ((bb >> 2) & 1) : 0};
        nid[bb] = nodeid(xb);
        ca[bb] = fa[nid[bb]];
      }
      // K_E phi_a (all corners), then dot with phi_b
      double ka[1 << D];
      for (int c = 0; c < (1 << D); c++) ka[c] = elem_row<D>(W, ca, c);
      for (int b = a; b < nr; b++) {
        const double* fb = field(b);
        double s = 0.0;
        for (int c = 0; c < (1 << D); c++) s += ka[c] * fb[nid[c]];
        v[b - a] += s;
      }
    }
    block_sum<16>(v, scratch, tot);
    if (threadIdx.x == 0) {
      for (int b = a; b < nr; b++) {
        Gout[a * nr + b] = tot[b - a];
        Gout[b * nr + a] = tot[b - a];
      }
    }
    __syncthreads();
  }
  // load vectors (NEXT-2, Eq. 7 with R_p = K_p): f cellwise constant and
  // phi_j Q1 on the fine grid, so int_e f phi_j = f_e (h^D / 2^D) sum_{corners} phi_j, exactly
  if (A.f == nullptr) return;
  double v[16];
  for (int i = 0; i < 16; i++) v[i] = 0.0;
  const int N = A.N;
  for (int idx = threadIdx.x; idx < cnt; idx += blockDim.x) {
    int e[3] = {lo[0] + idx % ext[0], lo[1] + (idx / ext[0]) % ext[1], lo[2] + idx / (ext[0] * ext[1])};
    int64_t gl = 0;
    for (int i = D - 1; i >= 0; i--) gl = gl * A.n + (P.lo[i] + e[i]);
    const double fe = A.f[gl];
    for (int j = 0; j < N; j++) {
      const double* fj = field(j);
      double s = 0.0;
      for (int bb = 0; bb < (1 << D); bb++) {
        int xb[3] = {e[0] + (bb & 1), e[1] + ((bb >> 1) & 1), (D == 3) ? e[2] + ((bb >> 2) & 1) : 0};
        s += fj[nodeid(xb)];
      }
      v[j] += fe * s;
    }
  }
  block_sum<16>(v, scratch, tot);
  if (threadIdx.x == 0) {
    const double wq = (D == 2) ? A.h * A.h * 0.25 : A.h * A.h * A.h * 0.125;
    for (int j = 0; j < N; j++) A.bload[P.lin * N + j] = tot[j] * wq;
  }
}

// ---------------------------------------------------------------------------------------
// input validation: kappa > 0 finite, ids < N
__global__ void k_validate(const double* kappa, const uint8_t* ids, int64_t cnt, int N, int* bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x) {
    const double k = kappa[i];
    if (!(k > 0.0) || !isfinite(k) || ids[i] >= N) atomicOr(bad, 1);
  }
}

// 64-bit fingerprint of the medium (checkpoints: the file does not hold kappa / ids): wrapping sum of
// per-cell mixed words, order-independent and so reproducible for any grid
__global__ void k_fingerprint(const double* kappa, const uint8_t* ids, int64_t cnt, unsigned long long* out) {
  unsigned long long acc = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long v = (unsigned long long)__double_as_longlong(kappa[i]);
    v ^= ((unsigned long long)ids[i] + 1ull) * 0x9E3779B97F4A7C15ull;
    v += (unsigned long long)i * 0xD6E8FEB86659FD93ull;
    v ^= v >> 32;
    v *= 0xD6E8FEB86659FD93ull;
    v ^= v >> 29;
    acc += v;
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(FULLMASK, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, acc);
}

cudaError_t launch_fingerprint(const double* kappa, const uint8_t* ids, int64_t cnt, unsigned long long* out,
                               cudaStream_t st) {
  const unsigned grid = (unsigned)std::min<int64_t>((cnt + 255) / 256, 148 * 8);
  k_fingerprint<<<grid, 256, 0, st>>>(kappa, ids, cnt, out);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// host launchers
size_t pcg_smem(const LevelArgs& A) {
  const size_t nc = A.ncon;
  const size_t mat = (A.band > 0) ? nc * (A.band + 1) + nc : nc * nc + 32 * nc;
  const size_t crs = A.coarse ? 2 * (size_t)A.ncmax : 0;
  return sizeof(double) * (mat + 5 * nc + crs + 32 * 4 + 4) + sizeof(int) * (A.nsub * 7 + 2);
}

size_t proj_setup_band_smem(const LevelArgs& A) {
  const size_t nc = A.ncon;
  return sizeof(double) * (nc * (A.band + 1) + nc + 32 * 16 + 16) + sizeof(int) * (A.nsub * 7 + 2);
}

cudaError_t launch_level_ops(const LevelArgs& A, cudaStream_t st) {
  const int64_t ncell = (A.D == 2) ? (int64_t)A.gn * A.gn : (int64_t)A.gn * A.gn * A.gn;
  const int bs = 128;
  const unsigned grid = (unsigned)((ncell + bs - 1) / bs);
  if (A.D == 2) k_level_ops<2><<<grid, bs, 0, st>>>(A);
  else k_level_ops<3><<<grid, bs, 0, st>>>(A);
  return cudaGetLastError();
}

cudaError_t launch_targets(const LevelArgs& A, cudaStream_t st) {
  if (A.D == 2) k_targets<2><<<A.nprob_mp, 256, 0, st>>>(A);
  else k_targets<3><<<A.nprob_mp, 256, 0, st>>>(A);
  return cudaGetLastError();
}

cudaError_t launch_transport(const LevelArgs& A, int threads, cudaStream_t st) {
  const bool generic = getenv("MCH_TRANSPORT_GENERIC") != nullptr;  // read per call (tests toggle it)
  // the multi-rhs kernel has one CTA per macropoint: below two per SM the per-(macropoint, rhs)
  // kernel fills the GPU better (config 2 level 2, 208 macropoints: 0.50 vs 0.41 ms)
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const bool force_mr = getenv("MCH_TRANSPORT_MR") != nullptr;  // tests: the multi-rhs kernel at any size
  // 3D: its fine windows are 8x larger per macropoint; from eight macropoints per SM up (config 5
  // level 4: 332 -> 306 ms; level 3, 604 macropoints: 66 -> 71 ms, kept per rhs)
  if (A.D == 3 && A.tphase != 0 && A.n_rhs <= kMaxR && (force_mr || A.nprob_level >= 8 * sms)) {
    k_transport3d_mr<<<(unsigned)A.nprob_mp, 256, 0, st>>>(A);
    return cudaGetLastError();
  }
  if (A.D == 2 && A.band == 0 && A.tphase == 0 && !generic && (force_mr || A.nprob_level >= 2 * sms) &&
      (A.n_rhs == 3 || A.n_rhs == 6 || A.n_rhs == 9)) {
    const size_t sm = sizeof(double) * ((A.nsub * 7 + 2 + 1) / 2 + (size_t)8 * A.ncon * A.n_rhs);
    if (sm <= 232448) {
      auto k = (A.n_rhs == 3) ? k_transport2d_mr<3> : ((A.n_rhs == 6) ? k_transport2d_mr<6> : k_transport2d_mr<9>);
      cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      if (e != cudaSuccess) return e;
      k<<<(unsigned)A.nprob_mp, 256, sm, st>>>(A);
      return cudaGetLastError();
    }
  }
  const size_t sm = sizeof(double) * ((A.nsub * 7 + 2 + 1) / 2 + (A.band > 0 ? 0 : 32 * A.ncon) + A.ncon);
  const unsigned grid = (unsigned)A.nprob_mp * A.n_rhs;
  if (A.D == 2) k_transport<2><<<grid, threads, sm, st>>>(A);
  else k_transport<3><<<grid, threads, sm, st>>>(A);
  return cudaGetLastError();
}

cudaError_t launch_proj_setup(const LevelArgs& A, int threads, cudaStream_t st) {
  if (A.band > 0) {
    if (A.D != 2) return cudaErrorInvalidValue;
    const size_t sm = proj_setup_band_smem(A);
    cudaError_t e = cudaFuncSetAttribute(k_proj_setup_band<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    k_proj_setup_band<2><<<A.nprob_mp, threads, sm, st>>>(A);
    return cudaGetLastError();
  }
  const size_t sm = sizeof(double) * (2 * (size_t)A.ncon * A.ncon + 32 * 16 + 16 + (A.nsub * 7 + 2 + 1) / 2 + 2 +
                                       (A.coarse ? (size_t)(A.ncon + 1) * A.ncmax : 0));
  cudaError_t e;
  if (A.D == 2) {
    e = cudaFuncSetAttribute(k_proj_setup<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_proj_setup<2><<<A.nprob_mp, threads, sm, st>>>(A);
  } else {
    e = cudaFuncSetAttribute(k_proj_setup<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_proj_setup<3><<<A.nprob_mp, threads, sm, st>>>(A);
  }
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_pinv(const LevelArgs& A, cudaStream_t st) {
  if (A.band > 0) return cudaSuccess;  // the banded projector reports dependent rows instead (flag 8)
  const int m = (A.ncon + 1) & ~1;
  if (m > 128) return cudaErrorInvalidValue;

  const size_t sm = sizeof(double) * (2 * (size_t)m * m + 128) + sizeof(int) * ((size_t)m + 128);
  cudaError_t e = cudaFuncSetAttribute(k_pinv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  const size_t smc = sizeof(double) * 3 * (size_t)A.ncon * A.ncon + sizeof(int) * (size_t)A.ncon;
  e = cudaFuncSetAttribute(k_pinv_chol, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smc);
  if (e != cudaSuccess) return e;
  if (getenv("MCH_PINV_JACOBI")) k_pinv_all_jacobi<<<(A.nprob_mp + 255) / 256, 256, 0, st>>>(A);  // dev A/B
  else k_pinv_chol<<<A.nprob_mp, 256, smc, st>>>(A);
  k_pinv<<<A.nprob_mp, 256, sm, st>>>(A);
  return cudaGetLastError();
}

cudaError_t launch_pcg(const LevelArgs& A, int threads, cudaStream_t st) {
  const size_t sm = pcg_smem(A);
  const unsigned grid = (unsigned)A.nprob_mp * A.n_rhs;
  cudaError_t e;
  if (A.D == 2) {
    e = cudaFuncSetAttribute(k_pcg<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_pcg<2><<<grid, threads, sm, st>>>(A);
  } else {
    e = cudaFuncSetAttribute(k_pcg<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_pcg<3><<<grid, threads, sm, st>>>(A);
  }
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_combine(const LevelArgs& A, int threads, cudaStream_t st) {
  int dev = 0, sms = 148;  // one CTA per macropoint once there are two per SM (as the transport)
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (getenv("MCH_TRANSPORT_MR") != nullptr || (A.nprob_level >= 2 * sms && getenv("MCH_TRANSPORT_GENERIC") == nullptr)) {
    if (A.D == 2) k_combine_mr<2><<<(unsigned)A.nprob_mp, 256, 0, st>>>(A);
    else k_combine_mr<3><<<(unsigned)A.nprob_mp, 256, 0, st>>>(A);
    return cudaGetLastError();
  }
  const unsigned grid = (unsigned)A.nprob_mp * A.n_rhs;
  if (A.D == 2) k_combine<2><<<grid, threads, 0, st>>>(A);
  else k_combine<3><<<grid, threads, 0, st>>>(A);
  return cudaGetLastError();
}

cudaError_t launch_gram(const LevelArgs& A, int threads, cudaStream_t st) {
  if (A.D == 2) k_gram<2><<<A.nprob_mp, threads, 0, st>>>(A);
  else k_gram<3><<<A.nprob_mp, threads, 0, st>>>(A);
  return cudaGetLastError();
}

cudaError_t launch_validate(const double* kappa, const uint8_t* ids, int64_t cnt, int N, int* bad, cudaStream_t st) {
  k_validate<<<592, 256, 0, st>>>(kappa, ids, cnt, N, bad);
  return cudaGetLastError();
}
