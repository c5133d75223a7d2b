// On-chip projected PCG for 2D windows (sm_100a) and its per-node setup.
//
// Same method as k_pcg (kernels.cu): for each problem (macropoint p, right-hand side r) the
// constrained minimisation  min 1/2 x^T A x - b^T x  s.t.  C x = g  of Eqs. (3)/(4) (level 1,
// PAPER.md:145-170) or of the correction problems of Eqs. (12)/(13) (levels >= 2,
// PAPER.md:392-419), solved by projected Jacobi-PCG with the residual re-projected every
// iteration (readings R16, R19).  What differs is where the state lives:
//
//   p          shared memory, zero halo (the 9-point stencil reads neighbours)
//   r          registers: every thread owns a run of RPT consecutive nodes of one column
//   q, x       tensor memory (TMEM as a register-file extension: tcgen05.st / tcgen05.ld 32x32b)
//   D^-1       shared memory, fp32-rounded (the projector setup used the same rounded values, so
//              the projection stays exact in the D^-1 metric)
//   level 1    kappa and continuum ids of the window's cells in shared memory; the Q1 stencil
//               and the constraint weights m_{E,j,a} = [id_E = j] h^2/4 are
//              formed on the fly from a sliding 2x2 cell window
//   level >= 2 per-node stencil rows of A_n = P_n^T A_1 P_n (reading R11) and constraint weights,
//              precomputed by k_node_ops2d (L2 resident, shared by the right-hand sides)
//
// One CTA per problem, three block barriers per iteration.  The constraint vector
// c = C D^-1 r is reduced per warp with a segmented scan keyed by subcell column, then summed
// over warps in a fixed order, so every run gives bitwise identical results.
//
// Thread layout: warp w handles column band wx = w % WX (32 node columns) of row chunk w / WX.
// Row chunks never straddle a subcell row (host plan, mch.cu): only the first row of the first
// chunk of a subcell row touches elements of the previous subcell row ("interface row").
#include <cuda_runtime.h>

#include "device_common.cuh"
#include "kernels.h"

namespace {

// ------------------------------------------------------------------------------------------
// TMEM helpers (32x32b shape: lane i of the warp <-> TMEM lane 32*(warp%4) + i)
__device__ __forceinline__ void tm_st2(uint32_t ta, double v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};\n" ::"r"(ta),
               "r"(__double2loint(v)), "r"(__double2hiint(v)));
}
__device__ __forceinline__ void tm_ld4(uint32_t ta, uint32_t (&v)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
               : "r"(ta));
}
// (no "memory" clobbers on the per-row TMEM asm: they would pin every address-taken local in
// local memory; volatile asm statements keep their relative order)
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n"); }
__device__ __forceinline__ double dbl(uint32_t lo, uint32_t hi) { return __hiloint2double((int)hi, (int)lo); }
// compiler-only fence between unrolled rows: keeps ptxas from hoisting every row's loads to the
// top of the sweep (which needs ~250 registers); latency is hidden by the other warps instead
__device__ __forceinline__ void row_fence() {}
// An opaque copy of v: values derived from it cannot be hoisted out of the CG loop (otherwise
// ptxas precomputes every row address of every sweep once and keeps them all live).
__device__ __forceinline__ int opaque(int v) {
  int r;
  asm volatile("mov.b32 %0, %1;\n" : "=r"(r) : "r"(v));
  return r;
}

// warp sum, reduced to lane 0 in a fixed tree and broadcast (identical in every lane and warp)
__device__ __forceinline__ double warp_sum0(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(FULLMASK, v, o);
  return __shfl_sync(FULLMASK, v, 0);
}

// y_lane = sum_j Sinv[lane][j] c_j with c_j held by lane j (Sinv symmetric: read column-wise)
__device__ __forceinline__ double warp_sinv(const double* Si, int nc, double cv) {
  const int lane = threadIdx.x & 31;
  double y = 0.0;
  for (int j = 0; j < nc; j++) {
    const double cj = __shfl_sync(FULLMASK, cv, j);
    if (lane < nc) y += Si[j * nc + lane] * cj;
  }
  return y;
}

__device__ __forceinline__ int sub_slot(const LevelArgs& A, const ProbDesc& P, int dim, int e) {
  return fdiv(P.lo[dim] + e * A.s + A.c / 2, A.inv_c) - P.k[dim] + A.l;
}

// Constraint weights of one node, by side (L: elements of column x-1, R: column x) summed over
// the lower (row y-1) and upper (row y) elements, and the lower element alone (interface rows).
template <int N, bool L1OP, int KX>
struct NodeW {
  // level 1: continuum ids of the window cells (border 0xFF), pitch KX
  const uint8_t* ids;
  double hq, hq2;
  uint8_t dL, dR;
  // levels >= 2: precomputed SoA [4N][nn]
  const double* base;
  int nn, nx;
  int xc;
  const uint8_t* ip;  // running row pointers
  const double* mp;
  int hqhi, hqlo;     // bit pattern of hq = h^2/4 (level-1 weight of one element corner)

  // c * hq for c in {0, 1, 2}, branch-free on the bit pattern (hq is a normal double, so
  // 2 hq is hq with the exponent incremented)
  __device__ __forceinline__ double cnt_w(int c) const {
    const int m = -(c != 0);
    return __hiloint2double((hqhi + ((c - 1) << 20)) & m, hqlo & m);
  }

  __device__ __forceinline__ void start(int y0) {
    if (L1OP) {
      ip = ids + y0 * KX + xc;
      dL = ip[0];
      dR = ip[1];
    } else {
      mp = base + y0 * nx + xc;
    }
  }
  // node (x, y0 + i) for consecutive i
  __device__ __forceinline__ void row(bool low, double (&mL)[N], double (&mR)[N], double (&lL)[N],
                                      double (&lR)[N]) {
    if (L1OP) {
      ip += KX;
      const uint8_t uL = ip[0], uR = ip[1];
#pragma unroll
      for (int j = 0; j < N; j++) {
        mL[j] = cnt_w((dL == j) + (uL == j));
        mR[j] = cnt_w((dR == j) + (uR == j));
        lL[j] = cnt_w(dL == j);
        lR[j] = cnt_w(dR == j);
      }
      dL = uL;
      dR = uR;
    } else {
#pragma unroll
      for (int j = 0; j < N; j++) {
        mL[j] = __ldg(mp + (int64_t)j * nn);
        mR[j] = __ldg(mp + (int64_t)(N + j) * nn);
        lL[j] = low ? __ldg(mp + (int64_t)(2 * N + j) * nn) : 0.0;
        lR[j] = low ? __ldg(mp + (int64_t)(3 * N + j) * nn) : 0.0;
      }
      mp += nx;
    }
  }
};

}  // namespace

// ------------------------------------------------------------------------------------------
// levels >= 2 (and, for cross-checks, level 1): per-node stencil rows and constraint weights of
// every window of the batch.  grid (ceil(max nodes / 128), macropoints)
template <int N>
__global__ void k_node_ops2d(LevelArgs A) {
  const int mp = blockIdx.y;
  const ProbDesc& P = A.probs[mp];
  const Geo<2> g = level_geo<2>(A, P);
  const int nx = g.nn[0], nn = g.nnodes;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nn) return;
  const int y = k / nx, x = k - y * nx;
  double st[9];
  double mL[N], mR[N], lL[N], lR[N];
  for (int i = 0; i < 9; i++) st[i] = 0.0;
  for (int j = 0; j < N; j++) mL[j] = mR[j] = lL[j] = lR[j] = 0.0;
  for (int o = 0; o < 4; o++) {
    const int ox = o & 1, oy = o >> 1;
    int e[3] = {x - 1 + ox, y - 1 + oy, 0};
    if (e[0] < 0 || e[0] >= g.nc[0] || e[1] < 0 || e[1] >= g.nc[1]) continue;
    double W[DimC<2>::NW];
    elem_W<2>(A, P, g, e, W);
    const int a = (1 - ox) + 2 * (1 - oy);  // corner of node k in element e
    for (int b = 0; b < 4; b++) {
      double c[4] = {0.0, 0.0, 0.0, 0.0};
      c[b] = 1.0;
      const int dx = e[0] + (b & 1) - x, dy = e[1] + (b >> 1) - y;
      st[(dy + 1) * 3 + (dx + 1)] += elem_row<2>(W, c, a);
    }
    for (int j = 0; j < N; j++) {
      const double m = elem_m<2>(A, P, g, e, j, a);
      if (ox == 0) {
        mL[j] += m;
        if (oy == 0) lL[j] += m;
      } else {
        mR[j] += m;
        if (oy == 0) lR[j] += m;
      }
    }
  }
  double* so = A.STC + P.node_off * 9;
  for (int c = 0; c < 9; c++) so[(int64_t)c * nn + k] = st[c];
  double* mo = A.MLR + P.node_off * 4 * N;
  for (int j = 0; j < N; j++) {
    mo[(int64_t)j * nn + k] = mL[j];
    mo[(int64_t)(N + j) * nn + k] = mR[j];
    mo[(int64_t)(2 * N + j) * nn + k] = lL[j];
    mo[(int64_t)(3 * N + j) * nn + k] = lR[j];
  }
}

// ------------------------------------------------------------------------------------------
// the solver: one CTA per problem (macropoint, rhs)
template <int RPT, int N, bool L1OP>
__global__ void __launch_bounds__(L1OP ? 768 : 384, L1OP ? 1 : 2) k_pcg2d(LevelArgs A) {
  constexpr int NBC = 4 * RPT;  // TMEM columns per thread: (q, x) per row
  // compile-time pitches (host checks nx <= NXM): per-row addresses become immediate offsets
  constexpr int NXM = L1OP ? PCG2D_NXMAX_L1 : PCG2D_NXMAX_GN;
  constexpr int PX = NXM + 2, KX = NXM + 1, DX = NXM;
  const int prob = blockIdx.x;
  const int mp = prob / A.n_rhs, rhs = prob - mp * A.n_rhs;
  const ProbDesc& P = A.probs[mp];
  const int nx = P.nc[0] + 1, ny = P.nc[1] + 1, nn = nx * ny;
  const int ncx = nx - 1, ncy = ny - 1;
  const int nc = A.ncon, ws = A.w;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int WX = (nx + 31) >> 5;
  const int sgi = warp / WX, wx = warp - sgi * WX;
  const bool wact = sgi < A.nseg[mp];
  const int x = wx * 32 + lane;
  const bool lact = wact && x < nx;
  const int xc = min(x, nx - 1);
  short4 sg = make_short4(0, 0, 0, -1);
  if (wact) sg = A.segs[mp * A.maxseg + sgi];
  const int y0 = sg.x, nrow = sg.y, sy = sg.z, syp = sg.w;

  extern __shared__ __align__(16) double smem[];
  double* Si = smem;                      // nc*nc
  double* Yw = Si + nc * nc;              // [nwarps][32] projector coefficients yhat, per warp
  double* bins = Yw + nwarps * 32;        // [nwarps][32] constraint partial sums, per warp
  double* slots = bins + nwarps * 32;     // [3][32] scalar partial sums (rz, pq, rr)
  double* p_s = slots + 3 * 32;           // (nx+2)(ny+2)
  double* kap_s = p_s + PX * (ny + 2);    // level 1: (nx+1)(ny+1)
  float* dinv_s = reinterpret_cast<float*>(kap_s + (L1OP ? KX * (ny + 1) : 0));  // DX*ny
  uint8_t* ids_s = reinterpret_cast<uint8_t*>(dinv_s + DX * ny);
  __shared__ uint32_t tm_base_s;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tm_base_s)),
                 "r"(A.tm_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  for (int i = threadIdx.x; i < PX * (ny + 2); i += blockDim.x) p_s[i] = 0.0;
  for (int i = threadIdx.x; i < nc * nc; i += blockDim.x) Si[i] = A.Sinv[(int64_t)mp * nc * nc + i];
  for (int i = threadIdx.x; i < nwarps * 32; i += blockDim.x) {
    bins[i] = 0.0;
    Yw[i] = 0.0;
  }
  {
    const double* dg = A.dinv + P.node_off;
    for (int k = threadIdx.x; k < nn; k += blockDim.x) dinv_s[(k / nx) * DX + k % nx] = (float)dg[k];
  }
  if (L1OP) {
    for (int i = threadIdx.x; i < KX * (ny + 1); i += blockDim.x) {
      const int ey = i / KX - 1, ex = i - (ey + 1) * KX - 1;
      double kv = 0.0;
      uint8_t id = 0xFF;
      if (ex >= 0 && ex < ncx && ey >= 0 && ey < ncy) {
        const int64_t f = (int64_t)(P.lo[1] + ey) * A.n + (P.lo[0] + ex);
        kv = A.kappa[f];
        id = A.ids[f];
      }
      kap_s[i] = kv;
      ids_s[i] = id;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tm = tm_base_s + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * NBC);

  // per-thread subcell columns of the left / right elements
  const int sxL = (xc >= 1) ? sub_slot(A, P, 0, xc - 1) : 0;
  const int sxR = (xc < ncx) ? sub_slot(A, P, 0, xc) : 0;
  NodeW<N, L1OP, KX> cw;
  cw.ids = ids_s;
  cw.hq = 0.25 * A.h * A.h;
  cw.hq2 = 0.5 * A.h * A.h;
  cw.hqhi = __double2hiint(cw.hq);
  cw.hqlo = __double2loint(cw.hq);
  cw.base = A.MLR + P.node_off * 4 * N;
  cw.nn = nn;
  cw.nx = nx;
  cw.xc = xc;
  const double* S9 = A.STC + P.node_off * 9;

  auto Pref = [&](int yy, int xx) -> double& { return p_s[(yy + 1) * PX + (xx + 1)]; };
  auto Kld = [&](int ey, int ex) { return kap_s[(ey + 1) * KX + (ex + 1)]; };
  auto dinv = [&](int y) { return (double)dinv_s[y * DX + xc]; };

  double r[RPT];
#pragma unroll
  for (int i = 0; i < RPT; i++) r[i] = 0.0;

  // ---- C^T yhat per row: f(i, y, ct) -------------------------------------------------------
  auto sweep_ct = [&](auto&& f) {
    const double* Y = Yw + warp * 32;
    double YL[N], YR[N];
#pragma unroll
    for (int j = 0; j < N; j++) {
      YL[j] = Y[(sy * ws + sxL) * N + j];
      YR[j] = Y[(sy * ws + sxR) * N + j];
    }
    const int yb = opaque(y0);
    cw.start(yb);
#pragma unroll
    for (int i = 0; i < RPT; i++) {
      if (i < nrow) {
        const int y = yb + i;
        const bool split = (i == 0) && (syp >= 0);
        double mL[N], mR[N], lL[N], lR[N];
        cw.row(split, mL, mR, lL, lR);
        double ct = 0.0;
        if (split) {
#pragma unroll
          for (int j = 0; j < N; j++) {
            const double YLp = Y[(syp * ws + sxL) * N + j], YRp = Y[(syp * ws + sxR) * N + j];
            ct += lL[j] * YLp + (mL[j] - lL[j]) * YL[j] + lR[j] * YRp + (mR[j] - lR[j]) * YR[j];
          }
        } else {
#pragma unroll
          for (int j = 0; j < N; j++) ct += mL[j] * YL[j] + mR[j] * YR[j];
        }
        f(i, y, ct);
      }
      row_fence();
    }
  };

  // ---- (A p)_k per row from the smem vector p_s: f(i, y, Ap, p_k) ----------------------------
  auto sweep_stencil = [&](auto&& f) {
    const int yb = opaque(y0);
    double a0 = Pref(yb - 1, xc - 1), b0 = Pref(yb - 1, xc), c0 = Pref(yb - 1, xc + 1);
    double a1 = Pref(yb, xc - 1), b1 = Pref(yb, xc), c1 = Pref(yb, xc + 1);
    double kL0 = 0.0, kR0 = 0.0;
    if (L1OP) {
      kL0 = Kld(yb - 1, xc - 1);
      kR0 = Kld(yb - 1, xc);
    }
    const double* s9 = S9 + yb * nx + xc;
#pragma unroll
    for (int i = 0; i < RPT; i++) {
      if (i < nrow) {
        const int y = yb + i;
        const double a2 = Pref(y + 1, xc - 1), b2 = Pref(y + 1, xc), c2 = Pref(y + 1, xc + 1);
        double Ap;
        if (L1OP) {
          // Q1 element rows kappa/6 (4 v_a - v_a^1 - v_a^2 - 2 v_a^3) summed over the 4 cells
          const double kL1 = Kld(y, xc - 1), kR1 = Kld(y, xc);
          const double sL = kL0 + kL1, sR = kR0 + kR1, sD = kL0 + kR0, sU = kL1 + kR1;
          double acc = 4.0 * (sL + sR) * b1 - sR * c1 - sL * a1 - sU * b2 - sD * b0;
          acc -= 2.0 * (kR1 * c2 + kL1 * a2 + kR0 * c0 + kL0 * a0);
          Ap = acc * (1.0 / 6.0);
          kL0 = kL1;
          kR0 = kR1;
        } else {
          const double* s = s9;
          s9 += nx;
          Ap = __ldg(s) * a0 + __ldg(s + nn) * b0 + __ldg(s + 2 * nn) * c0 + __ldg(s + 3 * nn) * a1 +
               __ldg(s + 4 * nn) * b1 + __ldg(s + 5 * nn) * c1 + __ldg(s + 6 * nn) * a2 +
               __ldg(s + 7 * nn) * b2 + __ldg(s + 8 * nn) * c2;
        }
        f(i, y, Ap, b1);
        a0 = a1; b0 = b1; c0 = c1;
        a1 = a2; b1 = b2; c1 = c2;
      }
      row_fence();
    }
  };

  // ---- constraint accumulation: aC (current subcell row), aP (previous, interface row) -------
  double aC[2][N], aP[2][N];
  auto acc_zero = [&]() {
#pragma unroll
    for (int j = 0; j < N; j++) aC[0][j] = aC[1][j] = aP[0][j] = aP[1][j] = 0.0;
  };
  auto acc_row = [&](int i, int y, double u, const double (&mL)[N], const double (&mR)[N],
                     const double (&lL)[N], const double (&lR)[N]) {
    if (i == 0 && syp >= 0) {
#pragma unroll
      for (int j = 0; j < N; j++) {
        aP[0][j] += lL[j] * u;
        aP[1][j] += lR[j] * u;
        aC[0][j] += (mL[j] - lL[j]) * u;
        aC[1][j] += (mR[j] - lR[j]) * u;
      }
    } else {
#pragma unroll
      for (int j = 0; j < N; j++) {
        aC[0][j] += mL[j] * u;
        aC[1][j] += mR[j] * u;
      }
    }
  };
  // warp part of the c reduction: bins[warp][(sy*w + sx)*N + j]
  auto c_reduce = [&]() {
    double* B = bins + warp * 32;
    B[lane] = 0.0;
    __syncwarp();
    double cC[N], cP[N];
#pragma unroll
    for (int j = 0; j < N; j++) {
      // element column x-1 (left side) is the right side of lane-1
      const double tC = __shfl_down_sync(FULLMASK, aC[0][j], 1);
      const double tP = __shfl_down_sync(FULLMASK, aP[0][j], 1);
      cC[j] = aC[1][j] + ((lane < 31) ? tC : 0.0);
      cP[j] = aP[1][j] + ((lane < 31) ? tP : 0.0);
    }
    const int key = (lact && x < ncx) ? sxR : 1000;
    const int kup = __shfl_up_sync(FULLMASK, key, 1);
    const unsigned hm = __ballot_sync(FULLMASK, lane == 0 || key != kup);
    const int head = 31 - __clz(hm & (0xffffffffu >> (31 - lane)));
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
      for (int j = 0; j < N; j++) {
        const double tC = __shfl_up_sync(FULLMASK, cC[j], d);
        const double tP = __shfl_up_sync(FULLMASK, cP[j], d);
        if (lane - d >= head) {
          cC[j] += tC;
          cP[j] += tP;
        }
      }
    }
    const bool tail = (lane == 31) || ((hm >> (lane + 1)) & 1u);
    if (tail && key < 1000) {
#pragma unroll
      for (int j = 0; j < N; j++) {
        B[(sy * ws + key) * N + j] = cC[j];
        if (syp >= 0) B[(syp * ws + key) * N + j] = cP[j];
      }
    }
    __syncwarp();
    if (lane == 0 && lact && x >= 1) {  // left side of lane 0 belongs to the previous warp's band
#pragma unroll
      for (int j = 0; j < N; j++) {
        B[(sy * ws + sxL) * N + j] += aC[0][j];
        if (syp >= 0) B[(syp * ws + sxL) * N + j] += aP[0][j];
      }
    }
  };
  auto fin_c = [&]() -> double {
    double s = 0.0;
    if (lane < nc)
      for (int w2 = 0; w2 < nwarps; w2++) s += bins[w2 * 32 + lane];
    return s;
  };
  auto put_y = [&](double yv) {
    Yw[warp * 32 + lane] = (lane < nc) ? yv : 0.0;
    __syncwarp();
  };
  auto slot_put = [&](int which, double v) {
    v = warp_sum0(v);
    if (lane == 0) slots[which * 32 + warp] = v;
  };
  auto slot_fin = [&](int which) { return warp_sum0((lane < nwarps) ? slots[which * 32 + lane] : 0.0); };

  // ---- init: x0 = D^-1 C^T S^-1 t (minimum-norm feasible point), r0 = A x0 - b,
  //      c = C D^-1 r0, yhat = S^-1 c; returns r0^T D^-1 r0 -----------------------------------
  const bool lev2 = !L1OP && A.level >= 2;  // the level-1 variant is only launched at level 1
  const double* bvec = lev2 ? A.B + P.vec_off + (int64_t)rhs * nn : nullptr;
  auto init = [&](double tval) -> double {
    put_y(warp_sinv(Si, nc, tval));
    if (wact) {
      sweep_ct([&](int i, int y, double ct) {
        const double x0 = dinv(y) * ct;
        if (lact) Pref(y, x) = x0;
        tm_st2(tm + 4 * i + 2, x0);
      });
      tm_wait_st();
    }
    __syncthreads();
    double rr = 0.0;
    if (wact) {
      sweep_stencil([&](int i, int y, double Ap, double) {
        r[i] = lact ? Ap - (bvec ? bvec[y * nx + xc] : 0.0) : 0.0;
      });
      acc_zero();
      const int yb = opaque(y0);
      cw.start(yb);
#pragma unroll
      for (int i = 0; i < RPT; i++) {
        if (i < nrow) {
          const int y = yb + i;
          double mL[N], mR[N], lL[N], lR[N];
          cw.row(i == 0 && syp >= 0, mL, mR, lL, lR);
          const double u = dinv(y) * r[i];
          rr += r[i] * u;
          acc_row(i, y, u, mL, mR, lL, lR);
        }
        row_fence();
      }
      c_reduce();
    }
    slot_put(2, rr);
    __syncthreads();
    rr = slot_fin(2);
    put_y(warp_sinv(Si, nc, fin_c()));
    return rr;
  };

  const double* gsrc = lev2 ? A.g : A.g0;
  const double gcol = (lane < nc) ? gsrc[((int64_t)mp * nc + lane) * A.n_rhs + rhs] : 0.0;
  double rz_ref = 0.0, rr_ref = 0.0;
  if (lev2) {
    // reference scale: initial projected residual of the full (non-hierarchical) problem
    const double g0c = (lane < nc) ? A.g0[((int64_t)mp * nc + lane) * A.n_rhs + rhs] : 0.0;
    const double* bsave = bvec;
    bvec = nullptr;
    rr_ref = init(g0c);
    bvec = bsave;
    double v = 0.0;
    if (wact) {
      sweep_ct([&](int i, int y, double ct) {
        const double w = r[i] - ct;
        v += lact ? dinv(y) * w * w : 0.0;
      });
    }
    slot_put(0, v);
    __syncthreads();
    rz_ref = slot_fin(0);
  }
  const double rr0 = init(gcol);

  const double tol2 = A.rtol * A.rtol;
  const double floor2 = 1e-30 * fmax(rr0, rr_ref);
  double beta = 0.0, rz = 0.0, ref = 0.0;
  int it = 0, breakdown = 0;
  for (;; it++) {
    // pass A: r <- r - C^T yhat (re-projection), z = D^-1 r, p <- -z + beta p, rz = r.z
    double v = 0.0;
    if (wact) {
      const bool first = (it == 0);
      sweep_ct([&](int i, int y, double ct) {
        const double rk = lact ? r[i] - ct : 0.0;
        r[i] = rk;
        const double z = dinv(y) * rk;
        if (lact) {
          double& pk = Pref(y, x);
          pk = first ? -z : -z + beta * pk;
        }
        v += rk * z;
      });
    }
    slot_put(0, v);
    __syncthreads();  // B1: p complete
    rz = slot_fin(0);
    if (it == 0) ref = fmax(rz, rz_ref);
    if (!(rz > fmax(tol2 * ref, floor2)) || it >= A.max_iter) break;
    // pass B: q = A p, pq
    double w = 0.0;
    if (wact) {
      sweep_stencil([&](int i, int y, double Ap, double pk) {
        w += lact ? pk * Ap : 0.0;
        tm_st2(tm + 4 * i, Ap);
      });
      tm_wait_st();
    }
    slot_put(1, w);
    __syncthreads();  // B2
    const double pq = slot_fin(1);
    if (!(pq > 0.0) || !isfinite(pq)) {  // loss of definiteness: report, do not loop
      breakdown = 1;
      break;
    }
    const double alpha = rz / pq;
    // pass C: x += alpha p, r += alpha q, rr = r^T D^-1 r, c = C D^-1 r (warp part)
    double rr = 0.0;
    if (wact) {
      acc_zero();
      const int yb = opaque(y0);
      cw.start(yb);
#pragma unroll
      for (int i0 = 0; i0 < RPT; i0 += 4) {
        if (i0 < nrow) {
          uint32_t tv[4][4];
#pragma unroll
          for (int u = 0; u < 4; u++)
            if (i0 + u < RPT) tm_ld4(tm + 4 * (i0 + u), tv[u]);
          tm_wait_ld();
#pragma unroll
          for (int u = 0; u < 4; u++) {
            const int i = i0 + u;
            if (i < RPT && i < nrow) {
              const int y = yb + i;
              const double q = dbl(tv[u][0], tv[u][1]);
              const double xv = dbl(tv[u][2], tv[u][3]) + alpha * Pref(y, xc);
              const double rk = lact ? r[i] + alpha * q : 0.0;
              r[i] = rk;
              const double uu = dinv(y) * rk;
              rr += rk * uu;
              double mL[N], mR[N], lL[N], lR[N];
              cw.row(i == 0 && syp >= 0, mL, mR, lL, lR);
              acc_row(i, y, uu, mL, mR, lL, lR);
              tm_st2(tm + 4 * i + 2, xv);
            }
            row_fence();
          }
        }
      }
      tm_wait_st();
      c_reduce();
    }
    slot_put(2, rr);
    __syncthreads();  // B3
    rr = slot_fin(2);
    const double cv = fin_c();
    const double yv = warp_sinv(Si, nc, cv);
    const double cy = warp_sum0((lane < nc) ? cv * yv : 0.0);
    put_y(yv);
    beta = (rr - cy) / rz;
  }

  // feasibility restoration: x += D^-1 C^T S^-1 (g - C x)
  auto sweep_x = [&](auto&& f) {  // f(i, y, x_k) with x from TMEM
    const int yb = opaque(y0);
#pragma unroll
    for (int i0 = 0; i0 < RPT; i0 += 4) {
      if (i0 < nrow) {
        uint32_t tv[4][4];
#pragma unroll
        for (int u = 0; u < 4; u++)
          if (i0 + u < RPT) tm_ld4(tm + 4 * (i0 + u), tv[u]);
        tm_wait_ld();
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const int i = i0 + u;
          if (i < RPT && i < nrow) f(i, yb + i, dbl(tv[u][2], tv[u][3]));
          row_fence();
        }
      }
    }
  };
  if (wact) {
    acc_zero();
    cw.start(opaque(y0));
    sweep_x([&](int i, int y, double xv) {
      double mL[N], mR[N], lL[N], lR[N];
      cw.row(i == 0 && syp >= 0, mL, mR, lL, lR);
      acc_row(i, y, lact ? xv : 0.0, mL, mR, lL, lR);
    });
    c_reduce();
  }
  __syncthreads();
  put_y(warp_sinv(Si, nc, gcol - fin_c()));
  if (wact) {
    double ctv[RPT];
    sweep_ct([&](int i, int y, double ct) { ctv[i] = ct; });
    double* xo = A.X + P.vec_off + (int64_t)rhs * nn;
    double* po = (A.level == 1 && P.pool_off >= 0) ? A.pool + P.pool_off + (int64_t)rhs * nn : nullptr;
    sweep_x([&](int i, int y, double xv) {
      const double xf = xv + dinv(y) * ctv[i];
      if (lact) {
        xo[y * nx + x] = xf;
        if (po) po[y * nx + x] = xf;
      }
    });
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
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tm_base_s), "r"(A.tm_cols)
                 : "memory");
  }
}

// ------------------------------------------------------------------------------------------
size_t pcg2d_smem(int nx, int ny, int nc, int nwarps, bool l1op) {
  const int nxm = l1op ? PCG2D_NXMAX_L1 : PCG2D_NXMAX_GN;
  (void)nx;
  size_t d = (size_t)nc * nc + 2 * (size_t)nwarps * 32 + 3 * 32 + (size_t)(nxm + 2) * (ny + 2);
  if (l1op) d += (size_t)(nxm + 1) * (ny + 1);
  size_t b = d * sizeof(double) + (size_t)nxm * ny * sizeof(float);
  if (l1op) b += (size_t)(nxm + 1) * (ny + 1);
  return (b + 15) & ~(size_t)15;
}

cudaError_t launch_node_ops2d(const LevelArgs& A, int max_nodes, cudaStream_t st) {
  dim3 grid((unsigned)((max_nodes + 127) / 128), (unsigned)A.nprob_mp);
  switch (A.N) {
    case 1: k_node_ops2d<1><<<grid, 128, 0, st>>>(A); break;
    case 2: k_node_ops2d<2><<<grid, 128, 0, st>>>(A); break;
    case 3: k_node_ops2d<3><<<grid, 128, 0, st>>>(A); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

template <int RPT, int N, bool L1OP>
static cudaError_t launch_one(const LevelArgs& A, int threads, size_t smem, cudaStream_t st) {
  auto k = k_pcg2d<RPT, N, L1OP>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k<<<(unsigned)A.nprob_mp * A.n_rhs, threads, smem, st>>>(A);
  return cudaGetLastError();
}

cudaError_t launch_pcg2d(const LevelArgs& A, bool l1op, int threads, size_t smem, cudaStream_t st) {
  if (l1op) {
    switch (A.N) {
      case 1: return launch_one<PCG2D_RPT_L1, 1, true>(A, threads, smem, st);
      case 2: return launch_one<PCG2D_RPT_L1, 2, true>(A, threads, smem, st);
      case 3: return launch_one<PCG2D_RPT_L1, 3, true>(A, threads, smem, st);
    }
  } else {
    switch (A.N) {
      case 1: return launch_one<PCG2D_RPT_GN, 1, false>(A, threads, smem, st);
      case 2: return launch_one<PCG2D_RPT_GN, 2, false>(A, threads, smem, st);
      case 3: return launch_one<PCG2D_RPT_GN, 3, false>(A, threads, smem, st);
    }
  }
  return cudaErrorInvalidValue;
}
