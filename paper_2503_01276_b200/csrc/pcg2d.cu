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

#include <cstdio>

#include "device_common.cuh"
#include "kernels.h"

namespace {

constexpr int kCrsMax = 256;  // coarse components per window of the two-level preconditioner

// ------------------------------------------------------------------------------------------
// TMEM helpers (32x32b shape: lane i of the warp <-> TMEM lane 32*(warp%4) + i).  No "memory"
// clobbers: they would pin every address-taken local in local memory; volatile asm statements
// keep their relative order.
__device__ __forceinline__ void tm_st8(uint32_t ta, const double (&v)[4]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(ta),
               "r"(__double2loint(v[0])), "r"(__double2hiint(v[0])), "r"(__double2loint(v[1])),
               "r"(__double2hiint(v[1])), "r"(__double2loint(v[2])), "r"(__double2hiint(v[2])),
               "r"(__double2loint(v[3])), "r"(__double2hiint(v[3])));
}
__device__ __forceinline__ void tm_ld8(uint32_t ta, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                 "=r"(v[7])
               : "r"(ta));
}
__device__ __forceinline__ void tm_st1(uint32_t ta, uint32_t v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};\n" ::"r"(ta), "r"(v));
}
__device__ __forceinline__ uint32_t tm_ld1(uint32_t ta) {
  uint32_t v;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(v) : "r"(ta));
  return v;
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n"); }
__device__ __forceinline__ double dbl(uint32_t lo, uint32_t hi) { return __hiloint2double((int)hi, (int)lo); }
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

// y_lane = sum_j Sinv[lane][j] c_j with c_j held by lane j (Sinv symmetric: read column-wise);
// NC rows at compile time (unrolled, two partial sums), nc <= NC the rows in use
template <int NC>
__device__ __forceinline__ double warp_sinv(const double* Si, int nc, double cv) {
  const int lane = threadIdx.x & 31;
  const int l = (lane < nc) ? lane : 0;
  double y0 = 0.0, y1 = 0.0;
#pragma unroll
  for (int j = 0; j < NC; j++) {
    const double cj = __shfl_sync(FULLMASK, cv, j);
    if (j < nc) {
      if (j & 1) y1 += Si[j * nc + l] * cj;
      else y0 += Si[j * nc + l] * cj;
    }
  }
  return (lane < nc) ? y0 + y1 : 0.0;
}

__device__ __forceinline__ int sub_slot(const LevelArgs& A, const ProbDesc& P, int dim, int e) {
  return fdiv(P.lo[dim] + e * A.s + A.coff, A.inv_c) - P.k[dim] + A.l;
}

// multiset state of two element ids a, b in {0..N-1, 0xFF = no element}: index of (min, max)
// in the triangular enumeration of pairs over N+1 symbols (N continua + "none")
template <int N>
__device__ __forceinline__ int pair_state(int a, int b) {
  a = (a == 0xFF) ? N : a;
  b = (b == 0xFF) ? N : b;
  const int lo = min(a, b), hi = max(a, b);
  return lo * (N + 1) - (lo * (lo - 1)) / 2 + (hi - lo);
}
template <int N> struct PairStates { static constexpr int value = (N + 1) * (N + 2) / 2; };

template <int N, bool L1OP, int KX, bool SMLR = false, int PLANE = 0>
struct NodeW {
  static constexpr int LW = (N == 1) ? 1 : ((N + 1) & ~1);  // padded table row (16-byte loads)
  // level 1: per-node side states (low nibble: left pair of elements, high: right pair) and
  // the table lut[state][j] = h^2/4 * multiplicity of continuum j in the pair
  const uint8_t* codes;
  const double* lut;
  const uint8_t* ids;  // cell ids (border 0xFF), only for interface rows
  int hqhi, hqlo;      // bit pattern of hq = h^2/4
  // levels >= 2: precomputed SoA [4N][nn]
  const double* base;
  int nn, nx;
  int xc;
  const uint8_t* cp;  // running row pointers
  const double* mp;
  const double* ms;   // SMLR: side sums staged in shared memory, [2N][PLANE] with pitch KX-1
  const double* msp;
  int y0;

  // c * hq for c in {0, 1}, branch-free on the bit pattern
  __device__ __forceinline__ double one_w(bool c) const {
    const int m = -(int)c;
    return __hiloint2double(hqhi & m, hqlo & m);
  }
  __device__ __forceinline__ void start(int y) {
    y0 = y;
    if (L1OP) cp = codes + y * (KX - 1) + xc;
    else mp = base + y * nx + xc;
    if (SMLR) msp = ms + y * (KX - 1) + xc;
  }
  // node (x, y0 + i) for consecutive i; low: also the weights of the lower elements alone
  __device__ __forceinline__ void row(bool low, double (&mL)[N], double (&mR)[N], double (&lL)[N],
                                      double (&lR)[N]) {
    if (L1OP) {
      const int code = *cp;
      cp += KX - 1;
      const double* tl = lut + (code & 15) * LW;
      const double* tr = lut + (code >> 4) * LW;
      if (N == 1) {
        mL[0] = tl[0];
        mR[0] = tr[0];
      } else {
#pragma unroll
        for (int j = 0; j < N; j += 2) {  // 16-byte loads of the (padded) table rows
          const double2 vl = *reinterpret_cast<const double2*>(tl + j);
          const double2 vr = *reinterpret_cast<const double2*>(tr + j);
          mL[j] = vl.x;
          mR[j] = vr.x;
          if (j + 1 < N) {
            mL[j + 1] = vl.y;
            mR[j + 1] = vr.y;
          }
        }
      }
#pragma unroll
      for (int j = 0; j < N; j++) lL[j] = lR[j] = 0.0;
      if (low) {  // interface row (first row of a chunk): elements of row y0 - 1
        const int dL = ids[y0 * KX + xc], dR = ids[y0 * KX + xc + 1];
#pragma unroll
        for (int j = 0; j < N; j++) {
          lL[j] = one_w(dL == j);
          lR[j] = one_w(dR == j);
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < N; j++) {
        if (SMLR) {
          mL[j] = msp[j * PLANE];
          mR[j] = msp[(N + j) * PLANE];
        } else {
          mL[j] = __ldg(mp + (int64_t)j * nn);
          mR[j] = __ldg(mp + (int64_t)(N + j) * nn);
        }
        lL[j] = low ? __ldg(mp + (int64_t)(2 * N + j) * nn) : 0.0;
        lR[j] = low ? __ldg(mp + (int64_t)(3 * N + j) * nn) : 0.0;
      }
      mp += nx;
      if (SMLR) msp += KX - 1;
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
#ifdef PCG2D_TIMING
__device__ unsigned long long g_pcg2d_phase[16];
__device__ unsigned long long g_pcg2d_crs[8];
void pcg2d_phase_dump(const char* tag) {
  unsigned long long h[16];
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(h, g_pcg2d_phase, sizeof h);
  const char* nm[7] = {"passA", "B1", "passB", "B2", "passC", "c_reduce", "B3+fin"};
  double tot = 0;
  for (int k = 0; k < 7; k++) tot += (double)h[k];
  fprintf(stderr, "[pcg2d timing %s] active-warp cycles per warp-iteration:", tag);
  for (int k = 0; k < 7; k++) fprintf(stderr, " %s=%.0f", nm[k], (double)h[k] / (double)h[7]);
  fprintf(stderr, " total=%.0f\n", tot / (double)h[7]);
  unsigned long long cc[8];
  cudaMemcpyFromSymbol(cc, g_pcg2d_crs, sizeof cc);
  fprintf(stderr, "  coarse sub-phases per warp-iteration: zr=%.0f csum=%.0f warp0+B4=%.0f vv=%.0f\n",
          (double)cc[0] / h[7], (double)cc[1] / h[7], (double)cc[2] / h[7], (double)cc[3] / h[7]);
  unsigned long long zz[8] = {0};
  cudaMemcpyToSymbol(g_pcg2d_crs, zz, sizeof zz);
  unsigned long long z[16] = {0};
  cudaMemcpyToSymbol(g_pcg2d_phase, z, sizeof z);
}
#else
void pcg2d_phase_dump(const char*) {}
#endif

template <int RPT, int N, bool L1OP, int NXM, int MAXW, int MINB, bool SSTC, bool SMLR, bool CRS = false>
__global__ void __launch_bounds__(MAXW * 32, MINB) k_pcg2d(LevelArgs A) {
  constexpr int RP4 = (RPT + 3) & ~3;  // rows rounded to the 4-row TMEM groups
  constexpr int NBC = 4 * RP4;         // TMEM columns per thread: q block, then x block
  constexpr int NBCW = NBC + (CRS ? RP4 / 4 : 0);  // CRS: + one column of 4 component bytes per 4 rows
  // compile-time pitches and shared-memory offsets (host checks nx, ny <= NXM and warps <= MAXW):
  // every per-row address is an immediate offset from one per-thread base
  constexpr int PX = NXM + 2, KX = NXM + 1, DX = NXM;
  const int prob = blockIdx.x;
  const int mp = prob / A.n_rhs, rhs = prob - mp * A.n_rhs;
  const ProbDesc& P = A.probs[mp];
  const int nx = P.nc[0] + 1, ny = P.nc[1] + 1, nn = nx * ny;
  const int ncx = nx - 1, ncy = ny - 1;
  const int nc = A.ncon, ws = A.w;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
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
  constexpr int LW = NodeW<N, L1OP, KX>::LW;
  constexpr int PLANE = DX * NXM;
  constexpr int NCM = 9 * N;              // constraint rows of a 3x3-subcell window (host: nc <= NCM)
  constexpr int NCC = CRS ? kCrsMax : 0;  // two-level preconditioner: coarse components per window
  constexpr int O_Y = (NCM * NCM + 1) & ~1, O_SL = O_Y + 64, O_B = O_SL + (CRS ? 4 : 3) * 32;
  constexpr int O_P = O_B + MAXW * 32;
  constexpr int O_K = O_P + PX * (NXM + 2), O_LUT = (O_K + (L1OP ? KX * (NXM + 1) : 0) + 1) & ~1;
  constexpr int O_S9 = O_LUT + (L1OP ? 16 * LW : 0);  // levels >= 2, SSTC: 9 x DX*NXM stencil
  constexpr int O_ML = O_S9 + (SSTC ? 9 * PLANE : 0);    // levels >= 2, SMLR: 2N x DX*NXM side sums
  constexpr int O_ZR = O_ML + (SMLR ? 2 * N * PLANE : 0);  // CRS: E^-1 Z^T r per component
  constexpr int O_VV = O_ZR + NCC;                        // CRS: coarse part of z per component
  constexpr int O_CS = O_VV + NCC;                        // CRS: (CZ) E^-1 Z^T r per constraint row
  // CSM (coarse data resident in shared memory; the precomputed-operator variants have room):
  // r mirror, CZ, E^-1 and the component node lists (ints)
  constexpr bool CSM = CRS && !L1OP;
  // level 1: Z^T r by the recurrence over (A z_a) lists; 49-node windows (r mirror in shared
  // memory): direct component sums every iteration
  constexpr bool REC = CRS && L1OP;
  constexpr int O_RS = O_CS + (CRS ? 32 : 0);
  constexpr int O_CZ = O_RS + (CSM ? PLANE : 0);
  constexpr int O_EI = O_CZ + (CSM ? NCM * kCrsMax : 0);
  constexpr int O_CL = O_EI + (CSM ? kCrsMax : 0);
  constexpr int O_D = O_CL + (CSM ? (PLANE + kCrsMax + 2) / 2 : 0);  // end of the double region
  double* Si = smem;                      // [NCM*NCM] S^-1 (nc*nc used)
  double* Ysh = smem + O_Y;               // [32] yhat, [32] beta (written by warp 0)
  double* slots = smem + O_SL;            // [3][32] scalar partial sums (rz, pq, rr)
  double* bins = smem + O_B;              // [MAXW][32] constraint partial sums, per warp
  double* p_s = smem + O_P;               // PX*(NXM+2), zero halo
  double* kap_s = smem + O_K;             // level 1: KX*(NXM+1), zero border
  double* lut_s = smem + O_LUT;           // level 1: 16*LW
  float* dinv_s = reinterpret_cast<float*>(smem + O_D);                   // DX*NXM
  uint8_t* ids_s = reinterpret_cast<uint8_t*>(dinv_s + DX * NXM);         // KX*(NXM+1), border 0xFF
  uint8_t* codes_s = ids_s + (L1OP ? KX * (NXM + 1) : 0);                 // DX*NXM
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
  for (int i = threadIdx.x; i < MAXW * 32; i += blockDim.x) bins[i] = 0.0;
  for (int i = threadIdx.x; i < (CRS ? 4 : 3) * 32; i += blockDim.x) slots[i] = 0.0;  // incl. absent warps
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
    for (int i = threadIdx.x; i < PairStates<N>::value * LW; i += blockDim.x) {
      // lut[state][j]: decode the state back to its pair (a <= b) and count j
      const int st = i / LW, j = i - st * LW;
      int a = 0, rem = st;
      while (rem >= N + 1 - a) {
        rem -= N + 1 - a;
        a++;
      }
      const int b = a + rem;
      lut_s[i] = 0.25 * A.h * A.h * (double)((a == j) + (b == j));
    }
    __syncthreads();
    for (int k = threadIdx.x; k < nn; k += blockDim.x) {
      const int y = k / nx, xx = k - y * nx;
      const uint8_t* c0 = ids_s + y * KX + xx;  // element (xx-1, y-1)
      const int sL = pair_state<N>(c0[0], c0[KX]), sR = pair_state<N>(c0[1], c0[KX + 1]);
      codes_s[y * DX + xx] = (uint8_t)(sL | (sR << 4));
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmq = tm_base_s + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * NBCW);
  const uint32_t tmx = tmq + 2 * RP4;
  const uint32_t tmc = tmq + NBC;  // CRS: component ids of this thread's rows, 4 per column

  // per-thread subcell columns of the left / right elements
  const int sxL = (xc >= 1) ? sub_slot(A, P, 0, xc - 1) : 0;
  const int sxR = (xc < ncx) ? sub_slot(A, P, 0, xc) : 0;
  NodeW<N, L1OP, KX, SMLR, PLANE> cw;
  double* ml_s = smem + O_ML;
  if (SMLR) {  // stage the side sums [L|R][j] of the window (pitch DX), once per problem
    const double* src = A.MLR + P.node_off * 4 * N;
    for (int i = threadIdx.x; i < 2 * N * nn; i += blockDim.x) {
      const int tt = i / nn, k = i - tt * nn, y = k / nx;
      ml_s[tt * PLANE + y * DX + (k - y * nx)] = src[i];
    }
    __syncthreads();
  }
  cw.ms = ml_s;
  cw.ids = ids_s;
  cw.codes = codes_s;
  cw.lut = lut_s;
  cw.hqhi = __double2hiint(0.25 * A.h * A.h);
  cw.hqlo = __double2loint(0.25 * A.h * A.h);
  cw.base = A.MLR + P.node_off * 4 * N;
  cw.nn = nn;
  cw.nx = nx;
  cw.xc = xc;
  const double* S9 = A.STC + P.node_off * 9;
  double* s9_s = smem + O_S9;
  if (SSTC) {  // stage the window's stencil rows in shared memory (pitch DX), once per problem
    for (int i = threadIdx.x; i < 9 * nn; i += blockDim.x) {
      const int cc = i / nn, k = i - cc * nn, y = k / nx;
      s9_s[cc * DX * NXM + y * DX + (k - y * nx)] = S9[i];
    }
    __syncthreads();
  }

  double r[RPT];
#pragma unroll
  for (int i = 0; i < RPT; i++) r[i] = 0.0;
  double yh = 0.0;  // projector coefficients: lane t holds yhat_t (identical in every warp)

  // ---- C^T yhat per row: f(i, y, ct) -------------------------------------------------------
  auto sweep_ct = [&](auto&& f) {
    double YL[N], YR[N], YLp[N], YRp[N];
#pragma unroll
    for (int j = 0; j < N; j++) {
      YL[j] = __shfl_sync(FULLMASK, yh, (sy * ws + sxL) * N + j);
      YR[j] = __shfl_sync(FULLMASK, yh, (sy * ws + sxR) * N + j);
      YLp[j] = __shfl_sync(FULLMASK, yh, (max(syp, 0) * ws + sxL) * N + j);
      YRp[j] = __shfl_sync(FULLMASK, yh, (max(syp, 0) * ws + sxR) * N + j);
    }
    const int yb = opaque(y0);
    cw.start(yb);
#pragma unroll
    for (int i = 0; i < RPT; i++) {
      if (i >= nrow) break;
      const bool split = (i == 0) && (syp >= 0);
      double mL[N], mR[N], lL[N], lR[N];
      cw.row(split, mL, mR, lL, lR);
      double ct = 0.0;
      if (split) {
#pragma unroll
        for (int j = 0; j < N; j++)
          ct += lL[j] * YLp[j] + (mL[j] - lL[j]) * YL[j] + lR[j] * YRp[j] + (mR[j] - lR[j]) * YR[j];
      } else {
#pragma unroll
        for (int j = 0; j < N; j++) ct += mL[j] * YL[j] + mR[j] * YR[j];
      }
      f(i, yb + i, ct);
    }
  };

  // ---- (A p)_k per row from the smem vector p_s: f(i, y, Ap, p_k) ----------------------------
  auto sweep_stencil = [&](auto&& f) {
    const int yb = opaque(y0);
    const double* pp = p_s + (yb + 1) * PX + (xc + 1);  // node (xc, yb)
    double a0 = pp[-PX - 1], b0 = pp[-PX], c0 = pp[-PX + 1];
    double a1 = pp[-1], b1 = pp[0], c1 = pp[1];
    const double* kp = kap_s + yb * KX + xc;  // element (xc-1, yb-1)
    double kL0 = 0.0, kR0 = 0.0;
    if (L1OP) {
      kL0 = kp[0];
      kR0 = kp[1];
    }
    const double* s9 = S9 + yb * nx + xc;
    const double* s9s = s9_s + yb * DX + xc;
#pragma unroll
    for (int i = 0; i < RPT; i++) {
      if (i >= nrow) break;
      const double a2 = pp[(i + 1) * PX - 1], b2 = pp[(i + 1) * PX], c2 = pp[(i + 1) * PX + 1];
      double Ap;
      if (L1OP) {
        // Q1 element rows kappa/6 (4 v_a - v_a^1 - v_a^2 - 2 v_a^3) summed over the 4 cells
        const double kL1 = kp[(i + 1) * KX], kR1 = kp[(i + 1) * KX + 1];
        const double sL = kL0 + kL1, sR = kR0 + kR1, sD = kL0 + kR0, sU = kL1 + kR1;
        double acc = 4.0 * (sL + sR) * b1 - sR * c1 - sL * a1 - sU * b2 - sD * b0;
        acc -= 2.0 * (kR1 * c2 + kL1 * a2 + kR0 * c0 + kL0 * a0);
        Ap = acc * (1.0 / 6.0);
        kL0 = kL1;
        kR0 = kR1;
      } else if (SSTC) {
        constexpr int CS = DX * NXM;
        const double* s = s9s + i * DX;
        Ap = s[0] * a0 + s[CS] * b0 + s[2 * CS] * c0 + s[3 * CS] * a1 + s[4 * CS] * b1 + s[5 * CS] * c1 +
             s[6 * CS] * a2 + s[7 * CS] * b2 + s[8 * CS] * c2;
      } else {
        const double* s = s9 + i * nx;
        Ap = __ldg(s) * a0 + __ldg(s + nn) * b0 + __ldg(s + 2 * nn) * c0 + __ldg(s + 3 * nn) * a1 +
             __ldg(s + 4 * nn) * b1 + __ldg(s + 5 * nn) * c1 + __ldg(s + 6 * nn) * a2 +
             __ldg(s + 7 * nn) * b2 + __ldg(s + 8 * nn) * c2;
      }
      f(i, yb + i, Ap, b1);
      a0 = a1; b0 = b1; c0 = c1;
      a1 = a2; b1 = b2; c1 = c2;
    }
  };

  // ---- TMEM row groups: a value per row is buffered and stored 4 rows at a time -------------
  double gb[4] = {0.0, 0.0, 0.0, 0.0};
  auto gput = [&](uint32_t base, int i, double v) {
    gb[i & 3] = v;
    if ((i & 3) == 3) tm_st8(base + 2 * (i - 3), gb);
  };
  auto gflush = [&](uint32_t base) {  // the partial last group
    if (nrow & 3) tm_st8(base + 2 * (nrow & ~3), gb);
    tm_wait_st();
  };
  // x from TMEM per row: f(i, y, x_k); x_k returned by f is stored back
  auto sweep_x = [&](auto&& f) {
    const int yb = opaque(y0);
#pragma unroll
    for (int g = 0; g < RPT; g += 4) {
      if (g >= nrow) break;
      uint32_t xa[8];
      tm_ld8(tmx + 2 * g, xa);
      tm_wait_ld();
      double xv[4];
#pragma unroll
      for (int u = 0; u < 4; u++) {
        xv[u] = dbl(xa[2 * u], xa[2 * u + 1]);
        if (g + u < RPT && g + u < nrow) xv[u] = f(g + u, yb + g + u, xv[u]);
      }
      tm_st8(tmx + 2 * g, xv);
    }
    tm_wait_st();
  };

  // ---- constraint accumulation: aC (current subcell row), aP (previous, interface row) -------
  double aC[2][N], aP[2][N];
  auto acc_zero = [&]() {
#pragma unroll
    for (int j = 0; j < N; j++) aC[0][j] = aC[1][j] = aP[0][j] = aP[1][j] = 0.0;
  };
  auto acc_row = [&](int i, double u, const double (&mL)[N], const double (&mR)[N], const double (&lL)[N],
                     const double (&lR)[N]) {
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
  // after a barrier, every warp: c and yhat summed over warps in a fixed order (lane t: entry t)
  auto fin_c = [&]() -> double {
    double s = 0.0;
#pragma unroll
    for (int w2 = 0; w2 < MAXW; w2++) s += bins[w2 * 32 + lane];
    return s;
  };

  auto slot_put = [&](int which, double v) {
    v = warp_sum0(v);
    if (lane == 0) slots[which * 32 + warp] = v;
  };
  // every lane sums the per-warp slots itself from broadcast reads: no shuffle chain after the
  // barriers (two fixed-order chains)
  auto slot_fin = [&](int which) {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int w2 = 0; w2 < MAXW; w2 += 2) {
      s0 += slots[which * 32 + w2];
      if (w2 + 1 < MAXW) s1 += slots[which * 32 + w2 + 1];
    }
    return s0 + s1;
  };

  // ---- two-level preconditioner M^-1 = D^-1 + Z E^-1 Z^T: s = Z^T r summed per
  //      component from a mirror of r (start; every iteration in the 49-node windows) or carried
  //      by the recurrence over the (A z_a) lists (level 1); the projection uses S_M = C M^-1 C^T
  //      (k_proj_setup) ----
  const bool crs = CRS && A.ncomp[mp] > 0;
  const int nca = crs ? A.ncomp[mp] : 0;
  const int* cmp = A.cmap + P.node_off;
  const int* cpt = A.cptr + (int64_t)mp * (A.ncmax + 1);
  const int* cls = A.clist + P.node_off;
  const int* azp = A.azp + (int64_t)mp * (A.ncmax + 1);
  const int* azi = A.azi + (int64_t)kAzCap * P.node_off;
  const double* azw = A.azw + (int64_t)kAzCap * P.node_off;
  const double* Eiv = A.Einv + (int64_t)mp * A.ncmax;
  const double* CZm = A.CZ + (int64_t)mp * nc * A.ncmax;
  double* Rg = A.R + P.vec_off + (int64_t)rhs * nn;
  double* zr = smem + O_ZR;
  double* vv = smem + O_VV;
  double* csum = smem + O_CS;
  double* rsm = smem + O_RS;                                // CSM: r mirror [ny][nx]
  double* czs = smem + O_CZ;                                // CSM: CZ [nc][kCrsMax]
  double* eis = smem + O_EI;                                // CSM: E^-1
  int* cls_s = reinterpret_cast<int*>(smem + O_CL);         // CSM: node lists
  int* cpt_s = cls_s + PLANE;                               // CSM: list starts [nca+1]
  if (CSM && crs) {
    for (int i = threadIdx.x; i < nc * nca; i += blockDim.x) {
      const int t = i / nca, a = i - t * nca;
      czs[t * kCrsMax + a] = __ldg(CZm + (int64_t)t * A.ncmax + a);
    }
    for (int a = threadIdx.x; a < nca; a += blockDim.x) eis[a] = __ldg(Eiv + a);
    for (int a = threadIdx.x; a <= nca; a += blockDim.x) cpt_s[a] = __ldg(cpt + a);
    const int nl = __ldg(cpt + nca);
    for (int i = threadIdx.x; i < nl; i += blockDim.x) cls_s[i] = __ldg(cls + i);
    __syncthreads();
  }
  const int nwarps = blockDim.x >> 5;
  // csum = (CZ) E^-1 s (s = Z^T r in zr).  One barrier.
  auto coarse_csum = [&]() {
    for (int t = warp; t < nc; t += nwarps) {
      double sv = 0.0;
      for (int a = lane; a < nca; a += 32)
        sv += (CSM ? czs[t * kCrsMax + a] : __ldg(CZm + (int64_t)t * A.ncmax + a)) *
              (CSM ? eis[a] : __ldg(Eiv + a)) * zr[a];
      sv = warp_sum0(sv);
      if (lane == 0) csum[t] = sv;
    }
    __syncthreads();
  };
  // recurrence (after B3): s += alpha (A Z)^T p (the latter in vv, formed in pass B), slot 3 =
  // s^T E^-1 s, then csum.  Two barriers.
  auto coarse_rec = [&](double alpha_) {
    double part = 0.0;
    for (int a = threadIdx.x; a < nca; a += blockDim.x) {
      const double sv = zr[a] + alpha_ * vv[a];
      zr[a] = sv;
      part += sv * sv * (CSM ? eis[a] : __ldg(Eiv + a));
    }
    part = warp_sum0(part);
    if (lane == 0) slots[3 * 32 + warp] = part;
    __syncthreads();
    coarse_csum();
  };
  // (A Z)^T p from p_s (after B1) into vv: 4-lane groups over each component's (A z_a) list
  auto coarse_zq = [&]() {
    const int sub = lane & 3, ngrp = blockDim.x >> 2;
    for (int base = 0; base < nca; base += ngrp) {  // warp-uniform trip count
      const int a = base + (threadIdx.x >> 2);
      double sv = 0.0;
      if (a < nca) {
        const int i0 = __ldg(azp + a), i1 = __ldg(azp + a + 1);
#pragma unroll 4
        for (int i = i0 + sub; i < i1; i += 4) {
          const int xy = __ldg(azi + i);
          sv += __ldg(azw + i) * p_s[((xy >> 16) + 1) * PX + (xy & 0xFFFF) + 1];
        }
      }
      sv += __shfl_xor_sync(FULLMASK, sv, 1);
      sv += __shfl_xor_sync(FULLMASK, sv, 2);
      if (a < nca && sub == 0) vv[a] = sv;
    }
  };
  // zr = E^-1 Z^T Rg, slot 3 = (Z^T r)^T E^-1 (Z^T r); then csum = (CZ) zr.  Two barriers.
  auto coarse_c = [&]() {
    double part = 0.0;
    // groups of 4 lanes per component, each lane a strided quarter of its node list, combined by
    // two xor shuffles (fixed order); rounds over the components are uniform per warp
    const int sub = lane & 3, ngrp = blockDim.x >> 2;
    for (int base = 0; base < nca; base += ngrp) {  // warp-uniform trip count
      const int a = base + (threadIdx.x >> 2);
      double sv = 0.0;
      if (a < nca) {
        if (CSM) {
          const int i0 = cpt_s[a], i1 = cpt_s[a + 1];
          for (int i = i0 + sub; i < i1; i += 4) sv += rsm[cls_s[i]];
        } else {
          const int i0 = __ldg(cpt + a), i1 = __ldg(cpt + a + 1);
#pragma unroll 8
          for (int i = i0 + sub; i < i1; i += 4) sv += __ldcg(Rg + __ldg(cls + i));
        }
      }
      sv += __shfl_xor_sync(FULLMASK, sv, 1);
      sv += __shfl_xor_sync(FULLMASK, sv, 2);
      if (a < nca && sub == 0) {
        const double ei = CSM ? eis[a] : __ldg(Eiv + a);
        zr[a] = sv;  // s_a = (Z^T r)_a, carried by the recurrence from here on
        part += sv * sv * ei;
      }
    }
    part = warp_sum0(part);
    if (lane == 0) slots[3 * 32 + warp] = part;
    __syncthreads();
    coarse_csum();
  };
  // vv = s0 zr - E^-1 (CZ)^T Ysh (s0 = 0: minus the coarse part of M^-1 C^T yhat).  One barrier.
  // s0 != 0: vv = E^-1 (s - (CZ)^T yhat) (coarse part of z = M^-1 r~) and s <- s - (CZ)^T yhat
  // (= Z^T r~); s0 == 0: vv = -E^-1 (CZ)^T yhat (minus the coarse part of M^-1 C^T yhat), s kept
  auto coarse_v = [&](double s0) {
    for (int a = threadIdx.x; a < nca; a += blockDim.x) {
      double acc = 0.0;
      for (int t = 0; t < nc; t++) acc += (CSM ? czs[t * kCrsMax + a] : __ldg(CZm + (int64_t)t * A.ncmax + a)) * Ysh[t];
      const double ei = CSM ? eis[a] : __ldg(Eiv + a);
      if (s0 != 0.0) {
        const double sr = zr[a] - acc;
        vv[a] = ei * sr;
        zr[a] = sr;
      } else {
        vv[a] = -ei * acc;
      }
    }
    __syncthreads();
  };
  auto vv_at = [&](int y) -> double {
    if (!crs) return 0.0;
    const int a = __ldg(cmp + y * nx + xc);
    return (a >= 0) ? vv[a] : 0.0;
  };
  auto vv_w = [&](uint32_t word, int u) -> double {  // component byte u of a TMEM word (255: none)
    const uint32_t a = (word >> (8 * u)) & 255u;
    return (a == 255u) ? 0.0 : vv[a];
  };
  if (CRS && crs && wact) {  // this thread's component ids into TMEM, 4 rows per column
#pragma unroll
    for (int gq = 0; gq < RP4 / 4; gq++) {
      uint32_t word = 0;
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int i = gq * 4 + u;
        int a = -1;
        if (lact && i < nrow) a = __ldg(cmp + (y0 + i) * nx + xc);
        word |= (uint32_t)((a >= 0) ? a : 255) << (8 * u);
      }
      tm_st1(tmc + gq, word);
    }
    tm_wait_st();
  }

  // ---- init: x0 = D^-1 C^T S^-1 t (minimum-norm feasible point), r0 = A x0 - b,
  //      c = C D^-1 r0, yhat = S^-1 c; returns r0^T D^-1 r0 -----------------------------------
  const bool lev2 = !L1OP && A.level >= 2;  // the level-1 variant is only launched at level 1
  const double* bvec = lev2 ? A.B + P.vec_off + (int64_t)rhs * nn : nullptr;
  auto init = [&](double tval) -> double {
    yh = warp_sinv<NCM>(Si, nc, tval);
    if (crs) {  // x0 = M^-1 C^T S_M^-1 t: coarse part -vv with vv = -E^-1 (CZ)^T yhat
      if (warp == 0) Ysh[lane] = yh;
      __syncthreads();
      coarse_v(0.0);
    }
    if (wact) {
      sweep_ct([&](int i, int y, double ct) {
        const double x0 = (double)dinv_s[y * DX + xc] * ct - vv_at(y);
        if (lact) p_s[(y + 1) * PX + x + 1] = x0;
        gput(tmx, i, x0);
      });
      gflush(tmx);
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
        if (i >= nrow) break;
        double mL[N], mR[N], lL[N], lR[N];
        cw.row(i == 0 && syp >= 0, mL, mR, lL, lR);
        const double u = (double)dinv_s[(yb + i) * DX + xc] * r[i];
        rr += r[i] * u;
        acc_row(i, u, mL, mR, lL, lR);
        if (crs && lact) {
          if (CSM) rsm[(yb + i) * nx + x] = r[i];
          else Rg[(yb + i) * nx + x] = r[i];
        }
      }
      c_reduce();
    }
    slot_put(2, rr);
    __syncthreads();
    if (crs) coarse_c();
    rr = slot_fin(2) + (crs ? slot_fin(3) : 0.0);
    yh = warp_sinv<NCM>(Si, nc, fin_c() + ((crs && lane < nc) ? csum[lane] : 0.0));
    if (crs) {  // z of the first pass A: coarse part vv = zr - E^-1 (CZ)^T yhat
      if (warp == 0) Ysh[lane] = yh;
      __syncthreads();
      coarse_v(1.0);
    }
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
        v += lact ? (double)dinv_s[y * DX + xc] * w * w : 0.0;
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
#ifdef PCG2D_TIMING
  unsigned long long tacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  unsigned long long tprev = clock64();
#define TMARK(k)                              \
  {                                           \
    const unsigned long long t_ = clock64();  \
    tacc[k] += t_ - tprev;                    \
    tprev = t_;                               \
  }
#else
#define TMARK(k)
#endif
  double alpha = 0.0;
  for (;; it++) {
    // pass A: x += alpha_prev p_prev (deferred update), r <- r - C^T yhat (re-projection),
    // z = D^-1 r, p <- -z + beta p, rz = r.z
    double v = 0.0;
    if (wact) {
      const bool first = (it == 0);
      double YL[N], YR[N], YLp[N], YRp[N];
#pragma unroll
      for (int j = 0; j < N; j++) {
        YL[j] = __shfl_sync(FULLMASK, yh, (sy * ws + sxL) * N + j);
        YR[j] = __shfl_sync(FULLMASK, yh, (sy * ws + sxR) * N + j);
        YLp[j] = __shfl_sync(FULLMASK, yh, (max(syp, 0) * ws + sxL) * N + j);
        YRp[j] = __shfl_sync(FULLMASK, yh, (max(syp, 0) * ws + sxR) * N + j);
      }
      const int yb = opaque(y0);
      cw.start(yb);
#pragma unroll
      for (int g = 0; g < RPT; g += 4) {
        if (g >= nrow) break;
        uint32_t xa[8];
        tm_ld8(tmx + 2 * g, xa);
        uint32_t cword = 0;
        if (CRS && crs) cword = tm_ld1(tmc + g / 4);
        tm_wait_ld();
        double xv[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const int i = g + u;
          xv[u] = dbl(xa[2 * u], xa[2 * u + 1]);
          if (i < RPT && i < nrow) {
            const int y = yb + i;
            double mL[N], mR[N], lL[N], lR[N];
            const bool split = (i == 0) && (syp >= 0);
            cw.row(split, mL, mR, lL, lR);
            double ct = 0.0;
            if (split) {
#pragma unroll
              for (int j = 0; j < N; j++)
                ct += lL[j] * YLp[j] + (mL[j] - lL[j]) * YL[j] + lR[j] * YRp[j] + (mR[j] - lR[j]) * YR[j];
            } else {
#pragma unroll
              for (int j = 0; j < N; j++) ct += mL[j] * YL[j] + mR[j] * YR[j];
            }
            const double rk = lact ? r[i] - ct : 0.0;
            r[i] = rk;
            const double z = (double)dinv_s[y * DX + xc] * rk + ((CRS && crs && lact) ? vv_w(cword, u) : 0.0);
            double& pk = p_s[(y + 1) * PX + xc + 1];
            const double pold = pk;
            xv[u] += alpha * pold;
            if (lact) pk = first ? -z : -z + beta * pold;
            v += rk * z;
          }
        }
        tm_st8(tmx + 2 * g, xv);
      }
      tm_wait_st();
    }
    TMARK(0);
    slot_put(0, v);
    __syncthreads();  // B1: p complete
    TMARK(1);
    // pass B: q = A p (to TMEM), pq
    double w = 0.0;
    if (wact) {
      sweep_stencil([&](int i, int y, double Ap, double pk) {
        w += lact ? pk * Ap : 0.0;
        gput(tmq, i, Ap);
      });
      gflush(tmq);
    }
    if (REC && crs) coarse_zq();
    TMARK(2);
    slot_put(1, w);
    __syncthreads();  // B2
    rz = slot_fin(0);
    const double pq = slot_fin(1);
    TMARK(3);
    if (it == 0) ref = fmax(rz, rz_ref);
    if (!(rz > fmax(tol2 * ref, floor2)) || it >= A.max_iter) break;
    if (!(pq > 0.0) || !isfinite(pq)) {  // loss of definiteness: report, do not loop
      breakdown = 1;
      break;
    }
    alpha = rz / pq;
    // pass C: r += alpha q, rr = r^T D^-1 r, c = C D^-1 r (warp part)
    double rr = 0.0;
    if (wact) {
      acc_zero();
      const int yb = opaque(y0);
      cw.start(yb);
#pragma unroll
      for (int g = 0; g < RPT; g += 4) {
        if (g >= nrow) break;
        uint32_t qa[8];
        tm_ld8(tmq + 2 * g, qa);
        uint32_t cw4 = 0xFFFFFFFFu;
        if (CSM && crs) cw4 = tm_ld1(tmc + g / 4);
        tm_wait_ld();
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const int i = g + u;
          if (i < RPT && i < nrow) {
            const int y = yb + i;
            const double rk = lact ? r[i] + alpha * dbl(qa[2 * u], qa[2 * u + 1]) : 0.0;
            r[i] = rk;
            const double uu = (double)dinv_s[y * DX + xc] * rk;
            rr += rk * uu;
            double mL[N], mR[N], lL[N], lR[N];
            cw.row(i == 0 && syp >= 0, mL, mR, lL, lR);
            acc_row(i, uu, mL, mR, lL, lR);
            if (CSM && crs && lact && ((cw4 >> (8 * u)) & 255u) != 255u) rsm[y * nx + x] = rk;
          }
        }
      }
      TMARK(4);
      c_reduce();
    }
    TMARK(5);
    slot_put(2, rr);
    __syncthreads();  // B3
#ifdef PCG2D_TIMING
    unsigned long long tc0 = clock64();
#endif
    if (REC && crs) coarse_rec(alpha);
    else if (crs) coarse_c();
#ifdef PCG2D_TIMING
    unsigned long long tc1 = clock64();
#endif
    if (warp == 0) {  // yhat = S^-1 c, beta = (r^T D^-1 r - c.yhat) / rz  (M-metric with the coarse space)
      const double cv = fin_c() + ((crs && lane < nc) ? csum[lane] : 0.0);
      const double yv = warp_sinv<NCM>(Si, nc, cv);
      const double cy = warp_sum0(cv * yv);
      const double rrs = slot_fin(2) + (crs ? slot_fin(3) : 0.0);
      Ysh[lane] = yv;
      if (lane == 0) Ysh[32] = (rrs - cy) / rz;
    }
    __syncthreads();  // B4
    yh = Ysh[lane];
    beta = Ysh[32];
#ifdef PCG2D_TIMING
    unsigned long long tc2 = clock64();
#endif
    if (crs) coarse_v(1.0);
#ifdef PCG2D_TIMING
    unsigned long long tc3 = clock64();
    if (lane == 0 && wact) {
      atomicAdd(&g_pcg2d_crs[0], tc1 - tc0);
      atomicAdd(&g_pcg2d_crs[2], tc2 - tc1);
      atomicAdd(&g_pcg2d_crs[3], tc3 - tc2);
    }
#endif
    if (A.dbg && prob == A.dbg_prob && threadIdx.x == 0 && it < A.dbg_cap) {  // dev: MCH_PCG_DEBUG
      double* o = A.dbg + 8 * it;
      o[0] = rz; o[1] = pq; o[2] = alpha; o[3] = beta;
    }
    TMARK(6);
  }
#ifdef PCG2D_TIMING
  if (lane == 0)
    for (int k = 0; k < 7; k++) atomicAdd(&g_pcg2d_phase[(wact ? 0 : 8) + k], tacc[k]);
  if (lane == 0 && wact) atomicAdd(&g_pcg2d_phase[7], (unsigned long long)it);
#endif

  // feasibility restoration: x += D^-1 C^T S^-1 (g - C x)
  if (wact) {
    acc_zero();
    cw.start(opaque(y0));
    sweep_x([&](int i, int, double xv) {
      double mL[N], mR[N], lL[N], lR[N];
      cw.row(i == 0 && syp >= 0, mL, mR, lL, lR);
      acc_row(i, lact ? xv : 0.0, mL, mR, lL, lR);
      return xv;
    });
    c_reduce();
  }
  __syncthreads();
  yh = warp_sinv<NCM>(Si, nc, gcol - fin_c());
  if (crs) {  // x += M^-1 C^T yhat: coarse part -vv with vv = -E^-1 (CZ)^T yhat
    if (warp == 0) Ysh[lane] = yh;
    __syncthreads();
    coarse_v(0.0);
  }
  if (wact) {
    double ctv[RPT];
    sweep_ct([&](int i, int y, double ct) { ctv[i] = ct - vv_at(y) / (double)dinv_s[y * DX + xc]; });
    double* xo = A.X + P.vec_off + (int64_t)rhs * nn;
    double* po = (A.level == 1 && P.pool_off >= 0) ? A.pool + P.pool_off + (int64_t)rhs * nn : nullptr;
    sweep_x([&](int i, int y, double xv) {
      const double xf = xv + (double)dinv_s[y * DX + xc] * ctv[i];
      if (lact) {
        xo[y * nx + x] = xf;
        if (po) po[y * nx + x] = xf;
      }
      return xf;
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
size_t pcg2d_smem_t(int N, bool l1op, int nxm, int maxw, bool sstc, bool smlr, bool crs) {
  const int PX = nxm + 2, KX = nxm + 1, DX = nxm, LW = (N == 1) ? 1 : ((N + 1) & ~1);
  size_t d = ((81 * N * N + 1) & ~1) + 64 + (crs ? 4 : 3) * 32 + (size_t)maxw * 32 + (size_t)PX * (nxm + 2);
  if (crs) d += 2 * kCrsMax + 32;
  if (crs && !l1op) d += (size_t)DX * nxm + 9 * N * kCrsMax + kCrsMax + ((size_t)DX * nxm + kCrsMax + 2) / 2;
  d += 1;  // O_LUT rounded up to 16 bytes
  if (sstc) d += 9 * (size_t)DX * nxm;
  if (smlr) d += 2 * (size_t)N * DX * nxm;
  if (l1op) d += (size_t)KX * (nxm + 1) + 16 * LW;
  size_t b = d * sizeof(double) + (size_t)DX * nxm * sizeof(float);
  if (l1op) b += (size_t)KX * (nxm + 1) + (size_t)DX * nxm;
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

template <int RPT, int N, bool L1OP, int NXM, int MAXW, int MINB, bool SSTC, bool SMLR, bool CRS = false>
static cudaError_t launch_one(const LevelArgs& A, int threads, cudaStream_t st) {
  auto k = k_pcg2d<RPT, N, L1OP, NXM, MAXW, MINB, SSTC, SMLR, CRS>;
  const size_t smem = pcg2d_smem_t(N, L1OP, NXM, MAXW, SSTC, SMLR, CRS);
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k<<<(unsigned)A.nprob_mp * A.n_rhs, threads, smem, st>>>(A);
  return cudaGetLastError();
}

#ifndef L1_RPT
#define L1_RPT 33
#endif
#ifndef L1_MAXW
#define L1_MAXW 12
#endif
#ifndef GN49_RPT
#define GN49_RPT 9
#endif
#ifndef GN49_MAXW
#define GN49_MAXW 12
#endif
#ifndef GN49_MINB
#define GN49_MINB 1
#endif
#ifndef GN49_SSTC
#define GN49_SSTC false
#endif
#ifndef GN49_SMLR
#define GN49_SMLR true
#endif
#ifndef GN25_SMLR
#define GN25_SMLR true
#endif
#ifndef GN25_SSTC
#define GN25_SSTC false
#endif
#ifndef GN25_MINB
#define GN25_MINB 4
#endif

template <int N>
static cudaError_t launch_n(const LevelArgs& A, int variant, int threads, cudaStream_t st) {
  switch (variant) {
    case PCG2D_V_L1:
      if (A.coarse) return launch_one<L1_RPT, N, true, 97, L1_MAXW, 1, false, false, true>(A, threads, st);
      return launch_one<L1_RPT, N, true, 97, L1_MAXW, 1, false, false>(A, threads, st);
    case PCG2D_V_GN49:
      if (A.coarse)
        return launch_one<GN49_RPT, N, false, 49, GN49_MAXW, GN49_MINB, GN49_SSTC, GN49_SMLR, true>(A, threads, st);
      return launch_one<GN49_RPT, N, false, 49, GN49_MAXW, GN49_MINB, GN49_SSTC, GN49_SMLR>(A, threads, st);
    case PCG2D_V_GN25: return launch_one<9, N, false, 25, 4, GN25_MINB, GN25_SSTC, GN25_SMLR>(A, threads, st);
    case PCG2D_V_GN97: return launch_one<17, N, false, 97, 24, 1, false, false>(A, threads, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_pcg2d(const LevelArgs& A, int variant, int threads, cudaStream_t st) {
  switch (A.N) {
    case 1: return launch_n<1>(A, variant, threads, st);
    case 2: return launch_n<2>(A, variant, threads, st);
    case 3: return launch_n<3>(A, variant, threads, st);
  }
  return cudaErrorInvalidValue;
}

// variant limits: rows per thread, widest window (nodes), warps per CTA
void pcg2d_variant(int variant, int* rpt, int* nxm, int* maxw, int* l1op, int* sstc, int* smlr) {
  *sstc = (variant == PCG2D_V_GN49) ? (int)GN49_SSTC : ((variant == PCG2D_V_GN25) ? (int)GN25_SSTC : 0);
  *smlr = (variant == PCG2D_V_GN49) ? (int)GN49_SMLR : ((variant == PCG2D_V_GN25) ? (int)GN25_SMLR : 0);
  static const int T[4][4] = {{L1_RPT, 97, L1_MAXW, 1}, {GN49_RPT, 49, GN49_MAXW, 0}, {9, 25, 4, 0}, {17, 97, 24, 0}};
  *rpt = T[variant][0];
  *nxm = T[variant][1];
  *maxw = T[variant][2];
  *l1op = T[variant][3];
}
