// Fused fine-window passes of the 3D correction problems (levels n >= 2, fine windows of at most
// 49 nodes per side), SURVEY.md §8(a) rows a4 and a6:
//
//   k_fine3d_transport   I_p = sum_t c_t phi_t(x_t + .)           (Eq. 11, reading R9)
//                        b   = -P_n^T A_1 I_p                       (Eqs. 12/13 first lines, R5)
//                        g   = g^0 - C_1 I_p                        (Eqs. 12/13 second lines)
//   k_fine3d_combine     phi_p = P_n xi + I_p on K_p (for Eq. 7) and, for parents, on R_p^+
//
// PAPER.md:382-419.  The transported field I_p and A_1 I_p never leave the chip: one CTA per
// (child, rhs) walks the window plane by plane (z), forms I_p on plane z+1 from the parents' fine
// fields (L2-resident, read once per node), keeps three I planes in shared memory, applies the
// kappa-weighted Q1 element rows to the nodes of plane z (each thread owns a strip of 7 node rows
// of one column and slides a 3x3x3 register window along it), accumulates the constraint sums
// C_1 I_p per (subcell, continuum) from the cells' corner sums, and restricts A_1 I_p to the
// level-n nodes with the separable 1D hat weights (x and y per plane, z into two running level
// planes).  Every sum runs in a fixed order, so results are bitwise reproducible.
#include <cuda_runtime.h>

#include <cstdio>
#include <type_traits>

#include "device_common.cuh"
#include "kernels.h"

namespace {

constexpr int kFX = 49;                       // max fine nodes per side
constexpr int kFC = kFX - 1;                  // max fine cells per side
constexpr int kIP = kFX + 2;                  // padded I plane pitch (zero halo)
constexpr int kKP = kFC + 2;                  // padded kappa layer pitch (zero halo)
constexpr int kStrip = 7;                     // node rows per thread
constexpr int kFThreads = kFX * kStrip;       // 343 (49 columns x 7 strips)
constexpr int kFBlock = 352;                  // 11 warps

__device__ __forceinline__ int slot_f(const LevelArgs& A, const ProbDesc& P, int dim, int e) {
  return fdiv(P.lo[dim] + e + A.coff, A.inv_c) - P.k[dim] + A.l;  // subcell slot of fine cell e
}

}  // namespace

size_t fine3d_transport_smem(int N) {
  // I ring 4 x 51^2, kappa ring 3 x 50^2, ids ring 3 x 48^2 (bytes), z-restricted accumulators
  // 2 x 49^2, Yx 49 x 25, constraint partials, constraint sums
  const size_t d = 4 * kIP * kIP + 3 * kKP * kKP + 2 * kFX * kFX + kFX * 25 + (size_t)kFThreads * 3 * N + 27 * N;
  return d * sizeof(double) + 3 * kFC * kFC;
}

template <int N>
__global__ void __launch_bounds__(kFBlock, 1) k_fine3d_transport(LevelArgs A) {
  const int r = blockIdx.x / A.nprob_mp, mp = blockIdx.x - r * A.nprob_mp;  // rhs-major: siblings share parents in L2
  const ProbDesc& P = A.probs[mp];
  const int nx = P.ncf[0] + 1, ny = P.ncf[1] + 1, nz = P.ncf[2] + 1;
  const int ncx = nx - 1, ncy = ny - 1, ncz = nz - 1;
  const int s = A.s;
  const int nlx = P.nc[0] + 1, nly = P.nc[1] + 1;
  const int64_t n = A.n;
  const int tid = threadIdx.x;
  const int x = tid % kFX, strip = tid / kFX;
  const int y0 = strip * kStrip;
  const bool act = tid < kFThreads && x < nx && y0 < ny;
  const bool full_strip = act && y0 + kStrip <= ny;  // no row of the strip outside the window

  extern __shared__ __align__(16) double smem[];
  double* Ir = smem;                    // [4][51*51] I_p planes (slot = plane & 3), zero halo
  double* Kr = Ir + 4 * kIP * kIP;      // [3][50*50] kappa of cell layers (slot = (layer + 3) % 3), 0 outside
  double* Za = Kr + 3 * kKP * kKP;      // [2][49*49] A_1 I_p restricted in z to level plane Z (slot Z & 1)
  double* Yx = Za + 2 * kFX * kFX;      // [ny][nlx]
  double* cb = Yx + kFX * 25;           // [kFThreads][3][N] constraint partials
  double* cs = cb + kFThreads * 3 * N;  // [27][N] constraint sums
  uint8_t* Dr = reinterpret_cast<uint8_t*>(cs + 27 * N);  // [3][48*48] ids of cell layers
  for (int i = tid; i < 4 * kIP * kIP; i += blockDim.x) Ir[i] = 0.0;
  for (int i = tid; i < 3 * kKP * kKP; i += blockDim.x) Kr[i] = 0.0;
  for (int i = tid; i < 2 * kFX * kFX; i += blockDim.x) Za[i] = 0.0;
  for (int i = tid; i < 27 * N; i += blockDim.x) cs[i] = 0.0;

  // parents: per CTA table in shared memory (window origin's element in parent t at plane 0, row and
  // plane strides, weight); a thread adds its column offset y0 px + x at use (kept out of registers:
  // eight 64-bit bases, strides and weights per thread cost ~48 registers)
  const int npar = P.npar;
  __shared__ long long pbs[MCH_MAXPAR];
  __shared__ int pxs[MCH_MAXPAR], pxys[MCH_MAXPAR];
  __shared__ double pws[MCH_MAXPAR];
  if (tid < npar) {
    const int t = tid;
    const int px = P.par_ncf[t][0] + 1, py = P.par_ncf[t][1] + 1, pz = P.par_ncf[t][2] + 1;
    const int xt = P.lo[0] + (P.par_k[t][0] - P.k[0]) * A.c - P.par_lo[t][0];
    const int yt = P.lo[1] + (P.par_k[t][1] - P.k[1]) * A.c - P.par_lo[t][1];
    const int zt = P.lo[2] + (P.par_k[t][2] - P.k[2]) * A.c - P.par_lo[t][2];
    pxs[t] = px;
    pxys[t] = px * py;
    pbs[t] = P.par_pool[t] + (int64_t)r * px * py * pz + ((int64_t)zt * py + yt) * px + xt;
    pws[t] = P.par_w[t];
  }
  // global cell (x-1, y-1, z-1) of the window
  const int64_t cbase = ((int64_t)(P.lo[2] - 1) * n + (P.lo[1] - 1)) * n + (P.lo[0] - 1);
  // stage I_p on plane p: all loads of a group of up to four parents in flight before the first
  // use; the parent count is a compile-time constant per CTA (dispatch below), so no load slot is
  // predicated off
  auto stage_np = [&](auto npc, int p) {
    constexpr int NP = decltype(npc)::value;
    double* dst = Ir + (p & 3) * kIP * kIP + (y0 + 1) * kIP + (x + 1);
    double v[kStrip];
#pragma unroll
    for (int t0 = 0; t0 < NP; t0 += 4) {
      constexpr int G0 = 4;
      double raw[G0][kStrip];
#pragma unroll
      for (int u = 0; u < G0; u++) {
        const int t = t0 + u;
        if (t >= NP) break;
        const int px = pxs[t];
        const double* src = A.pool + pbs[t] + (p * pxys[t] + y0 * px + x);
        if (full_strip) {
#pragma unroll
          for (int i = 0; i < kStrip; i++) raw[u][i] = __ldg(src + i * px);
        } else {
#pragma unroll
          for (int i = 0; i < kStrip; i++) raw[u][i] = (y0 + i < ny) ? __ldg(src + i * px) : 0.0;
        }
      }
#pragma unroll
      for (int i = 0; i < kStrip; i++)
#pragma unroll
        for (int u = 0; u < G0; u++) {
          const int t = t0 + u;
          if (t >= NP) break;
          v[i] = (t == 0) ? pws[0] * raw[0][i] : v[i] + pws[t] * raw[u][i];
        }
    }
#pragma unroll
    for (int i = 0; i < kStrip; i++)
      if (y0 + i < ny) dst[i * kIP] = v[i];
  };
  auto stage_I = [&](int p) {
    if (!act || p >= nz) return;
    switch (npar) {
      case 1: stage_np(std::integral_constant<int, 1>{}, p); break;
      case 2: stage_np(std::integral_constant<int, 2>{}, p); break;
      case 3: stage_np(std::integral_constant<int, 3>{}, p); break;
      case 4: stage_np(std::integral_constant<int, 4>{}, p); break;
      case 5: stage_np(std::integral_constant<int, 5>{}, p); break;
      case 6: stage_np(std::integral_constant<int, 6>{}, p); break;
      case 7: stage_np(std::integral_constant<int, 7>{}, p); break;
      default: stage_np(std::integral_constant<int, 8>{}, p); break;
    }
  };
  // kappa and ids of cell layer cz (0 / 0xFF outside the window): loads into registers first, the
  // shared-memory stores after the stencil of the current plane (latency hidden behind it)
  const bool kact = act && x < ncx;
  double kreg[kStrip];
  int dreg[kStrip];
  auto load_K = [&](int cz) {
    const bool zin = kact && cz >= 0 && cz < ncz;
    const int64_t g0 = cbase + ((int64_t)(cz + 1) * n + (y0 + 1)) * n + (x + 1);
#pragma unroll
    for (int i = 0; i < kStrip; i++) {
      const bool ok = zin && y0 + i < ncy;
      kreg[i] = ok ? __ldg(A.kappa + g0 + (int64_t)i * n) : 0.0;
      dreg[i] = ok ? (int)__ldg(A.ids + g0 + (int64_t)i * n) : 0xFF;
    }
  };
  auto store_K = [&](int cz) {
    if (!kact) return;
    double* kd = Kr + ((cz + 3) % 3) * kKP * kKP + (y0 + 1) * kKP + (x + 1);
    uint8_t* dd = Dr + ((cz + 3) % 3) * kFC * kFC + y0 * kFC + x;
#pragma unroll
    for (int i = 0; i < kStrip; i++)
      if (y0 + i < ncy) {
        kd[i * kKP] = kreg[i];
        dd[i * kFC] = (uint8_t)dreg[i];
      }
  };

  // constraint partials: cell column x (subcell slot kx); the 7 rows of a strip lie in at most three
  // subcell rows ky0 + a (host: at least 4 fine cells per H); rows [0, i1) have a = 0, [i1, i2) a = 1
  const int kx = (act && x < ncx) ? slot_f(A, P, 0, x) : -1;
  const int ky0 = (act && y0 < ncy) ? slot_f(A, P, 1, y0) : -1;
  int i1 = kStrip, i2 = kStrip;
  for (int i = kStrip - 1; i >= 0; i--) {
    const int a = (act && y0 + i < ncy) ? slot_f(A, P, 1, y0 + i) - ky0 : 9;
    if (a >= 1) i1 = i;
    if (a >= 2) i2 = i;
  }
  double acc[3][N];
#pragma unroll
  for (int a = 0; a < 3; a++)
#pragma unroll
    for (int j = 0; j < N; j++) acc[a][j] = 0.0;
  // subcell slots of the cell columns and of the strips' first rows (-1: no cells), for flush()
  __shared__ int sxs[kFX], sys[kFX / kStrip];
  for (int u = tid; u < kFX; u += blockDim.x) sxs[u] = (u < ncx) ? slot_f(A, P, 0, u) : -1;
  for (int u = tid; u < kFX / kStrip; u += blockDim.x) sys[u] = (u * kStrip < ncy) ? slot_f(A, P, 1, u * kStrip) : -100;
  auto flush = [&](int kz) {
    double* mine = cb + tid * 3 * N;
    if (tid < kFThreads) {
#pragma unroll
      for (int a = 0; a < 3; a++)
#pragma unroll
        for (int j = 0; j < N; j++) {
          mine[a * N + j] = acc[a][j];
          acc[a][j] = 0.0;
        }
    }
    __syncthreads();
    // target (qy, qx, j) of layer kz: one warp each, fixed order over the threads
    const int lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;
    for (int tg = warp; tg < 9 * N; tg += nwarp) {
      const int j = tg % N, q2 = tg / N, qy = q2 / 3, qx = q2 % 3;
      double sum = 0.0;
      for (int u = lane; u < kFThreads; u += 32) {
        const int ust = u / kFX, ux = u - ust * kFX;
        if (sxs[ux] != qx) continue;
        const int a = qy - sys[ust];
        if (a >= 0 && a < 3) sum += cb[(u * 3 + a) * N + j];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(FULLMASK, sum, o);
      if (lane == 0) cs[((kz * 3 + qy) * 3 + qx) * N + j] += sum;
    }
    __syncthreads();
  };

  __syncthreads();
  stage_I(0);
  stage_I(1);
  load_K(0);
  store_K(0);
  __syncthreads();
  const double kh = A.h * (1.0 / 12.0);
  const double inv_s = 1.0 / (double)s;
  double* bvec = A.B + P.vec_off + (int64_t)r * nlx * nly * (P.nc[2] + 1);
  int Z0 = 0, rem = 0;  // level plane below z and z's offset above it (z = Z0 s + rem)
  for (int z = 0; z < nz; z++, rem = (rem + 1 == s) ? 0 : rem + 1, Z0 += (rem == 0) ? 1 : 0) {
    // stage plane z+2 and cell layer z+1 (slots not read in this iteration) while the stencil of
    // plane z runs: no barrier between the two
    load_K(z + 1);
    stage_I(z + 2);
    const double wlo = 1.0 - rem * inv_s, whi = rem * inv_s;
    if (act) {
      const double* pl[3] = {Ir + ((z + 3) & 3) * kIP * kIP, Ir + (z & 3) * kIP * kIP, Ir + ((z + 1) & 3) * kIP * kIP};
      const double* kl[2] = {Kr + ((z + 2) % 3) * kKP * kKP, Kr + (z % 3) * kKP * kKP};  // layers z-1, z
      const uint8_t* dl = Dr + (z % 3) * kFC * kFC;
      double* zlo = Za + (Z0 & 1) * kFX * kFX + x;        // level plane Z0
      double* zhi = Za + ((Z0 + 1) & 1) * kFX * kFX + x;  // level plane Z0 + 1
      double v[3][3][3];   // [dz][dy][dx]
      double kc[2][2][2];  // [oz][oy][ox]
      double apr[kStrip];  // A_1 I_p of the strip's nodes: the z-restriction read-modify-writes of the
                           // shared accumulators after the row loop, so no shared store sits between
                           // the rows' shared loads (the compiler cannot prove they do not alias)
      auto ld_row = [&](int yy, int slot) {
#pragma unroll
        for (int dz = 0; dz < 3; dz++)
#pragma unroll
          for (int dx = 0; dx < 3; dx++) {
            v[dz][slot][dx] = pl[dz][(yy + 1) * kIP + x + dx];  // zero halo / unwritten = outside
          }
      };
      auto ld_kap = [&](int cy, int slot) {  // cells of row cy, columns x-1, x; layers z-1, z
#pragma unroll
        for (int oz = 0; oz < 2; oz++)
#pragma unroll
          for (int ox = 0; ox < 2; ox++) {
            kc[oz][slot][ox] = kl[oz][(cy + 1) * kKP + x + ox];  // zero halo / unwritten = outside
          }
      };
      ld_row(y0 - 1, 0);
      ld_row(y0, 1);
      ld_kap(y0 - 1, 0);
      const bool cl = kx >= 0 && z < ncz;  // this column has cells in layer z
#pragma unroll
      for (int i = 0; i < kStrip; i++) {
        const int y = y0 + i;
        if (y >= ny) break;
        ld_row(y + 1, 2);
        ld_kap(y, 1);
        // (A_1 I)_node = h/12 sum over the 8 cells o around the node of kappa_o (4 v_node - the
        // node's two face-diagonal and one body-diagonal partners in o ... as 4 terms a^3, a^5, a^6,
        // a^7 of the cell-local corner a): octant terms formed independently, summed as a tree
        const double c4 = 4.0 * v[1][1][1];
        double t[8];
#pragma unroll
        for (int o = 0; o < 8; o++) {
          const int ox = o & 1, oy = (o >> 1) & 1, oz = o >> 2;
          const int a = (~o) & 7;
          auto vb = [&](int b) { return v[oz + ((b >> 2) & 1)][oy + ((b >> 1) & 1)][ox + (b & 1)]; };
          t[o] = kc[oz][oy][ox] * ((c4 - (vb(a ^ 3) + vb(a ^ 5))) - (vb(a ^ 6) + vb(a ^ 7)));
        }
        const double Ap = (((t[0] + t[1]) + (t[2] + t[3])) + ((t[4] + t[5]) + (t[6] + t[7]))) * kh;
        apr[i] = Ap;
        // cell (x, y, z): corners on planes z, z+1, rows y, y+1, columns x, x+1
        if (cl && y < ncy) {
          const double sig = ((v[1][1][1] + v[1][1][2]) + (v[1][2][1] + v[1][2][2])) +
                             ((v[2][1][1] + v[2][1][2]) + (v[2][2][1] + v[2][2][2]));
          const int id = dl[y * kFC + x];
          const int a = (i < i1) ? 0 : ((i < i2) ? 1 : 2);
#pragma unroll
          for (int j = 0; j < N; j++) {
            const double tj = (id == j) ? sig : 0.0;
            if (a == 0) acc[0][j] += tj;
            else if (a == 1) acc[1][j] += tj;
            else acc[2][j] += tj;
          }
        }
#pragma unroll
        for (int dz = 0; dz < 3; dz++)
#pragma unroll
          for (int dx = 0; dx < 3; dx++) {
            v[dz][0][dx] = v[dz][1][dx];
            v[dz][1][dx] = v[dz][2][dx];
          }
#pragma unroll
        for (int oz = 0; oz < 2; oz++)
#pragma unroll
          for (int ox = 0; ox < 2; ox++) kc[oz][0][ox] = kc[oz][1][ox];
      }
      // z restriction (1D hat of level plane Z0 and Z0 + 1) into the accumulators; x and y once per
      // completed level plane below
#pragma unroll
      for (int i = 0; i < kStrip; i++) {
        const int y = y0 + i;
        if (y >= ny) break;
        zlo[y * kFX] += wlo * apr[i];
        if (rem > 0) zhi[y * kFX] += whi * apr[i];
      }
    }
    store_K(z + 1);
    // constraint layer complete after cell layer z?
    if (z < ncz) {
      const int kz = slot_f(A, P, 2, z);
      if (z + 1 == ncz || slot_f(A, P, 2, z + 1) != kz) flush(kz);
    }
    // level plane Z0 complete: restrict it in x, then y, into b; its accumulator slot is zeroed for
    // level plane Z0 + 2 (first written at plane (Z0 + 1) s + 1, after the barriers below)
    if (rem == s - 1 || z == nz - 1) {
      __syncthreads();
      const double* zp = Za + (Z0 & 1) * kFX * kFX;
      for (int u = tid; u < ny * nlx; u += blockDim.x) {
        const int y = u / nlx, X = u - y * nlx, c0 = X * s;
        const double* row = zp + y * kFX;
        double a = row[c0];
        for (int d = 1; d < s; d++) {
          const double w = 1.0 - d * inv_s;
          if (c0 - d >= 0) a += w * row[c0 - d];
          if (c0 + d < nx) a += w * row[c0 + d];
        }
        Yx[y * nlx + X] = a;
      }
      __syncthreads();
      for (int u = tid; u < nly * nlx; u += blockDim.x) {
        const int Yl = u / nlx, X = u - Yl * nlx, c0 = Yl * s;
        double a = Yx[c0 * nlx + X];
        for (int d = 1; d < s; d++) {
          const double w = 1.0 - d * inv_s;
          if (c0 - d >= 0) a += w * Yx[(c0 - d) * nlx + X];
          if (c0 + d < ny) a += w * Yx[(c0 + d) * nlx + X];
        }
        bvec[((int64_t)Z0 * nly + Yl) * nlx + X] = -a;
      }
      double* zw = Za + (Z0 & 1) * kFX * kFX;
      for (int u = tid; u < kFX * kFX; u += blockDim.x) zw[u] = 0.0;
    }
    __syncthreads();  // staged plane z+2 / layer z+1 visible from here on
  }
  const double hq = 0.125 * A.h * A.h * A.h;
  for (int i = tid; i < 27 * N; i += blockDim.x) {
    const int64_t gi = ((int64_t)mp * A.ncon + i) * A.n_rhs + r;
    A.g[gi] = A.g0[gi] - cs[i] * hq;
  }
}

cudaError_t launch_fine3d_transport(const LevelArgs& A, cudaStream_t st) {
  if (A.ncon != 27 * A.N) return cudaErrorInvalidValue;
  const size_t smem = fine3d_transport_smem(A.N);
  auto go = [&](auto k) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k<<<(unsigned)(A.nprob_mp * A.n_rhs), kFBlock, smem, st>>>(A);
    return cudaGetLastError();
  };
  switch (A.N) {
    case 1: return go(k_fine3d_transport<1>);
    case 2: return go(k_fine3d_transport<2>);
    case 3: return go(k_fine3d_transport<3>);
    case 4: return go(k_fine3d_transport<4>);
  }
  return cudaErrorInvalidValue;
}

// ------------------------------------------------------------------------------------------
// phi_p = P_n xi + I_p (Eq. 11) for all right-hand sides of a macropoint: on the K_p node box
// into FK (read by k_gram for Eq. 7), and on the whole window into the parent pool if p is
// stored (parents of later levels, or keep_all).  I_p is formed again from the parents (the
// transport kept it on chip); per value the arithmetic is k_combine's.
__global__ void __launch_bounds__(256, 3) k_fine3d_combine(LevelArgs A) {
  const int mp = blockIdx.y;
  const ProbDesc& P = A.probs[mp];
  const Geo<3> gf = fine_geo<3>(P);
  const Geo<3> gl = level_geo<3>(A, P);
  const int s = A.s, nr = A.n_rhs;
  const int64_t nnf = gf.nnodes, nnl = gl.nnodes;
  int klo[3], kn[3];
  for (int i = 0; i < 3; i++) {
    klo[i] = P.kp_lo[i] - P.lo[i];
    kn[i] = P.kp_hi[i] - P.kp_lo[i] + 1;
  }
  const int nkp = kn[0] * kn[1] * kn[2];
  const bool full = P.pool_off >= 0;
  const int cnt = full ? (int)nnf : nkp;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= cnt) return;
  int xf[3];
  if (full) {
    node_xyz<3>(gf, k, xf);
  } else {
    const int zz = k / (kn[0] * kn[1]), t = k - zz * kn[0] * kn[1], yy = t / kn[0];
    xf[0] = klo[0] + t - yy * kn[0];
    xf[1] = klo[1] + yy;
    xf[2] = klo[2] + zz;
  }
  const int kf = node_id<3>(gf, xf);
  // K_p box index (-1 outside)
  int kk = -1;
  {
    const int a = xf[0] - klo[0], b = xf[1] - klo[1], c = xf[2] - klo[2];
    if (a >= 0 && a < kn[0] && b >= 0 && b < kn[1] && c >= 0 && c < kn[2]) kk = (c * kn[1] + b) * kn[0] + a;
  }
  int c0[3];
  double t[3];
  for (int i = 0; i < 3; i++) {
    c0[i] = xf[i] / s;
    t[i] = (double)(xf[i] - c0[i] * s) / s;
    if (c0[i] == gl.nc[i]) { c0[i] -= 1; t[i] = 1.0; }
  }
  double wgt[8];
  int nid[8];
#pragma unroll
  for (int a = 0; a < 8; a++) {
    double w = 1.0;
    int xc[3];
    for (int i = 0; i < 3; i++) {
      const int ai = (a >> i) & 1;
      w *= ai ? t[i] : 1.0 - t[i];
      xc[i] = c0[i] + ai;
    }
    wgt[a] = w;
    nid[a] = node_id<3>(gl, xc);
  }
  // right-hand sides in chunks of four (80 registers: three CTAs per SM): per parent (runtime loop, index formed in place) the
  // loads of all eight rhs are in flight together, I accumulated in registers (one rhs at a time
  // left the loop long-scoreboard bound); the coarse-node values (L1-resident) are read at use
  constexpr int RC = 4;
  for (int r0 = 0; r0 < nr; r0 += RC) {
    double Iv[RC];
#pragma unroll
    for (int u = 0; u < RC; u++) Iv[u] = 0.0;
    for (int q = 0; q < P.npar; q++) {
      int64_t idx = 0;
      for (int i = 2; i >= 0; i--) {
        const int xt = P.lo[i] + xf[i] + (P.par_k[q][i] - P.k[i]) * A.c - P.par_lo[q][i];
        idx = idx * (P.par_ncf[q][i] + 1) + xt;
      }
      const int pn = (P.par_ncf[q][0] + 1) * (P.par_ncf[q][1] + 1) * (P.par_ncf[q][2] + 1);
      const double* src = A.pool + P.par_pool[q] + idx + (int64_t)r0 * pn;
      const double w = P.par_w[q];
      double pv[RC];
#pragma unroll
      for (int u = 0; u < RC; u++) pv[u] = (r0 + u < nr) ? __ldg(src + (int64_t)u * pn) : 0.0;
#pragma unroll
      for (int u = 0; u < RC; u++) Iv[u] += w * pv[u];
    }
#pragma unroll
    for (int u = 0; u < RC; u++) {
      const int r = r0 + u;
      if (r >= nr) break;
      const double* xi = A.X + P.vec_off + (int64_t)r * nnl;
      double v = 0.0;
#pragma unroll
      for (int a = 0; a < 8; a++)
        if (wgt[a] != 0.0) v += wgt[a] * xi[nid[a]];
      const double phi = Iv[u] + v;
      if (kk >= 0) A.FK[((int64_t)mp * nr + r) * A.nkp_max + kk] = phi;
      if (full) A.pool[P.pool_off + (int64_t)r * nnf + kf] = phi;
    }
  }
}

cudaError_t launch_fine3d_combine(const LevelArgs& A, int max_fine_nodes, cudaStream_t st) {
  dim3 grid((unsigned)((max_fine_nodes + 255) / 256), (unsigned)A.nprob_mp);
  k_fine3d_combine<<<grid, 256, 0, st>>>(A);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// Eq. (7) on the fused 3D path (R_p = K_p, prefactor 1: reading R12):
// G[a][b] = sum over the fine cells e of K_p of kappa_e (phi_a|_e)^T K_e (phi_b|_e), all NR
// right-hand sides of a macropoint in one pass over the cells (k_gram re-reads every cell per a).
// K_e is the Q1 element stiffness of a cube of side h: (K_e v)_c = h/12 (4 v_c - the four corners
// that differ from c in >= 2 coordinates) = h/12 (5 v_c - E_{par(c)} - v_{c^7}), E_par the sum over
// the four corners of c's parity.  Fixed-order block reduction: bitwise reproducible.
template <int NR>
__global__ void __launch_bounds__(256) k_gram3_kp(LevelArgs A) {
  const int mp = blockIdx.x;
  const ProbDesc& P = A.probs[mp];
  __shared__ double scratch[32 * (NR * (NR + 1) / 2)];
  __shared__ double tot[NR * (NR + 1) / 2];
  constexpr int NP = NR * (NR + 1) / 2;
  int lo[3], ext[3];
  for (int i = 0; i < 3; i++) {
    lo[i] = P.kp_lo[i] - P.lo[i];
    ext[i] = P.kp_hi[i] - P.kp_lo[i];
  }
  const int kn0 = ext[0] + 1, kn1 = ext[1] + 1;
  const int cnt = ext[0] * ext[1] * ext[2];
  const double* F = A.FK + (int64_t)mp * NR * A.nkp_max;
  const double kh = A.h * (1.0 / 12.0);
  double acc[NP];
#pragma unroll
  for (int i = 0; i < NP; i++) acc[i] = 0.0;
  for (int idx = threadIdx.x; idx < cnt; idx += blockDim.x) {
    const int ex = idx % ext[0], ey = (idx / ext[0]) % ext[1], ez = idx / (ext[0] * ext[1]);
    const int64_t gc = ((int64_t)(P.kp_lo[2] + ez) * A.n + (P.kp_lo[1] + ey)) * A.n + (P.kp_lo[0] + ex);
    const double w = __ldg(A.kappa + gc) * kh;
    const int base = (ez * kn1 + ey) * kn0 + ex;
    int nid[8];
#pragma unroll
    for (int c = 0; c < 8; c++) nid[c] = base + (c & 1) + ((c >> 1) & 1) * kn0 + ((c >> 2) & 1) * kn0 * kn1;
    double ph[NR][8];
#pragma unroll
    for (int r = 0; r < NR; r++)
#pragma unroll
      for (int c = 0; c < 8; c++) ph[r][c] = F[(int64_t)r * A.nkp_max + nid[c]];
    int pi = 0;
#pragma unroll
    for (int a = 0; a < NR; a++) {
      const double ev = ph[a][0] + ph[a][3] + ph[a][5] + ph[a][6];  // even-parity corners
      const double od = ph[a][1] + ph[a][2] + ph[a][4] + ph[a][7];
      double y[8];
#pragma unroll
      for (int c = 0; c < 8; c++) {
        const bool evn = ((c ^ (c >> 1) ^ (c >> 2)) & 1) == 0;
        y[c] = w * (5.0 * ph[a][c] - (evn ? ev : od) - ph[a][c ^ 7]);
      }
#pragma unroll
      for (int b = a; b < NR; b++, pi++) {
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < 8; c++) s += y[c] * ph[b][c];
        acc[pi] += s;
      }
    }
  }
  block_sum<NP>(acc, scratch, tot);
  if (threadIdx.x == 0) {
    double* Gout = A.G + P.lin * NR * NR;
    int pi = 0;
    for (int a = 0; a < NR; a++)
      for (int b = a; b < NR; b++, pi++) {
        Gout[a * NR + b] = tot[pi];
        Gout[b * NR + a] = tot[pi];
      }
  }
}

cudaError_t launch_gram3_kp(const LevelArgs& A, cudaStream_t st) {
  switch (A.n_rhs) {
    case 4: k_gram3_kp<4><<<A.nprob_mp, 256, 0, st>>>(A); break;
    case 8: k_gram3_kp<8><<<A.nprob_mp, 256, 0, st>>>(A); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}
