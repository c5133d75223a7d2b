// 3D level-1 projected PCG with a thread-block cluster per problem (sm_100a).
//
// Same method and arithmetic per node as k_pcg3d_l1 (pcg3d.cu): for each problem (macropoint p,
// right-hand side r) the constrained cell problem of Eqs. (3)/(4) on the fine
// window, projected Jacobi-PCG with the residual re-projected every iteration and the two-level
// (inclusion coarse space) preconditioner (readings R16, R19).
//
// A 49^3 window does not fit on chip, and one CTA per problem leaves the
// iteration latency-bound: config 5 has 216 problems on 148 SMs (1.46 waves) and its slowest
// problem sets the level time.  Here a cluster of CS CTAs shares one problem: CTA c walks the
// node planes z in [c nz / CS, (c+1) nz / CS) (each with all 98 row tasks of the plane), p, r, q, x
// stay in global memory (L2), the p planes at the slab boundaries are read from the neighbour's
// slab after the cluster barrier (barrier.cluster also invalidates L1, so they come from L2), and
// every reduction — the scalars rz, pq, rr and the constraint vector c = C D^-1 r — is formed per
// CTA, published in shared memory and summed over the cluster's CTAs in rank order through DSMEM.
// Three cluster barriers per iteration; every CTA then holds identical scalars, so all take the same
// branch and the projector solve (S^+ c) is done redundantly per CTA.  Fixed summation orders
// throughout: bitwise reproducible.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "kernels.h"
#include "pcg3d_common.cuh"

#ifndef MCH_L1_NW
#define MCH_L1_NW 14  // warps per CTA of the level-1 cluster kernel (98 row tasks of a 49-node window: 7 per warp)
#endif
#ifndef MCH_L1_NW2
#define MCH_L1_NW2 20  // the same for a cluster of two (half the planes per CTA): 20 warps at 96 registers, c5 level-1 PCG 44.5 -> 42.6 ms (25 warps at 72 registers: 52 ms; one CTA per problem, config 4: 14 warps 373 ms, 20 warps 386 ms)
#endif
#ifndef MCH_P25_RW
#define MCH_P25_RW 1  // node rows per warp of the 25-node cluster kernel (1: 25 warps at 72 registers, c5 level-2 PCG 35.4 -> 33.1 ms)
#endif
#ifndef MCH_P25_MINB
#define MCH_P25_MINB 1  // CTAs per SM of the 25-node cluster kernel (2: 72 registers, 968 B spills, 44 -> 69 ms)
#endif

namespace cg = cooperative_groups;

namespace {
struct VA { double r, p, x, d; int cm; };  // pass A loads of one node
struct VC { double r, q, d; };             // pass C loads
struct VX { double x, d; int cm; };        // x / D^-1 / component of one node
}  // namespace

template <int N, int NW, int CS>
__global__ void __launch_bounds__(NW * 32, (NW * 32 <= 448) ? 448 / (NW * 32) : 1) k_pcg3d_l1c(LevelArgs A) {
  constexpr int NT = 98;  // at most 98 row tasks = 49 rows x 2 segments
  constexpr int NQ = 27 * N;
  cg::cluster_group cl = cg::this_cluster();
  const int cr = (int)cl.block_rank();
  const int prob = blockIdx.x / CS;
  const int mp = prob / A.n_rhs, rhs = prob - mp * A.n_rhs;
  const ProbDesc& P = A.probs[mp];
  const int* ncv = P.nc;
  const int nx = ncv[0] + 1, ny = ncv[1] + 1, nz = ncv[2] + 1, nn = nx * ny * nz;
  const int ncx = nx - 1, ncy = ny - 1, ncz = nz - 1;
  const int nc = A.ncon;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int z0 = (cr * nz) / CS, z1 = ((cr + 1) * nz) / CS;  // this CTA's node planes

  extern __shared__ __align__(16) double smem[];
  double* bins = smem;          // [NT task rows][NQ]
  double* Ysh = bins + NT * NQ;  // [NQ]
  double* csh = Ysh + NQ;        // [NQ]
  double* slots = csh + NQ;      // [5][32]
  double* zr = slots + 5 * 32;   // [256] coarse: E^-1 Z^T r
  double* vv = zr + 256;         // [256] coarse: coarse part of z
  double* red = vv + 256;        // [3][NQ + 2] cluster reduction buffers (published partials)
  int* zsm = reinterpret_cast<int*>(red + 3 * (NQ + 2));  // [49][3]
  __shared__ double bc[2];       // broadcast scalars
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
  unsigned pvm = 0;   // bit dy*3+dx: p neighbour (x+dx-1, y+dy-1) inside the window
  unsigned cvm = 0;   // bit oy*2+ox: cell (x-1+ox, y-1+oy) inside the window
  int64_t cbase = 0;  // global index of cell (x-1, y-1, -1) of the window
  auto tside = [](int pm, int ob) { return (pm == 3) ? ob : ((pm == 2) ? 1 : 0); };
  auto kxy = [&](int oxy) {
    const int ox = oxy & 1, oy = oxy >> 1;
    const int kx = ox ? ((sx.pm == 1) ? sx.k0 : sx.k1) : sx.k0;
    const int ky = oy ? ((sy.pm == 1) ? sy.k0 : sy.k1) : sy.k0;
    return ky * 3 + kx;
  };
  int kq[4];
  // row tasks of this window: nseg x-segments of 32 lanes per node row (1 if nx <= 32), dealt
  // round-robin to the warps so a clipped window keeps every warp busy
  const int nseg = (nx + 31) >> 5, ntask = ny * nseg;
  auto set_task = [&](int tt) {
    t = tt;
    y = t / nseg;
    seg = t - y * nseg;
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
#pragma unroll
    for (int o = 0; o < 4; o++) kq[o] = kxy(o);
  };
  auto tasks = [&](auto&& f) {
    for (int tt = warp; tt < ntask; tt += NW) {
      set_task(tt);
      f();
    }
  };

  const double* dg = A.dinv + P.node_off;
  double* pv = A.P + P.vec_off + (int64_t)rhs * nn;
  double* Xv = A.X + P.vec_off + (int64_t)rhs * nn;
  double* Rv = A.R + P.vec_off + (int64_t)rhs * nn;
  double* Qv = A.Q + P.vec_off + (int64_t)rhs * nn;
  const double* Si = A.Sinv + (int64_t)mp * nc * nc;
  const double hq = 0.125 * A.h * A.h * A.h, kh = A.h * (1.0 / 12.0);

  // column walker over this CTA's planes z in [z0, z1): f(z, k, id[8]) with id[o] of cell octant o
  auto walk_ids = [&](auto&& f) {
    int idc[8];
    const int oxy[4] = {0, 1, (int)A.n, (int)A.n + 1};
    const uint8_t* ip = A.ids + cbase + (int64_t)(z0 + 1) * n2;  // cell layer z0
#pragma unroll
    for (int o = 0; o < 4; o++) {
      idc[o] = (((cvm >> o) & 1u) && z0 >= 1) ? __ldg(ip - n2 + oxy[o]) : 0xFF;   // layer z0 - 1
      idc[4 + o] = (((cvm >> o) & 1u) && z0 < ncz) ? __ldg(ip + oxy[o]) : 0xFF;  // layer z0
    }
    int k = (z0 * ny + y) * nx + x;
    for (int z = z0; z < z1; z++) {
      ip += n2;
      const bool nv = z + 1 < ncz;
      int nxt[4];
#pragma unroll
      for (int o = 0; o < 4; o++) nxt[o] = (((cvm >> o) & 1u) && nv) ? __ldg(ip + oxy[o]) : 0xFF;
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

  // walker with the loads of the next DP-1 node planes in flight: pre(k, live) -> V is issued DP-1
  // steps ahead of f(z, k, idc, V) (the z-walk is otherwise one memory round trip per plane)
  constexpr int DP = 3;
  auto walk_pf = [&](auto&& pre, auto&& f) {
    using V = decltype(pre(0, false));
    V ring[DP];
    int idq[DP][4];
    const int oxy[4] = {0, 1, (int)A.n, (int)A.n + 1};
    const uint8_t* ip0 = A.ids + cbase + (int64_t)(z0 + 1) * n2;  // cell layer z0
    int lo4[4];
#pragma unroll
    for (int o = 0; o < 4; o++) lo4[o] = (((cvm >> o) & 1u) && z0 >= 1) ? __ldg(ip0 - n2 + oxy[o]) : 0xFF;
    auto issue = [&](V& slot, int (&iq)[4], int z) {
      const bool live = z < z1;
      slot = pre((z * ny + y) * nx + x, live && lact);
      const uint8_t* ip = ip0 + (int64_t)(z - z0) * n2;
#pragma unroll
      for (int o = 0; o < 4; o++) iq[o] = (live && ((cvm >> o) & 1u) && z < ncz) ? __ldg(ip + oxy[o]) : 0xFF;
    };
#pragma unroll
    for (int d = 0; d < DP - 1; d++) issue(ring[d], idq[d], z0 + d);
    for (int zb = z0; zb < z1; zb += DP) {
#pragma unroll
      for (int d = 0; d < DP; d++) {
        const int z = zb + d;
        if (z < z1) {
          issue(ring[(d + DP - 1) % DP], idq[(d + DP - 1) % DP], z + DP - 1);
          int idc[8];
#pragma unroll
          for (int o = 0; o < 4; o++) {
            idc[o] = lo4[o];
            idc[4 + o] = idq[d][o];
            lo4[o] = idq[d][o];
          }
          f(z, (z * ny + y) * nx + x, idc, ring[d]);
        }
      }
    }
  };

  double acc[4][N];
  auto acc_zero = [&]() {
#pragma unroll
    for (int a = 0; a < 4; a++)
#pragma unroll
      for (int j = 0; j < N; j++) acc[a][j] = 0.0;
  };
  auto acc_add = [&](int zsel, int z, const int (&idc)[8], double u) {
    const int pmz = zsm[z * 3];
    const double w = u * hq;
#pragma unroll
    for (int oz = 0; oz < 2; oz++) {
      if (tside(pmz, oz) != zsel) continue;
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
      if (!((sy.pm >> ys) & 1)) continue;
      const int ky = ys ? sy.k1 : sy.k0;
      double g[2][N];
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
      if (lane == 0 && lact && x >= 1) {
#pragma unroll
        for (int j = 0; j < N; j++) B[((kz * 3 + ky) * 3 + sx.k0) * N + j] += g[0][j];
      }
      __syncwarp();
    }
    acc_zero();
  };
  // constraint sums of u over this CTA's planes into the task bins (zeroed first)
  auto sweep_c = [&](auto&& ufun) {
    for (int i = lane; i < NQ; i += 32) bins[t * NQ + i] = 0.0;
    __syncwarp();
    acc_zero();
    int layer = -1;
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
    if (layer >= 0) flush(layer);
  };
  // sweep_c with pipelined loads: u = ufun(z, k, V)
  auto sweep_c_pf = [&](auto&& pre, auto&& ufun) {
    for (int i = lane; i < NQ; i += 32) bins[t * NQ + i] = 0.0;
    __syncwarp();
    acc_zero();
    int layer = -1;
    walk_pf(pre, [&](int z, int k, const int (&idc)[8], const auto& V) {
      const double u = ufun(z, k, V);
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
    if (layer >= 0) flush(layer);
  };
  // (A p)_k over this CTA's planes; p planes z0 - 1 and z1 belong to the neighbours (L2 loads)
  auto sweep_stencil = [&](auto&& f) {
    const double* pz = pv + (int64_t)z0 * nxy + y * nx + x;
    const double* kp = A.kappa + cbase + (int64_t)(z0 + 1) * n2;  // cells of layer z0
    const int oxy[4] = {0, 1, (int)A.n, (int)A.n + 1};
    int poff[9];
#pragma unroll
    for (int dy = 0; dy < 3; dy++)
#pragma unroll
      for (int dx = 0; dx < 3; dx++) poff[dy * 3 + dx] = (dy - 1) * nx + (dx - 1);
    double v[3][3][3];
    double kc[2][2][2];
#pragma unroll
    for (int dy = 0; dy < 3; dy++)
#pragma unroll
      for (int dx = 0; dx < 3; dx++) {
        const bool in = (pvm >> (dy * 3 + dx)) & 1u;
        v[0][dy][dx] = (in && z0 >= 1) ? __ldcg(pz - nxy + poff[dy * 3 + dx]) : 0.0;
        v[1][dy][dx] = in ? pz[poff[dy * 3 + dx]] : 0.0;
      }
#pragma unroll
    for (int o = 0; o < 4; o++) {
      const bool in = (cvm >> o) & 1u;
      kc[0][o >> 1][o & 1] = (in && z0 >= 1) ? __ldg(kp - n2 + oxy[o]) : 0.0;
      kc[1][o >> 1][o & 1] = (in && z0 < ncz) ? __ldg(kp + oxy[o]) : 0.0;
    }
    int k = (z0 * ny + y) * nx + x;
    for (int z = z0; z < z1; z++) {
      pz += nxy;
      kp += n2;
      const bool pn = z + 1 < nz, cn = z + 1 < ncz, halo = z + 1 >= z1;
#pragma unroll
      for (int dy = 0; dy < 3; dy++)
#pragma unroll
        for (int dx = 0; dx < 3; dx++) {
          const bool in = ((pvm >> (dy * 3 + dx)) & 1u) && pn;
          const double* a = pz + poff[dy * 3 + dx];
          v[2][dy][dx] = in ? (halo ? __ldcg(a) : *a) : 0.0;
        }
      double kn[4];
#pragma unroll
      for (int o = 0; o < 4; o++) kn[o] = (((cvm >> o) & 1u) && cn) ? __ldg(kp + oxy[o]) : 0.0;
      double Ap = 0.0;
#pragma unroll
      for (int o = 0; o < 8; o++) {
        const int ox = o & 1, oy = (o >> 1) & 1, oz = o >> 2;
        const int a = (~o) & 7;
        auto pv_b = [&](int b) { return v[oz + ((b >> 2) & 1)][oy + ((b >> 1) & 1)][ox + (b & 1)]; };
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
  // cluster reductions: CTA partials published in red[b][0..m), summed over ranks in rank order
  auto publish = [&](int b, int i, double v) { red[b * (NQ + 2) + i] = v; };
  auto cluster_sum = [&](int b, int i) -> double {
    double s = 0.0;
#pragma unroll
    for (int r = 0; r < CS; r++) s += *cl.map_shared_rank(red + b * (NQ + 2) + i, r);
    return s;
  };
  // csh = [sub -] cluster sum of the constraint bins (publish, cluster barrier, gather)
  auto reduce_c_pub = [&](int b) {  // per CTA: bins over task rows -> red[b][0..nc)
    for (int i = warp; i < nc; i += NW) {
      double s = 0.0;
      for (int tt = lane; tt < NT; tt += 32) s += bins[tt * NQ + i];
      s = wsum0(s);
      if (lane == 0) publish(b, i, s);
    }
  };
  auto gather_c = [&](int b, const double* sub) {
    for (int i = threadIdx.x; i < nc; i += blockDim.x) {
      const double s = cluster_sum(b, i);
      csh[i] = sub ? sub[((int64_t)mp * nc + i) * A.n_rhs + rhs] - s : s;
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

  const bool crs = A.coarse && A.ncomp[mp] > 0;
  const int nca = crs ? A.ncomp[mp] : 0;
  const int* cmp = A.cmap + P.node_off;
  const int* cpt = A.cptr + (int64_t)mp * (A.ncmax + 1);
  const int* cls = A.clist + P.node_off;
  // coarse data staged in shared memory once: CZ [nc][nca] and E^-1 [nca]
  double* czs = reinterpret_cast<double*>(zsm + 3 * 49 + 1) ;
  czs = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(czs) + 15) & ~uintptr_t(15));
  double* eis = czs + (size_t)nc * nca;
  if (crs) {
    const double* CZm = A.CZ + (int64_t)mp * nc * A.ncmax;
    for (int i = threadIdx.x; i < nc * nca; i += blockDim.x) {
      const int tq = i / nca, a = i - tq * nca;
      czs[i] = __ldg(CZm + (int64_t)tq * A.ncmax + a);
    }
    for (int a = threadIdx.x; a < nca; a += blockDim.x) eis[a] = __ldg(A.Einv + (int64_t)mp * A.ncmax + a);
    __syncthreads();
  }
  // zr = E^-1 Z^T R over every component (redundant per CTA; R of the whole window is complete
  // after the preceding cluster barrier): 4 lanes per component, up to 32 node loads in flight per
  // lane before the fixed-order sums; slot 4, then csh += (CZ) zr.  Two block barriers.
  auto coarse_c = [&]() {
    double part = 0.0;
    const int sub = lane & 3, ngrp = blockDim.x >> 2;
    for (int a0 = threadIdx.x >> 2; a0 - (int)(threadIdx.x >> 2) < nca; a0 += ngrp) {
      const int a = a0;
      double sv = 0.0;
      if (a < nca) {
        const int i0 = __ldg(cpt + a), i1 = __ldg(cpt + a + 1);
        for (int ib = i0 + sub; ib < i1; ib += 4 * 8) {
          double rv[8];
#pragma unroll
          for (int u = 0; u < 8; u++) {
            const int i = ib + 4 * u;
            rv[u] = (i < i1) ? __ldcg(Rv + __ldg(cls + i)) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 8; u++) sv += rv[u];
        }
      }
      sv += __shfl_xor_sync(FULLMASK, sv, 1);
      sv += __shfl_xor_sync(FULLMASK, sv, 2);
      if (a < nca && sub == 0) {
        const double ei = eis[a];
        zr[a] = sv * ei;
        part += sv * sv * ei;
      }
    }
    part = wsum0(part);
    if (lane == 0) slots[4 * 32 + warp] = part;
    __syncthreads();
    for (int tq = warp; tq < nc; tq += NW) {
      double sv = 0.0;
      for (int a = lane; a < nca; a += 32) sv += czs[tq * nca + a] * zr[a];
      sv = wsum0(sv);
      if (lane == 0) csh[tq] += sv;
    }
    __syncthreads();
  };
  // vv = s0 zr - E^-1 (CZ)^T Ysh: one warp per component, lanes over the constraint rows.  One barrier.
  auto coarse_v = [&](double s0) {
    for (int a = warp; a < nca; a += NW) {
      double ac = 0.0;
      for (int tq = lane; tq < nc; tq += 32) ac += czs[tq * nca + a] * Ysh[tq];
      ac = wsum0(ac);
      if (lane == 0) vv[a] = (s0 != 0.0 ? s0 * zr[a] : 0.0) - eis[a] * ac;
    }
    __syncthreads();
  };
  auto cz_at = [&](int k) -> double {
    if (!crs) return 0.0;
    const int a = __ldg(cmp + k);
    return (a >= 0) ? vv[a] : 0.0;
  };

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
  cl.sync();  // x0 (= p) complete over the cluster
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
  reduce_c_pub(2);
  if (warp == 0) {
    const double v = slot_fin(2);
    if (lane == 0) publish(2, NQ, v);
  }
  cl.sync();  // partials published; R complete (coarse_c reads it)
  gather_c(2, nullptr);
  if (threadIdx.x == 0) bc[0] = cluster_sum(2, NQ);
  __syncthreads();
  if (crs) coarse_c();
  solve_y();
  __syncthreads();
  rr0 = bc[0] + (crs ? slot_fin(4) : 0.0);
  if (crs) coarse_v(1.0);

  const double tol2 = A.rtol * A.rtol;
  const double floor2 = 1e-30 * rr0;
  double beta = 0.0, rz = 0.0, ref = 0.0, alpha = 0.0;
  int it = 0, breakdown = 0;
  for (;; it++) {
    // pass A: x += alpha_prev p_prev, r <- r - C^T yhat, z = M^-1 r, p <- -z + beta p
    double v = 0.0;
    const bool first = (it == 0);
    tasks([&] {
      if (!wact) return;
      walk_pf(
          [&](int k, bool live) {
            VA a;
            a.r = live ? Rv[k] : 0.0;
            a.p = (live && !first) ? pv[k] : 0.0;
            a.x = (live && !first) ? Xv[k] : 0.0;
            a.d = live ? dg[k] : 0.0;
            a.cm = (live && crs) ? __ldg(cmp + k) : -1;
            return a;
          },
          [&](int z, int k, const int (&idc)[8], const VA& a) {
            if (!lact) return;
            const double rk = a.r - ct_of(z, idc);
            const double zz = a.d * rk + ((a.cm >= 0) ? vv[a.cm] : 0.0);
            if (!first) Xv[k] = a.x + alpha * a.p;
            pv[k] = first ? -zz : -zz + beta * a.p;
            Rv[k] = rk;
            v += rk * zz;
          });
    });
    slot_put(0, v);
    __syncthreads();
    if (warp == 0) {
      const double s = slot_fin(0);
      if (lane == 0) publish(0, 0, s);
    }
    cl.sync();  // S1: p complete over the cluster, rz partials published
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
    if (threadIdx.x == 0) bc[0] = cluster_sum(0, 0);
    __syncthreads();
    if (warp == 0) {
      const double s = slot_fin(1);
      if (lane == 0) publish(1, 0, s);
    }
    cl.sync();  // S2: pq partials published
    if (threadIdx.x == 0) bc[1] = cluster_sum(1, 0);
    __syncthreads();
    rz = bc[0];
    const double pq = bc[1];
    if (it == 0) ref = rz;
    if (!(rz > fmax(tol2 * ref, floor2)) || it >= A.max_iter) break;
    if (!(pq > 0.0) || !isfinite(pq)) {
      breakdown = 1;
      break;
    }
    alpha = rz / pq;
    // pass C: r += alpha q, rr = r^T D^-1 r, c = C D^-1 r
    double rr = 0.0;
    tasks([&] {
      if (wact)
        sweep_c_pf(
            [&](int k, bool live) {
              VC c_;
              c_.r = live ? Rv[k] : 0.0;
              c_.q = live ? Qv[k] : 0.0;
              c_.d = live ? dg[k] : 0.0;
              return c_;
            },
            [&](int, int k, const VC& c_) -> double {
              if (!lact) return 0.0;
              const double rk = c_.r + alpha * c_.q;
              Rv[k] = rk;
              const double u = c_.d * rk;
              rr += rk * u;
              return u;
            });
    });
    slot_put(2, rr);
    __syncthreads();
    reduce_c_pub(2);
    if (warp == 0) {
      const double s = slot_fin(2);
      if (lane == 0) publish(2, NQ, s);
    }
    cl.sync();  // S3: c and rr partials published; R complete over the cluster
    gather_c(2, nullptr);
    if (threadIdx.x == 0) bc[0] = cluster_sum(2, NQ);
    __syncthreads();
    if (crs) coarse_c();
    solve_y();
    __syncthreads();
    beta = (bc[0] + (crs ? slot_fin(4) : 0.0) - slot_fin(3)) / rz;
    if (crs) coarse_v(1.0);
  }

  // feasibility restoration: x += M^-1-weighted C^T S^-1 (g - C x); parents also into the pool
  tasks([&] {
    if (wact) sweep_c([&](int, int k) -> double { return lact ? Xv[k] : 0.0; });
  });
  __syncthreads();
  reduce_c_pub(0);
  cl.sync();
  gather_c(0, A.g0);
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
  if (cr == 0 && threadIdx.x == 0) {
    A.iters[prob] = it;
    A.relres[prob] = (ref > 0.0) ? sqrt(fmax(rz, 0.0) / ref) : 0.0;
    double* dgo = A.diag + (int64_t)prob * 4;
    dgo[0] = rz;
    dgo[1] = ref;
    dgo[2] = floor2;
    dgo[3] = breakdown;
  }
  cl.sync();  // no CTA leaves while a peer may still read its shared memory
}

// ------------------------------------------------------------------------------------------
// Levels >= 2 (windows of <= 25 level nodes per side): k_pcg3d (pcg3d.cu) with a cluster of CS CTAs
// per problem.  CTA c owns the node planes [c nz / CS, (c+1) nz / CS) of p_s; the stencil reads the
// two boundary planes from the neighbours' shared memory (DSMEM) after the cluster barrier that
// follows the p update; reductions as in k_pcg3d_l1c.  Config 5 level 2: the four interior windows
// need ~280 iterations (vs ~45 elsewhere) and set the level time; the cluster shortens them.
template <int N, int NXM, int RW, int MINB, int CS>
__global__ void __launch_bounds__(32 * ((NXM + (32 / ((NXM > 16) ? 32 : ((NXM > 8) ? 16 : 8))) * RW - 1) /
                                        ((32 / ((NXM > 16) ? 32 : ((NXM > 8) ? 16 : 8))) * RW)),
                                  MINB) k_pcg3dc(LevelArgs A) {
  cg::cluster_group cl = cg::this_cluster();
  const int cr = (int)cl.block_rank();
  constexpr int LPR = (NXM > 16) ? 32 : ((NXM > 8) ? 16 : 8);  // lanes per row
  constexpr int RPW = 32 / LPR;                                 // rows per warp and round
  constexpr int NW = (NXM + RPW * RW - 1) / (RPW * RW);
  constexpr int PY = NXM + 2;   // p_s rows per plane (zero halo rows y = -1, ny)
  constexpr int PZ = PY * NXM;  // p_s plane (x pitch NXM, no x halo: x-neighbours by shuffle)
  constexpr int NQ = 27 * N;    // constraint rows of a 3x3x3-subcell window
  const int prob = blockIdx.x / CS;
  const int mp = prob / A.n_rhs, rhs = prob - mp * A.n_rhs;
  const ProbDesc& P = A.probs[mp];
  const int nx = P.nc[0] + 1, ny = P.nc[1] + 1, nz = P.nc[2] + 1, nn = nx * ny * nz;
  const int ncx = nx - 1;
  const int nc = A.ncon;  // == NQ (host check)
  const int z0 = (cr * nz) / CS, z1 = ((cr + 1) * nz) / CS;  // this CTA's node planes
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int x = lane & (LPR - 1), ry = lane / LPR;
  const bool xin = x < NXM;
  // current row of this lane group: set by set_row
  int y = warp;
  bool wact = false, lact = false;  // wact warp-uniform (some row of the warp is in the window)

  extern __shared__ __align__(16) double smem[];
  constexpr int SL = (NXM + CS - 1) / CS + 2;  // p planes held per CTA: its slab + a zero halo plane each side
  double* p_s = smem;                  // [SL][PY][NXM]: plane z of the slab at z - z0 + 1, zero halo rows
  double* bins = p_s + SL * PZ;        // [NXM rows][NQ]
  double* Ysh = bins + NXM * NQ;        // [NQ] yhat
  double* csh = Ysh + NQ;               // [NQ] c
  double* slots = csh + NQ;             // [5][32] scalar partial sums
  double* zr = slots + 5 * 32;          // [256] coarse: E^-1 Z^T r
  double* vv = zr + 256;                // [256] coarse: coarse part of z
  double* red = vv + 256;               // [3][NQ + 2] cluster reduction buffers
  int* zsm = reinterpret_cast<int*>(red + 3 * (NQ + 2));  // [NXM][3] z sides (pm, k0, k1)
  __shared__ double bc[2];

  for (int i = threadIdx.x; i < SL * PZ; i += blockDim.x) p_s[i] = 0.0;
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
  auto pidx = [&](int z) { return (z - z0 + 1) * PZ + (y + 1) * NXM + x; };

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
    int layer = -1;
    for (int z = z0; z < z1; z++) {
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
    if (layer >= 0) flush(layer);
  };
  // p_s plane z (planes z0 - 1 and z1 live in the neighbouring CTA: DSMEM)
  auto plane = [&](int z) -> const double* {
    // own slab and the window's zero halo planes -1 / nz: local plane z - z0 + 1; a neighbour's
    // boundary plane: its local index from its slab start
    if (z >= 0 && z < nz && z < z0) return cl.map_shared_rank(p_s, cr - 1) + (z - ((cr - 1) * nz) / CS + 1) * PZ;
    if (z >= 0 && z < nz && z >= z1) return cl.map_shared_rank(p_s, cr + 1) + (z - z1 + 1) * PZ;
    return p_s + (z - z0 + 1) * PZ;
  };
  // (A p)_k from p_s: f(z, k, Ap, p_k)  (wact warps; lanes >= nx carry zeros)
  auto sweep_stencil = [&](auto&& f) {
    const int ro = (y + 1) * NXM + x;
    double v[3][3];  // [dy][dz]
    {
      const double* pm1 = plane(z0 - 1) + ro;
      const double* p0 = plane(z0) + ro;
#pragma unroll
      for (int dy = 0; dy < 3; dy++) {
        v[dy][0] = xin ? pm1[(dy - 1) * NXM] : 0.0;
        v[dy][1] = xin ? p0[(dy - 1) * NXM] : 0.0;
      }
    }
    for (int z = z0; z < z1; z++) {
      const double* pn = plane(z + 1) + ro;
#pragma unroll
      for (int dy = 0; dy < 3; dy++) v[dy][2] = xin ? pn[(dy - 1) * NXM] : 0.0;
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

  auto publish = [&](int b, int i, double v) { red[b * (NQ + 2) + i] = v; };
  auto cluster_sum = [&](int b, int i) -> double {
    double s = 0.0;
#pragma unroll
    for (int r = 0; r < CS; r++) s += *cl.map_shared_rank(red + b * (NQ + 2) + i, r);
    return s;
  };
  // per CTA: row bins -> red[b][0..nc) (one warp per constraint row, fixed tree)
  auto reduce_c_pub = [&](int b) {
    for (int i = warp; i < nc; i += NW) {
      double s = 0.0;
      for (int yy = lane; yy < ny; yy += 32) s += bins[yy * NQ + i];
      s = wsum0(s);
      if (lane == 0) publish(b, i, s);
    }
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
        for (int z = z0; z < z1; z++) {
          const int k = nidx(z);
          const double x0 = dg[k] * ct_at(z, k) - cz_at(k);
          p_s[pidx(z)] = x0;
          Xv[k] = x0;
        }
    });
    cl.sync();  // x0 (= p_s) complete over the cluster
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
    reduce_c_pub(2);
    if (warp == 0) {
      const double s = slot_fin(2);
      if (lane == 0) publish(2, NQ, s);
    }
    cl.sync();  // partials published; R complete over the cluster
    for (int i = threadIdx.x; i < nc; i += blockDim.x) csh[i] = cluster_sum(2, i);
    if (threadIdx.x == 0) bc[0] = cluster_sum(2, NQ);
    __syncthreads();
    if (crs) coarse_c();
    solve_y();
    __syncthreads();
    const double rrt = bc[0] + (crs ? slot_fin(4) : 0.0);
    if (crs) coarse_v(1.0);
    cl.sync();  // red[2] free again before the next publication
    return rrt;
  };

  // reference scale: initial projected residual of the full (non-hierarchical) problem
  const double rr_ref = init(A.g0, nullptr);
  double rz_ref;
  {
    double v = 0.0;
    rows([&] {
      if (lact)
        for (int z = z0; z < z1; z++) {
          const int k = nidx(z);
          const double w = Rv[k] - ct_at(z, k);
          v += dg[k] * w * w;
        }
    });
    slot_put(0, v);
    __syncthreads();
    if (warp == 0) {
      const double s = slot_fin(0);
      if (lane == 0) publish(0, 0, s);
    }
    cl.sync();
    rz_ref = cluster_sum(0, 0);
    cl.sync();
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
      for (int z = z0; z < z1; z++) {
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
    __syncthreads();
    if (warp == 0) {
      const double s = slot_fin(0);
      if (lane == 0) publish(0, 0, s);
    }
    cl.sync();  // S1: p complete over the cluster, rz partials published
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
    if (threadIdx.x == 0) bc[0] = cluster_sum(0, 0);
    __syncthreads();
    if (warp == 0) {
      const double s = slot_fin(1);
      if (lane == 0) publish(1, 0, s);
    }
    cl.sync();  // S2: pq partials published
    if (threadIdx.x == 0) bc[1] = cluster_sum(1, 0);
    __syncthreads();
    rz = bc[0];
    const double pq = bc[1];
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
    __syncthreads();
    reduce_c_pub(2);
    if (warp == 0) {
      const double s = slot_fin(2);
      if (lane == 0) publish(2, NQ, s);
    }
    cl.sync();  // S3: c and rr partials published; R complete over the cluster
    for (int i = threadIdx.x; i < nc; i += blockDim.x) csh[i] = cluster_sum(2, i);
    if (threadIdx.x == 0) bc[0] = cluster_sum(2, NQ);
    __syncthreads();
    if (crs) coarse_c();
    solve_y();
    __syncthreads();
    const double cy = slot_fin(3);
    beta = (bc[0] + (crs ? slot_fin(4) : 0.0) - cy) / rz;
    if (crs) coarse_v(1.0);
  }

  // feasibility restoration: x += D^-1 C^T S^-1 (g - C x)
  rows([&] {
    if (wact) sweep_c([&](int, int k) -> double { return lact ? Xv[k] : 0.0; });
  });
  __syncthreads();
  reduce_c_pub(0);
  cl.sync();
  for (int i = threadIdx.x; i < nc; i += blockDim.x) csh[i] = gsrc[((int64_t)mp * nc + i) * A.n_rhs + rhs] - cluster_sum(0, i);
  __syncthreads();
  solve_y();
  __syncthreads();
  if (crs) coarse_v(0.0);
  rows([&] {
    if (lact)
      for (int z = z0; z < z1; z++) {
        const int k = nidx(z);
        Xv[k] += dg[k] * ct_at(z, k) - cz_at(k);
      }
  });
  if (cr == 0 && threadIdx.x == 0) {
    A.iters[prob] = it;
    A.relres[prob] = (ref > 0.0) ? sqrt(fmax(rz, 0.0) / ref) : 0.0;
    double* dgo = A.diag + (int64_t)prob * 4;
    dgo[0] = rz;
    dgo[1] = ref;
    dgo[2] = floor2;
    dgo[3] = breakdown;
  }
  cl.sync();  // no CTA leaves while a peer may still read its shared memory
}

size_t pcg3d_l1c_smem(int N) {
  // + the coarse data CZ [27N][255] and E^-1 [255] (two-level preconditioner), 16-byte aligned
  return (size_t)(98 * 27 * N + 2 * 27 * N + 5 * 32 + 512 + 3 * (27 * N + 2)) * sizeof(double) +
         (49 * 3 + 1) * sizeof(int) + 16 + (size_t)(27 * N + 1) * 255 * sizeof(double);
}

// cluster size from the level-global problem count: enough CTAs for ~3 waves of the GPU
int pcg3d_l1c_cluster(int level_problems, int sms) {
  const char* e = getenv("MCH_L1_CLUSTER");
  if (e) return atoi(e);
  int cs = 1;
  while (cs < 8 && level_problems * cs < 2 * sms) cs *= 2;  // config 5: 216 problems -> 2
  return cs;
}

template <int N, int NW, int CS>
static cudaError_t go_l1c(const LevelArgs& A, cudaStream_t st) {
  auto k = k_pcg3d_l1c<N, NW, CS>;
  const size_t smem = pcg3d_l1c_smem(N);
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(A.nprob_mp * A.n_rhs * CS));
  cfg.blockDim = dim3(NW * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, A);
}

template <int N>
static cudaError_t go_l1c_n(const LevelArgs& A, int cs, cudaStream_t st) {
  switch (cs) {
    case 1: return go_l1c<N, MCH_L1_NW, 1>(A, st);
    case 2: return go_l1c<N, MCH_L1_NW2, 2>(A, st);
    case 4: return go_l1c<N, MCH_L1_NW, 4>(A, st);
    case 8: return go_l1c<N, MCH_L1_NW, 8>(A, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_pcg3d_l1c(const LevelArgs& A, int cs, cudaStream_t st) {
  switch (A.N) {
    case 1: return go_l1c_n<1>(A, cs, st);
    case 2: return go_l1c_n<2>(A, cs, st);
    case 3: return go_l1c_n<3>(A, cs, st);
    case 4: return go_l1c_n<4>(A, cs, st);
  }
  return cudaErrorInvalidValue;
}

// ------------------------------------------------------------------------------------------
size_t pcg3dc_smem(int N, int nxm, int cs) {
  const size_t d = (size_t)((nxm + cs - 1) / cs + 2) * (nxm + 2) * nxm + (size_t)nxm * 27 * N + 2 * 27 * N + 5 * 32 + 512 +
                   3 * (27 * N + 2);
  return d * sizeof(double) + (size_t)nxm * 3 * sizeof(int);
}

template <int N, int NXM, int RW, int MINB, int CS>
static cudaError_t go_3dc(const LevelArgs& A, cudaStream_t st) {
  auto k = k_pcg3dc<N, NXM, RW, MINB, CS>;
  const size_t smem = pcg3dc_smem(N, NXM, CS);
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  constexpr int LPR = (NXM > 16) ? 32 : ((NXM > 8) ? 16 : 8), RPW = 32 / LPR;
  constexpr int NW = (NXM + RPW * RW - 1) / (RPW * RW);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(A.nprob_mp * A.n_rhs * CS));
  cfg.blockDim = dim3(32 * NW);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, A);
}

template <int N>
static cudaError_t go_3dc_n(const LevelArgs& A, int nxm, int cs, cudaStream_t st) {
  if (nxm == 25) {
    switch (cs) {
      case 2: return go_3dc<N, 25, MCH_P25_RW, MCH_P25_MINB, 2>(A, st);
      case 4: return go_3dc<N, 25, 2, 1, 4>(A, st);
    }
  } else if (nxm == 13) {
    switch (cs) {
      case 2: return go_3dc<N, 13, 1, 2, 2>(A, st);
    }
  }
  return cudaErrorInvalidValue;
}

int pcg3dc_cluster(int nxm, int level_problems, int sms) {
  const char* e = getenv("MCH_L2_CLUSTER");
  if (e) return atoi(e);
  (void)level_problems;
  (void)sms;
  return (nxm == 25) ? 2 : 1;
}

cudaError_t launch_pcg3dc(const LevelArgs& A, int nxm, int cs, cudaStream_t st) {
  switch (A.N) {
    case 1: return go_3dc_n<1>(A, nxm, cs, st);
    case 2: return go_3dc_n<2>(A, nxm, cs, st);
    case 3: return go_3dc_n<3>(A, nxm, cs, st);
    case 4: return go_3dc_n<4>(A, nxm, cs, st);
  }
  return cudaErrorInvalidValue;
}
