// C ABI (include/mch.h) and per-level orchestration of Algorithm 1.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <memory>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/mch.h"
#include "kernels.h"
#include "mch_internal.h"
#include "plan.h"
#include "shard.h"
#include "comm.h"

namespace {

thread_local std::string g_create_error;

// Device allocations go through the caller's allocator when mch_params supplies one (e.g.
// PyTorch's caching allocator), else cudaMalloc / cudaFree.
struct DevAlloc {
  void* (*alloc)(size_t, void*, void*) = nullptr;
  void (*free)(void*, void*, void*) = nullptr;
  void* user = nullptr;
  void* stream = nullptr;
};

cudaError_t dev_alloc(const DevAlloc* a, void** p, size_t bytes) {
  if (a && a->alloc) {
    *p = a->alloc(bytes, a->stream, a->user);
    return *p ? cudaSuccess : cudaErrorMemoryAllocation;
  }
  return cudaMalloc(p, bytes);
}

void dev_free(const DevAlloc* a, void* p) {
  if (!p) return;
  if (a && a->free) a->free(p, a->stream, a->user);
  else cudaFree(p);
}

struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  const DevAlloc* al = nullptr;
  cudaError_t ensure(size_t want) {
    if (want <= bytes && ptr) return cudaSuccess;
    dev_free(al, ptr);
    ptr = nullptr;
    bytes = 0;
    size_t alloc = std::max<size_t>(want, 256);
    cudaError_t e = dev_alloc(al, &ptr, alloc);
    if (e == cudaSuccess) bytes = alloc;
    else ptr = nullptr;
    return e;
  }
  void release() {
    dev_free(al, ptr);
    ptr = nullptr;
    bytes = 0;
  }
  template <typename T> T* as() const { return reinterpret_cast<T*>(ptr); }
};

// NVTX range for the lifetime of a scope (Nsight timelines: per level, per kernel group)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

constexpr int kCoarseMax = 255;  // coarse components per window (two-level preconditioner; id 255 = none)

int64_t ipow64(int64_t b, int e) {
  int64_t r = 1;
  while (e-- > 0) r *= b;
  return r;
}

}  // namespace

// Host plan of one level, built on its first solve and reused by every later solve (mch_reset):
// macropoint batches, their device descriptors and row-chunk tables, the chosen PCG variant,
// pinned result buffers and timing events, so a solve issues only kernel launches, async copies
// into pinned memory and one stream synchronisation.
struct LevelBatch {
  int nmp = 0;
  int64_t node_off = 0, vec_off = 0, fine_off = 0;
  int max_ln = 0, max_fn = 0, th_l = 64, th_f = 64;
  int max_comb = 0;     // fine3d combine: nodes written per macropoint (whole window if stored, else K_p box)
  std::vector<int64_t> mps, ln, lc;
  std::vector<int> lexpos;  // position of each batch macropoint in the lexicographic list of this rank
  DevBuf descs, segs, nseg;
  bool on2d = false, l1op = false;
  bool on3d = false;  // on-chip 3D PCG (pcg3d.cu), levels >= 2
  bool coarse = false;  // two-level preconditioner at level 1 (generic k_pcg or k_pcg2d level-1 variant)
  bool crs2d = false;   // the on-chip 2D variant was planned with the coarse space (shared memory, TMEM)
  bool fused3 = false;  // 3D level >= 2: fused fine passes (fine3d.cu), no FI/FY workspace
  int max_kp = 0;       // K_p node-box size (FK slot) of the fused path
  int l1cs = 1;         // 3D level 1: CTAs per problem (thread-block cluster, pcg3d_cl.cu)
  int l2cs = 1;         // 3D levels >= 2 (k_pcg3d windows): CTAs per problem (pcg3d_cl.cu)
  bool w7 = false;      // 3D level >= 2, <= 7 level nodes per side: block PCG, one warp per rhs (k_pcg3d_w7)
  bool tsplit = false;  // 3D transport through k_pcg3d_l1<MODE 1> (fine windows <= 49 nodes per side)
  int nxm3 = 0;
  int variant = -1, threads2 = 0, maxseg = 0, tm_cols = 32;
  int* h_flags = nullptr;  // pinned results
  int* h_iters = nullptr;
  double* h_relres = nullptr;
  double* h_diag = nullptr;
  cudaEvent_t ev[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};  // 4, 5: around the transport
  double tr_units = 0, tr_flops = 0;  // fine window nodes x rhs of the transport, its algorithmic flops
  ~LevelBatch() {
    descs.release();
    segs.release();
    nseg.release();
    if (h_flags) cudaFreeHost(h_flags);
    if (h_iters) cudaFreeHost(h_iters);
    if (h_relres) cudaFreeHost(h_relres);
    if (h_diag) cudaFreeHost(h_diag);
    for (cudaEvent_t& e : ev)
      if (e) cudaEventDestroy(e);
  }
};

struct mch_ctx {
  mch_params p{};
  int D = 2, N = 1, n_rhs = 3, l = 1, w = 3, nsub = 9, ncon = 9;
  cudaStream_t st = nullptr;
  cudaStream_t st2 = nullptr;  // side stream: the projector's C D^-1 C^T beside the coarse-space setup
  HostPlan plan;
  ShardPlan shard;          // ownership and parent transfers (world > 1)
  ncclComm_t comm = nullptr;  // params.nccl_comm (not owned)
  const NcclApi* nccl = nullptr;
  DevBuf Gall, ball;        // all-reduced coefficients / loads (world > 1)
  double* kappa = nullptr;
  uint8_t* ids = nullptr;
  double* pool = nullptr;
  int64_t pool_len = 0;
  std::vector<int64_t> pool_off;  // per lexicographic index
  double* G = nullptr;
  int solved = 0;
  int64_t launches = 0;
  std::vector<mch_level_stats> stats;
  std::string err;
  // grow-only scratch
  DevBuf FK, STC, MLR, pinv_ds, W, Mc, g0, g, meas, cm, flags, dinv, nwt, Sinv, X, R, P, Q, B, FI, FY, iters, relres, diag;
  cudaEvent_t ev[8];
  bool events = false;
  std::vector<std::vector<std::unique_ptr<LevelBatch>>> lplans;  // per level, built on first solve
  int* h_bad = nullptr;  // mch_set_medium validation flag (pinned / device)
  bool medium_ok = true;  // false after mch_set_medium rejected its inputs: solves return MCH_EINVAL
  int* d_bad = nullptr;
  // NEXT-2: source f (cellwise, n^D), load vectors [P][N], macro-solve workspace and results
  DevBuf fsrc, bload, mws, mG, mb, mU, mres;
  DevBuf fws, fbar, ff, fu, fkbox, fout;  // NEXT-3 fine solve / block averages
  DevBuf cmap, ncomp, cbox, einv, cz, cptr, clist;  // two-level preconditioner (level 1)
  DevBuf azp, azi, azw;                               // (A z_a) lists of the 2D on-chip kernels
  bool coarse = false;
  int coarse_erode = 1;  // MCH_COARSE_ERODE=0: one labelling pass only (oversized components dropped)
  DevAlloc al;
  std::vector<DevBuf*> bufs() {
    return {&FK, &STC, &MLR, &pinv_ds, &W, &Mc, &g0, &g, &meas, &cm, &flags, &dinv, &nwt, &Sinv, &X, &R, &P, &Q, &B,
            &FI, &FY, &iters, &relres, &diag, &fsrc, &bload, &mws, &mG, &mb, &mU, &mres, &fws, &fbar, &ff, &fu,
            &fkbox, &fout, &cmap, &ncomp, &cbox, &einv, &cz, &cptr, &clist, &azp, &azi, &azw};
  }
  bool has_source = false;
  int* h_mit = nullptr;
  double* h_mrel = nullptr;
  int band = 0;      // > 0: banded projector (large oversampling, 2D), half-bandwidth
  int pcg_mode = 0;  // 0: on-chip 2D PCG where it applies; 1: generic k_pcg; 2: on-chip, precomputed operator at level 1
};

static int fail(mch_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  else g_create_error = msg;
  return code;
}

#define CKC(ctx, call)                                                                        \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      return fail(ctx, e_ == cudaErrorMemoryAllocation ? MCH_ENOMEM : MCH_ECUDA,              \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                        \
  } while (0)

// Row chunks of a 2D window for the on-chip PCG (pcg2d.cu): node rows are grouped by the subcell
// row of the elements above them, and each group is cut into near-equal chunks of <= rpt rows.
// Chunk = (first node row, rows, subcell row, subcell row of the elements below the first row if
// those belong to the previous subcell row, else -1).
static void seg_plan_2d(const ProbDesc& P, int s, int c, int coff, int l, int rpt, std::vector<short4>& out) {
  out.clear();
  const int ncy = P.nc[1];
  auto slot = [&](int ey) { return (P.lo[1] + ey * s + coff) / c - P.k[1] + l; };
  int ea = 0;
  while (ea < ncy) {
    int eb = ea + 1;
    while (eb < ncy && slot(eb) == slot(ea)) eb++;
    const int G = eb - ea + (eb == ncy ? 1 : 0);
    const int nch = (G + rpt - 1) / rpt, base = G / nch, rem = G % nch;
    int y = ea;
    for (int ch = 0; ch < nch; ch++) {
      const int n = base + (ch < rem ? 1 : 0);
      out.push_back(make_short4((short)y, (short)n, (short)slot(ea), (short)((ch == 0 && ea > 0) ? slot(ea - 1) : -1)));
      y += n;
    }
    ea = eb;
  }
}

extern "C" int mch_create(const mch_params* prm, const double* kappa, const uint8_t* ids, int on_dev,
                          mch_ctx** out) {
  if (!out) return fail(nullptr, MCH_EINVAL, "out is NULL");
  *out = nullptr;
  if (!prm || !kappa || !ids) return fail(nullptr, MCH_EINVAL, "NULL argument");
  mch_params p = *prm;
  if (p.d != 2 && p.d != 3) return fail(nullptr, MCH_EINVAL, "d must be 2 or 3");
  if (p.n <= 0 || p.M <= 0 || p.levels < 1 || p.eta < 2 || p.num_continua < 1 || p.num_continua > 4)
    return fail(nullptr, MCH_EINVAL, "bad n / M / levels / eta / num_continua");
  if (p.oversample < 1) p.oversample = 1;
  if (p.rtol <= 0) p.rtol = 1e-12;
  if (p.max_iter <= 0) p.max_iter = 20000;
  if (p.world < 1) { p.world = 1; p.rank = 0; }
  if (p.rank < 0 || p.rank >= p.world) return fail(nullptr, MCH_EINVAL, "bad rank/world");
  const int w = 2 * p.oversample + 1;
  const int nsub = (p.d == 2) ? w * w : w * w * w;
  // more than 108 constraint rows (or MCH_FORCE_BAND): 2D only, banded projector (k_proj_setup_band)
  const int nrows = nsub * p.num_continua;
  const bool want_band = nrows > 108 || (p.d == 2 && getenv("MCH_FORCE_BAND") != nullptr);
  int band = 0;
  if (want_band) {
    if (p.d != 2) return fail(nullptr, MCH_EINVAL, "too many constraint rows (>108) for a 3D window");
    band = (w + 2) * p.num_continua - 1;
    const size_t need = sizeof(double) * ((size_t)nrows * (band + 1) + 6 * (size_t)nrows + 32 * 16 + 16) +
                        sizeof(int) * (nsub * 7 + 2);
    if (need > 232448) return fail(nullptr, MCH_EINVAL, "too many constraint rows for the banded projector");
  }
  if (p.n > (1 << 20)) return fail(nullptr, MCH_EINVAL, "n too large");

  mch_ctx* c = new mch_ctx();
  c->p = p;
  c->band = band;
  if ((p.alloc == nullptr) != (p.free == nullptr)) {
    delete c;
    return fail(nullptr, MCH_EINVAL, "alloc and free must both be given or both be NULL");
  }
  c->al.alloc = p.alloc;
  c->al.free = p.free;
  c->al.user = p.alloc_user;
  c->al.stream = p.stream;
  for (DevBuf* b : c->bufs()) b->al = &c->al;
  c->Gall.al = c->ball.al = &c->al;
  c->D = p.d;
  c->N = p.num_continua;
  c->n_rhs = p.num_continua * (1 + p.d);
  c->l = p.oversample;
  c->w = w;
  c->nsub = nsub;
  c->ncon = nsub * p.num_continua;
  c->st = reinterpret_cast<cudaStream_t>(p.stream);
  // two-level preconditioner at level 1: on unless MCH_COARSE=0
  c->coarse = !(getenv("MCH_COARSE") != nullptr && atoi(getenv("MCH_COARSE")) == 0);
  c->coarse_erode = getenv("MCH_COARSE_ERODE") != nullptr ? atoi(getenv("MCH_COARSE_ERODE")) : 1;
  if (const char* pm = getenv("MCH_PCG")) {
    if (!strcmp(pm, "old")) c->pcg_mode = 1;
    else if (!strcmp(pm, "gn")) c->pcg_mode = 2;
  }
  c->plan.D = p.d;
  c->plan.n = p.n;
  c->plan.M = p.M;
  c->plan.L = p.levels;
  c->plan.eta = p.eta;
  c->plan.l = p.oversample;
  if (p.interp < 0 || p.interp > 2) {
    delete c;
    return fail(nullptr, MCH_EINVAL, "interp must be MCH_INTERP_DLINEAR, MCH_INTERP_NEAREST_S1 or MCH_INTERP_PHYSICAL_S1");
  }
  if (p.interp == 2) {
    // NEXT-4: level-1 windows of l + eta^(L-1)/2 layers; built for 2D vertex windows whose level-1
    // constraint rows fit the dense projector of the generic PCG
    int64_t e = 1;
    for (int i = 1; i < p.levels; i++) e *= p.eta;
    const int l1 = p.oversample + (int)(e / 2), w1 = 2 * l1 + 1;
    if (p.d != 2 || p.layout != 0 || w1 * w1 * p.num_continua > 108 || c->band != 0) {
      delete c;
      return fail(nullptr, MCH_EINVAL,
                  "MCH_INTERP_PHYSICAL_S1 needs d = 2, the vertex layout and <= 108 level-1 constraint rows");
    }
  }
  c->plan.interp = p.interp;
  if (p.layout != 0 && p.layout != 1) {
    delete c;
    return fail(nullptr, MCH_EINVAL, "layout must be MCH_LAYOUT_VERTEX or MCH_LAYOUT_BLOCK");
  }
  c->plan.layout = p.layout;
  std::string perr;
  int rc = c->plan.build(perr);
  if (rc != 0) {
    delete c;
    return fail(nullptr, rc == -8 ? MCH_EPLAN : MCH_EDIVISIBILITY, perr);
  }
  const int64_t cells = (p.d == 2) ? p.n * p.n : p.n * p.n * p.n;
  // host-side validation when inputs are on the host
  if (!on_dev) {
    for (int64_t i = 0; i < cells; i++) {
      if (!(kappa[i] > 0.0) || !std::isfinite(kappa[i])) {
        delete c;
        return fail(nullptr, MCH_EINVAL, "kappa must be positive and finite");
      }
      if (ids[i] >= p.num_continua) {
        delete c;
        return fail(nullptr, MCH_EINVAL, "continuum id >= num_continua");
      }
    }
  }
  auto cleanup = [&](int code, const std::string& m) {
    mch_destroy(c);
    return fail(nullptr, code, m);
  };
  cudaError_t e;
  if ((e = dev_alloc(&c->al, (void**)&c->kappa, cells * sizeof(double))) != cudaSuccess) return cleanup(MCH_ENOMEM, "kappa alloc");
  if ((e = dev_alloc(&c->al, (void**)&c->ids, cells)) != cudaSuccess) return cleanup(MCH_ENOMEM, "ids alloc");
  const cudaMemcpyKind kind = on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  if ((e = cudaMemcpyAsync(c->kappa, kappa, cells * sizeof(double), kind, c->st)) != cudaSuccess)
    return cleanup(MCH_ECUDA, std::string("kappa copy: ") + cudaGetErrorString(e));
  if ((e = cudaMemcpyAsync(c->ids, ids, cells, kind, c->st)) != cudaSuccess)
    return cleanup(MCH_ECUDA, std::string("ids copy: ") + cudaGetErrorString(e));
  if (on_dev) {
    int* bad = nullptr;
    if (dev_alloc(&c->al, (void**)&bad, sizeof(int)) != cudaSuccess) return cleanup(MCH_ENOMEM, "alloc");
    cudaMemsetAsync(bad, 0, sizeof(int), c->st);
    launch_validate(c->kappa, c->ids, cells, p.num_continua, bad, c->st);
    int hb = 0;
    cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, c->st);
    e = cudaStreamSynchronize(c->st);
    dev_free(&c->al, bad);
    if (e != cudaSuccess) return cleanup(MCH_ECUDA, cudaGetErrorString(e));
    if (hb) return cleanup(MCH_EINVAL, "kappa must be positive and finite; ids < num_continua");
  }
  // sharding: contiguous cost-balanced runs of each S_n per rank, parent transfers
  shard_build(c->plan, p.world, c->shard);
  if (p.nccl_comm) {  // also with world == 1 (a one-rank communicator: the collectives are copies)
    std::string nerr;
    c->nccl = nccl_api(nerr);
    if (!c->nccl) return cleanup(MCH_ENCCL, nerr);
    c->comm = reinterpret_cast<ncclComm_t>(p.nccl_comm);
  }
  // parent pool: T_{L-1} (or everything with keep_all)
  const int64_t nmac = (int64_t)c->plan.all.size();
  c->pool_off.assign(nmac, -1);
  // layout: by level, then owner rank, then lexicographic, so the slots one rank produces at one
  // level are contiguous.  Every rank holds the whole pool layout.
  int64_t off = 0;
  for (int lev = 1; lev <= p.levels; lev++) {
    if (!(lev < p.levels || p.keep_all)) continue;
    const std::vector<int64_t>& Sl = c->plan.S[lev];
    for (int owner = 0; owner < p.world; owner++) {
      for (size_t pos = 0; pos < Sl.size(); pos++) {
        if (c->shard.owner[lev][pos] != owner) continue;
        const MacroHost& m = c->plan.all[Sl[pos]];
        int64_t fn = 1;
        for (int d = 0; d < p.d; d++) fn *= (m.hi[d] - m.lo[d] + 1);
        c->pool_off[Sl[pos]] = off;
        off += fn * c->n_rhs;
      }
    }
  }
  c->pool_len = off;
  if (off > 0 && dev_alloc(&c->al, (void**)&c->pool, off * sizeof(double)) != cudaSuccess) return cleanup(MCH_ENOMEM, "pool alloc");
  // world > 1: poison the pool (NaN) so a parent that should have been received but was not shows
  // up as a non-finite coefficient instead of a silently wrong one
  if (off > 0 && p.world > 1) cudaMemsetAsync(c->pool, 0xFF, off * sizeof(double), c->st);
  const size_t gbytes = (size_t)nmac * c->n_rhs * c->n_rhs * sizeof(double);
  if (dev_alloc(&c->al, (void**)&c->G, gbytes) != cudaSuccess) return cleanup(MCH_ENOMEM, "G alloc");
  cudaMemsetAsync(c->G, 0, gbytes, c->st);
  c->stats.assign(p.levels + 1, mch_level_stats{});
  for (int i = 0; i < 8; i++) cudaEventCreate(&c->ev[i]);
  c->events = true;
  if ((e = cudaStreamCreateWithFlags(&c->st2, cudaStreamNonBlocking)) != cudaSuccess)
    return cleanup(MCH_ECUDA, cudaGetErrorString(e));
  if ((e = cudaStreamSynchronize(c->st)) != cudaSuccess) return cleanup(MCH_ECUDA, cudaGetErrorString(e));
  *out = c;
  return MCH_OK;
}

// Geometry of one macropoint's problem at its level (offsets and parents are filled per batch).
static void fill_geometry(const HostPlan& pl, int D, int s, const MacroHost& m, ProbDesc& P) {
  memset(&P, 0, sizeof(P));
  for (int d = 0; d < 3; d++) {
    P.k[d] = m.k[d];
    P.lo[d] = (d < D) ? m.lo[d] : 0;
    P.ncf[d] = (d < D) ? m.hi[d] - m.lo[d] : 0;
    P.nc[d] = (d < D) ? P.ncf[d] / s : 0;
    P.glo[d] = (d < D) ? P.lo[d] / s : 0;
    const int64_t a = (int64_t)m.k[d] * pl.c - pl.coff(), b = a + pl.c;  // K_p
    P.kp_lo[d] = (d < D) ? (int)std::max<int64_t>(0, a) : 0;
    P.kp_hi[d] = (d < D) ? (int)std::min<int64_t>(pl.n, b) : 1;
  }
  P.lin = m.lin;
}

// Kernel variants of one level, decided over ALL macropoints of S_level (every rank decides the
// same), so a macropoint takes the same kernels and arithmetic whatever the sharding: results are
// bitwise independent of world.
struct LevelVariant {
  bool on2d = false, l1op = false, crs2d = false;
  int variant = -1, threads2 = 0, tm_cols = 32, rpt = 0;
  bool on3d = false, w7 = false, tsplit = false, fused3 = false;
  int nxm3 = 0, l1cs = 1, l2cs = 1;
  int th_l = 64, th_f = 64;
  int max_kp = 0;
  bool coarse = false;
};

// oversampling layers, subcells per dimension, subcells and constraint rows of a level's windows
// (level 1 of the physical-coordinate variant has more, NEXT-4)
static void level_geometry(const mch_ctx* c, int level, int& l, int& w, int& nsub, int& nc) {
  l = c->plan.lwin(level);
  w = 2 * l + 1;
  nsub = (c->D == 2) ? w * w : w * w * w;
  nc = nsub * c->N;
}

static int build_level(mch_ctx* c, int level, std::vector<std::unique_ptr<LevelBatch>>& out) {
  const int D = c->D, N = c->N, nr = c->n_rhs;
  int lvl_l, lvl_w, lvl_nsub, nc;
  level_geometry(c, level, lvl_l, lvl_w, lvl_nsub, nc);
  const HostPlan& pl = c->plan;
  const int s = (int)ipow64(c->p.eta, level - 1);
  const std::vector<int64_t>& Sl = pl.S[level];
  std::vector<int64_t> mine;
  for (size_t i = 0; i < Sl.size(); i++)
    if (c->shard.owner[level][i] == c->p.rank) mine.push_back(Sl[i]);
  auto sizes = [&](const MacroHost& m, int64_t& ln, int64_t& fnn, int64_t& lcells) {
    ln = 1; fnn = 1; lcells = 1;
    for (int d = 0; d < D; d++) {
      const int ncf = m.hi[d] - m.lo[d];
      ln *= (ncf / s + 1);
      fnn *= (ncf + 1);
      lcells *= ncf / s;
    }
  };
  // ---- level-global decisions
  LevelVariant V;
  std::vector<ProbDesc> gd(Sl.size());
  int gmaxn = 0, gmaxf = 0;
  int64_t gmax_ln = 0, gmax_fn = 0;
  for (size_t i = 0; i < Sl.size(); i++) {
    const MacroHost& m = pl.all[Sl[i]];
    fill_geometry(pl, D, s, m, gd[i]);
    int64_t ln, fnn, lc;
    sizes(m, ln, fnn, lc);
    gmax_ln = std::max(gmax_ln, ln);
    gmax_fn = std::max(gmax_fn, fnn);
    int kp = 1;
    for (int d = 0; d < D; d++) {
      gmaxn = std::max(gmaxn, gd[i].nc[d] + 1);
      gmaxf = std::max(gmaxf, gd[i].ncf[d] + 1);
      kp *= gd[i].kp_hi[d] - gd[i].kp_lo[d] + 1;
    }
    V.max_kp = std::max(V.max_kp, kp);
  }
  auto pick = [](int64_t nodes) {
    int64_t t = ((nodes / 4 + 31) / 32) * 32;
    return (int)std::max<int64_t>(64, std::min<int64_t>(512, t));
  };
  V.th_l = pick(gmax_ln);
  V.th_f = pick(gmax_fn);
  // on-chip 2D PCG (pcg2d.cu) unless MCH_PCG=old; MCH_PCG=gn forces the precomputed-operator
  // variant at level 1 as well (cross-check of the two operator paths)
  if ((D == 2) && N <= 3 && nc == 9 * N && c->pcg_mode != 1 && c->band == 0) {  // 3x3 subcells (l = 1)
    std::vector<int> cands;
    if (level == 1 && c->pcg_mode != 2) cands.push_back(PCG2D_V_L1);
    cands.push_back(PCG2D_V_GN25);
    cands.push_back(PCG2D_V_GN49);
    cands.push_back(PCG2D_V_GN97);
    std::vector<short4> tmp;
    for (int v : cands) {
      int rpt, nxm, maxw, l1op, sstc, smlr;
      pcg2d_variant(v, &rpt, &nxm, &maxw, &l1op, &sstc, &smlr);
      // the coarse-space variant where it is used and fits, else the same variant without it
      bool crs_v = c->coarse && ((level == 1 && v == PCG2D_V_L1) || (level == 2 && v == PCG2D_V_GN49));
      if (crs_v && pcg2d_smem_t(N, l1op != 0, nxm, maxw, sstc != 0, smlr != 0, true) > 232448) crs_v = false;
      if (gmaxn > nxm || pcg2d_smem_t(N, l1op != 0, nxm, maxw, sstc != 0, smlr != 0, crs_v) > 232448) continue;
      int maxwp = 0;
      for (size_t i = 0; i < gd.size(); i++) {
        seg_plan_2d(gd[i], s, (int)pl.c, (int)pl.coff(), lvl_l, rpt, tmp);
        maxwp = std::max(maxwp, ((gd[i].nc[0] + 1 + 31) / 32) * (int)tmp.size());
      }
      const int rp4 = (rpt + 3) & ~3;  // TMEM: warps per lane quarter x (q, x [, component ids])
      const int need = ((maxwp + 3) / 4) * (4 * rp4 + (crs_v ? rp4 / 4 : 0));
      int cols = 32;
      while (cols < need) cols *= 2;
      if (maxwp > maxw || cols > 512) continue;
      V.tm_cols = cols;
      V.threads2 = 32 * maxwp;
      V.variant = v;
      V.rpt = rpt;
      V.l1op = l1op != 0;
      V.on2d = true;
      V.crs2d = crs_v;
      break;
    }
  }
  // 3D: on-chip PCG at levels >= 2 (pcg3d.cu) for windows of <= 25 level nodes per side, at level
  // 1 (k_pcg3d_l1) for windows of <= 49 fine nodes per side; fused fine passes (fine3d.cu) at
  // levels >= 2 for 3x3x3 subcells, windows of <= 49 fine nodes per side and >= 4 fine cells per H
  // (a thread's 7-row strip spans <= 3 subcell rows)
  if (D == 3 && nc == 27 * N && N <= 4 && c->pcg_mode != 1) {
    const char* f3e = getenv("MCH_FINE3D");
    const bool generic_t = getenv("MCH_TRANSPORT_GENERIC") != nullptr;
    V.tsplit = level >= 2 && gmaxf <= 49 && pcg3d_l1_smem(N) <= 232448 && !generic_t;
    V.fused3 = level >= 2 && lvl_l == 1 && pl.c >= 4 && gmaxf <= 49 && fine3d_transport_smem(N) <= 232448 &&
               !(f3e && atoi(f3e) == 0) && !generic_t;
    if (level >= 2) {
      const int nxm = pcg3d_nxm(gmaxn);
      if (nxm > 0 && pcg3d_smem(N, nxm) <= 232448) {
        V.on3d = true;
        V.nxm3 = nxm;
      }
      if (V.on3d && (nxm == 25 || nxm == 13)) {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        V.l2cs = pcg3dc_cluster(nxm, (int)Sl.size() * nr, sms);
        if (pcg3dc_smem(N, nxm, V.l2cs) > 232448) V.l2cs = 1;
      }
      const char* w7e = getenv("MCH_PCG3D_W7");
      V.w7 = V.on3d && nxm == 7 && N <= 2 && nr == 4 * N && pcg3d_w7_smem(N) <= 232448 && !(w7e && atoi(w7e) == 0);
    } else if (gmaxn <= 49 && pcg3d_l1_smem(N) <= 232448) {
      V.on3d = true;
      V.nxm3 = 49;
      int dev = 0, sms = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      V.l1cs = pcg3d_l1c_cluster((int)Sl.size() * nr, sms);  // level-global count: same on every rank
      if (pcg3d_l1c_smem(N) > 232448 || (getenv("MCH_L1_OLD") && atoi(getenv("MCH_L1_OLD")))) V.l1cs = 0;  // 0: k_pcg3d_l1
    }
  }
  // two-level preconditioner: level 1 everywhere; level 2 on the 49-node on-chip 2D variant,
  // whose shared memory holds the coarse data; 3D level 1 and the 25-node level-2 windows (the 13-
  // and 7-node windows of deeper levels showed no iteration change)
  V.coarse = c->coarse && c->band == 0 && (V.on2d ? V.crs2d : (level == 1 || (V.on3d && V.nxm3 == 25)));
  // the projector setup stages S, its copy and (C Z) in shared memory: without the coarse space
  // where that does not fit (the 98-row level-1 windows of the physical-coordinate variant)
  if (V.coarse && sizeof(double) * (2.0 * nc * nc + 32 * 16 + 16 + (lvl_nsub * 7 + 2 + 1) / 2 + 2 +
                                    (double)(nc + 1) * kCoarseMax) > 232448)
    V.coarse = false;
  const double kpn = (double)V.max_kp;

  // ---- this rank's macropoints, batched by memory
  // solve order: largest (unclipped) windows first.  Their problems are the longest (more work per
  // iteration and more iterations), so starting them first shortens the tail of the launch
  // (longest-processing-time-first list scheduling over the SMs).  Stable: lexicographic within
  // a window size.  mch_level_iterations reports in the lexicographic order.
  std::vector<int64_t> lexi = mine;
  {
    std::vector<int64_t> key(pl.all.size(), 0);
    for (int64_t m : mine) {
      int64_t ln, fnn, lc;
      sizes(pl.all[m], ln, fnn, lc);
      key[m] = ln;
    }
    std::stable_sort(mine.begin(), mine.end(), [&](int64_t a, int64_t b) { return key[a] > key[b]; });
  }
  size_t freeb = 0, totb = 0;
  cudaMemGetInfo(&freeb, &totb);
  const double budget = std::min<double>(48e9, 0.5 * (double)freeb);
  size_t bstart = 0;
  while (bstart < mine.size()) {
    size_t bend = bstart;
    double bytes = 0;
    while (bend < mine.size()) {
      int64_t ln, fnn, lc;
      sizes(pl.all[mine[bend]], ln, fnn, lc);
      double b = 8.0 * (5.0 * nr * ln + ln * (10.0 + 4.0 * N) + (double)nc * nc + 3.0 * nc * nr + nc + 12) +
                 (level >= 2 ? (V.fused3 ? 8.0 * nr * kpn : 16.0 * nr * fnn) : 0.0);
      if (bend > bstart && bytes + b > budget) break;
      bytes += b;
      bend++;
    }
    std::unique_ptr<LevelBatch> B(new LevelBatch());
    B->descs.al = B->segs.al = B->nseg.al = &c->al;
    const int nmp = (int)(bend - bstart);
    B->nmp = nmp;
    std::vector<ProbDesc> descs(nmp);
    for (int i = 0; i < nmp; i++) {
      const MacroHost& m = pl.all[mine[bstart + i]];
      ProbDesc& P = descs[i];
      fill_geometry(pl, D, s, m, P);
      int64_t ln, fnn, lc;
      sizes(m, ln, fnn, lc);
      B->mps.push_back(mine[bstart + i]);
      B->lexpos.push_back((int)(std::lower_bound(lexi.begin(), lexi.end(), mine[bstart + i]) - lexi.begin()));
      B->ln.push_back(ln);
      B->lc.push_back(lc);
      P.node_off = B->node_off;
      P.vec_off = B->vec_off;
      P.fine_off = B->fine_off;
      P.pool_off = c->pool_off[m.lin];
      B->node_off += ln;
      B->vec_off += ln * nr;
      if (level >= 2) B->fine_off += fnn * nr;
      B->max_ln = std::max<int>(B->max_ln, (int)ln);
      B->max_fn = std::max<int>(B->max_fn, (int)fnn);
      B->max_comb = std::max<int>(B->max_comb, P.pool_off >= 0 ? (int)fnn : V.max_kp);
      if (level >= 2) {  // transport work: per fine node and rhs 2 npar (I_p) + 60
        B->tr_units += (double)fnn * nr;
        B->tr_flops += (double)fnn * nr * (2.0 * m.npar + 60.0);
      }
      P.npar = m.npar;
      for (int t = 0; t < m.npar; t++) {
        const MacroHost& pm = pl.all[m.par_lin[t]];
        for (int d = 0; d < 3; d++) {
          P.par_k[t][d] = pm.k[d];
          P.par_lo[t][d] = (d < D) ? pm.lo[d] : 0;
          P.par_ncf[t][d] = (d < D) ? pm.hi[d] - pm.lo[d] : 0;
        }
        P.par_pool[t] = c->pool_off[pm.lin];
        P.par_w[t] = m.par_w[t];
        if (P.par_pool[t] < 0) return fail(c, MCH_EPLAN, "parent not in pool");
      }
    }
    B->th_l = V.th_l;
    B->th_f = V.th_f;
    CKC(c, B->descs.ensure(sizeof(ProbDesc) * nmp));
    CKC(c, cudaMemcpy(B->descs.ptr, descs.data(), sizeof(ProbDesc) * nmp, cudaMemcpyHostToDevice));
    if (V.on2d) {
      std::vector<int> nsegs(nmp);
      std::vector<std::vector<short4>> per(nmp);
      int maxseg = 0;
      for (int i = 0; i < nmp; i++) {
        seg_plan_2d(descs[i], s, (int)pl.c, (int)pl.coff(), lvl_l, V.rpt, per[i]);
        nsegs[i] = (int)per[i].size();
        maxseg = std::max(maxseg, nsegs[i]);
      }
      std::vector<short4> all_segs((size_t)nmp * maxseg, make_short4(0, 0, 0, -1));
      for (int i = 0; i < nmp; i++)
        for (int k = 0; k < nsegs[i]; k++) all_segs[(size_t)i * maxseg + k] = per[i][k];
      CKC(c, B->segs.ensure(sizeof(short4) * all_segs.size()));
      CKC(c, B->nseg.ensure(sizeof(int) * nmp));
      CKC(c, cudaMemcpy(B->segs.ptr, all_segs.data(), sizeof(short4) * all_segs.size(), cudaMemcpyHostToDevice));
      CKC(c, cudaMemcpy(B->nseg.ptr, nsegs.data(), sizeof(int) * nmp, cudaMemcpyHostToDevice));
      B->maxseg = maxseg;
      B->tm_cols = V.tm_cols;
      B->threads2 = V.threads2;
      B->variant = V.variant;
      B->l1op = V.l1op;
      B->on2d = true;
      B->crs2d = V.crs2d;
    }
    B->on3d = V.on3d;
    B->nxm3 = V.nxm3;
    B->l1cs = V.l1cs;
    B->l2cs = V.l2cs;
    B->w7 = V.w7;
    B->tsplit = V.tsplit;
    B->fused3 = V.fused3;
    B->max_kp = V.max_kp;
    B->coarse = V.coarse;
    // scratch shared by all levels and batches (grow-only, allocated here, never in a solve)
    CKC(c, c->g0.ensure(sizeof(double) * nmp * nc * nr));
    CKC(c, c->g.ensure(sizeof(double) * nmp * nc * nr));
    CKC(c, c->meas.ensure(sizeof(double) * nmp * nc));
    CKC(c, c->cm.ensure(sizeof(double) * nmp * 12));
    CKC(c, c->flags.ensure(sizeof(int) * nmp));
    CKC(c, c->dinv.ensure(sizeof(double) * B->node_off));
    CKC(c, c->nwt.ensure(sizeof(double) * B->node_off * N));
    CKC(c, c->Sinv.ensure(sizeof(double) * nmp * nc * nc));
    CKC(c, c->pinv_ds.ensure(sizeof(double) * nmp * nc));
    CKC(c, c->X.ensure(sizeof(double) * B->vec_off));
    CKC(c, c->iters.ensure(sizeof(int) * nmp * nr));
    CKC(c, c->relres.ensure(sizeof(double) * nmp * nr));
    CKC(c, c->diag.ensure(sizeof(double) * nmp * nr * 4));
    if (!B->on2d) {  // the generic k_pcg keeps r, p, q in global memory
      CKC(c, c->R.ensure(sizeof(double) * B->vec_off));
      CKC(c, c->P.ensure(sizeof(double) * B->vec_off));
      CKC(c, c->Q.ensure(sizeof(double) * B->vec_off));
    }
    if (level >= 2) {
      CKC(c, c->B.ensure(sizeof(double) * B->vec_off));
      if (B->fused3) {
        CKC(c, c->FK.ensure(sizeof(double) * (size_t)nmp * nr * B->max_kp));
      } else {
        CKC(c, c->FI.ensure(sizeof(double) * B->fine_off));
        CKC(c, c->FY.ensure(sizeof(double) * B->fine_off));
      }
    }
    if (B->on2d && !B->l1op) {
      CKC(c, c->STC.ensure(sizeof(double) * 9 * B->node_off));
      CKC(c, c->MLR.ensure(sizeof(double) * 4 * N * B->node_off));
    }
    if (B->coarse) {
      if (B->on2d && B->variant == PCG2D_V_L1) CKC(c, c->R.ensure(sizeof(double) * B->vec_off));  // r mirror (L2)
      CKC(c, c->cmap.ensure(sizeof(int) * B->node_off));
      CKC(c, c->ncomp.ensure(sizeof(int) * nmp));
      CKC(c, c->cbox.ensure(sizeof(int) * 6 * kCoarseMax * (size_t)nmp));
      CKC(c, c->einv.ensure(sizeof(double) * kCoarseMax * (size_t)nmp));
      CKC(c, c->cz.ensure(sizeof(double) * kCoarseMax * (size_t)nmp * nc));
      CKC(c, c->cptr.ensure(sizeof(int) * (kCoarseMax + 1) * (size_t)nmp));
      CKC(c, c->clist.ensure(sizeof(int) * B->node_off));
      if (B->on2d && B->variant == PCG2D_V_L1) {
        CKC(c, c->azp.ensure(sizeof(int) * (kCoarseMax + 1) * (size_t)nmp));
        CKC(c, c->azi.ensure(sizeof(int) * kAzCap * B->node_off));
        CKC(c, c->azw.ensure(sizeof(double) * kAzCap * B->node_off));
      }
    }
    if (B->on3d && level >= 2) {
      const int64_t pad = B->w7 ? 0 : (int64_t)B->nxm3 * B->nxm3 * B->nxm3;
      const int64_t nodes = std::max<int64_t>(B->node_off, pad * nmp);
      CKC(c, c->STC.ensure(sizeof(double) * 27 * nodes));
      CKC(c, c->MLR.ensure(sizeof(double) * 8 * N * nodes));
    }
    CKC(c, cudaMallocHost(&B->h_flags, sizeof(int) * nmp));
    CKC(c, cudaMallocHost(&B->h_iters, sizeof(int) * nmp * nr));
    CKC(c, cudaMallocHost(&B->h_relres, sizeof(double) * nmp * nr));
    CKC(c, cudaMallocHost(&B->h_diag, sizeof(double) * nmp * nr * 4));
    for (cudaEvent_t& e : B->ev) CKC(c, cudaEventCreate(&e));
    out.push_back(std::move(B));
    bstart = bend;
  }
  return MCH_OK;
}

extern "C" int mch_solve_level(mch_ctx* c, int level) {
  if (!c) return MCH_EINVAL;
  if (!c->medium_ok) return fail(c, MCH_EINVAL, "the last mch_set_medium was rejected: set a valid medium first");
  if (level != c->solved + 1 || level > c->p.levels)
    return fail(c, MCH_EORDER, "levels must be solved 1..L in order");
  char nv_name[40];
  snprintf(nv_name, sizeof nv_name, "mch_solve_level %d", level);
  NvtxRange nv_level(nv_name);
  const int D = c->D, N = c->N, nr = c->n_rhs;
  int lvl_l, lvl_w, lvl_nsub, nc;
  level_geometry(c, level, lvl_l, lvl_w, lvl_nsub, nc);
  const HostPlan& pl = c->plan;
  const int s = (int)ipow64(c->p.eta, level - 1);
  const int gn = (int)(pl.n / s);
  cudaStream_t st = c->st;
  if ((int)c->lplans.size() <= level) c->lplans.resize(level + 1);
  std::vector<std::unique_ptr<LevelBatch>>& batches = c->lplans[level];
  if (batches.empty()) {
    const int rc = build_level(c, level, batches);
    if (rc != MCH_OK) {
      batches.clear();
      return rc;
    }
  }
  mch_level_stats& S = c->stats[level];
  S = mch_level_stats{};
  cudaEventRecord(c->ev[0], st);

  LevelArgs A{};
  A.D = D; A.N = N; A.n_rhs = nr; A.l = lvl_l; A.w = lvl_w; A.nsub = lvl_nsub; A.ncon = nc;
  A.phys = (c->p.interp == 2) ? 1 : 0;  // NEXT-4: parents evaluated at physical coordinates
  A.level = level; A.s = s; A.n = (int)pl.n; A.c = (int)pl.c; A.coff = (int)pl.coff(); A.gn = gn; A.h = 1.0 / (double)pl.n; A.inv_c = 1.0f / (float)pl.c;
  A.kappa = c->kappa; A.ids = c->ids; A.pool = c->pool; A.G = c->G;
  A.f = c->has_source ? c->fsrc.as<double>() : nullptr;
  A.band = c->band;
  A.bload = c->bload.as<double>();
  A.rtol = c->p.rtol; A.max_iter = c->p.max_iter;
  A.nprob_level = (int)pl.S[level].size();  // kernel heuristics use the level-global count (world-independent)
  if (level >= 2) {
    const int64_t gcells = (D == 2) ? (int64_t)gn * gn : (int64_t)gn * gn * gn;
    const int NW = (D == 2) ? 6 : 27;
    CKC(c, c->W.ensure(gcells * NW * sizeof(double)));
    CKC(c, c->Mc.ensure(gcells * (N << D) * sizeof(double)));
    A.W = c->W.as<double>();
    A.Mc = c->Mc.as<double>();
    CKC(c, launch_level_ops(A, st));
    S.launches += 1;
  }
  A.g0 = c->g0.as<double>(); A.g = c->g.as<double>(); A.meas = c->meas.as<double>();
  A.cm = c->cm.as<double>(); A.flags = c->flags.as<int>();
  A.dinv = c->dinv.as<double>(); A.NWt = c->nwt.as<double>(); A.Sinv = c->Sinv.as<double>();
  A.pinv_ds = c->pinv_ds.as<double>();
  A.X = c->X.as<double>(); A.R = c->R.as<double>(); A.P = c->P.as<double>(); A.Q = c->Q.as<double>();
  A.B = c->B.as<double>();
  A.FI = c->FI.as<double>(); A.FY = c->FY.as<double>();
  A.iters = c->iters.as<int>(); A.relres = c->relres.as<double>(); A.diag = c->diag.as<double>();
  A.STC = c->STC.as<double>(); A.MLR = c->MLR.as<double>();
  const bool multi = batches.size() > 1;
  for (size_t bi = 0; bi < batches.size(); bi++) {
    LevelBatch& B = *batches[bi];
    const int nmp = B.nmp;
    A.probs = B.descs.as<ProbDesc>();
    A.nprob_mp = nmp;
    A.segs = B.segs.as<short4>();
    A.nseg = B.nseg.as<int>();
    A.maxseg = B.maxseg;
    A.tm_cols = B.tm_cols;
    CKC(c, cudaMemsetAsync(c->flags.ptr, 0, sizeof(int) * nmp, st));
    cudaEventRecord(B.ev[0], st);
    S.launches += (level >= 2) ? 6 : 4;
    nvtxRangePushA("targets + transport + projector");
    CKC(c, launch_targets(A, st));
    A.FK = B.fused3 ? c->FK.as<double>() : nullptr;
    A.nkp_max = B.max_kp;
    A.stc_pad = (B.on3d && level >= 2 && !B.w7) ? B.nxm3 * B.nxm3 * B.nxm3 : 0;
    A.need_nwt = (B.on2d || B.on3d) ? 0 : 1;  // see the PCG dispatch below
    cudaEventRecord(B.ev[4], st);
    if (level >= 2 && B.fused3) {  // 3D: I_p, A_1 I_p, C_1 I_p and P_n^T in one pass (fine3d.cu)
      CKC(c, launch_fine3d_transport(A, st));
    } else if (level >= 2 && B.tsplit) {  // 3D: I_p, then the column-walking apply, then P_n^T
      A.tphase = 1;
      CKC(c, launch_transport(A, B.th_f, st));
      CKC(c, launch_tapply3d(A, st));
      A.tphase = 2;
      CKC(c, launch_transport(A, B.th_f, st));
      A.tphase = 0;
      S.launches += 2;
    } else if (level >= 2) {
      CKC(c, launch_transport(A, B.th_f, st));
    }
    cudaEventRecord(B.ev[5], st);
    // bit 1: second labelling pass that splits oversized components (k_coarse_setup)
    A.coarse = B.coarse ? (c->coarse_erode ? 3 : 1) : 0;
    A.ncmax = kCoarseMax;
    A.cmap = c->cmap.as<int>(); A.ncomp = c->ncomp.as<int>(); A.cbox = c->cbox.as<int>();
    A.Einv = c->einv.as<double>(); A.CZ = c->cz.as<double>();
    A.cptr = c->cptr.as<int>(); A.clist = c->clist.as<int>();
    A.azp = (B.coarse && B.on2d && B.variant == PCG2D_V_L1) ? c->azp.as<int>() : nullptr;
    A.azi = c->azi.as<int>(); A.azw = c->azw.as<double>();
    // with the coarse space, the projector's S = C D^-1 C^T (independent of it) is formed on the
    // side stream beside k_coarse_setup (81 / 208 CTAs each at config 2), then completed with
    // (CZ) E^-1 (CZ)^T and inverted
    const bool psplit = A.coarse && c->band == 0 && c->st2 != nullptr;
    if (psplit) {
      CKC(c, cudaEventRecord(c->ev[6], st));
      CKC(c, cudaStreamWaitEvent(c->st2, c->ev[6], 0));
      A.psplit = 1;
      CKC(c, launch_proj_setup(A, (D == 3) ? std::max(B.th_l, 256) : B.th_l, c->st2));
      CKC(c, cudaEventRecord(c->ev[7], c->st2));
      A.psplit = 2;
      S.launches += 1;
    }
    if (A.coarse) {
      CKC(c, launch_coarse_setup(A, st));
      S.launches += 1;
    }
    if (psplit) CKC(c, cudaStreamWaitEvent(st, c->ev[7], 0));
    CKC(c, launch_proj_setup(A, (D == 3) ? std::max(B.th_l, 256) : B.th_l, st));
    A.psplit = 0;
    CKC(c, launch_pinv(A, st));
    S.launches += 1;
    if (B.on2d && !B.l1op) {
      CKC(c, launch_node_ops2d(A, B.max_ln, st));
      S.launches += 1;
    }
    if (B.on3d && level >= 2) {
      CKC(c, launch_node_ops3d(A, B.max_ln, st));
      S.launches += 1;
    }
    cudaEventRecord(B.ev[1], st);
    nvtxRangePop();
    nvtxRangePushA("projected PCG");
    double* dbgp = nullptr;
    if (getenv("MCH_PCG_DEBUG") && B.on2d) {  // dev: per-iteration scalars of one problem to stderr
      A.dbg_prob = atoi(getenv("MCH_PCG_DEBUG"));
      A.dbg_cap = 400;
      cudaMalloc(&dbgp, 8 * sizeof(double) * A.dbg_cap);
      cudaMemset(dbgp, 0, 8 * sizeof(double) * A.dbg_cap);
      A.dbg = dbgp;
    }
    if (B.on2d) CKC(c, launch_pcg2d(A, B.variant, B.threads2, st));
    else if (B.on3d && level == 1 && B.l1cs > 0) CKC(c, launch_pcg3d_l1c(A, B.l1cs, st));
    else if (B.on3d && level == 1) CKC(c, launch_pcg3d_l1(A, st));
    else if (B.w7) CKC(c, launch_pcg3d_w7(A, st));
    else if (B.on3d && B.l2cs > 1) CKC(c, launch_pcg3dc(A, B.nxm3, B.l2cs, st));
    else if (B.on3d) CKC(c, launch_pcg3d(A, B.nxm3, st));
    else CKC(c, launch_pcg(A, B.th_l, st));
    if (dbgp) {
      std::vector<double> h(8 * A.dbg_cap);
      cudaMemcpy(h.data(), dbgp, h.size() * sizeof(double), cudaMemcpyDeviceToHost);
      for (int i = 0; i < A.dbg_cap && h[8 * i] != 0.0; i++)
        fprintf(stderr, "[dbg L%d prob %d] it %d rz %.17e pq %.17e alpha %.17e beta %.17e\n", level, A.dbg_prob, i,
                h[8 * i], h[8 * i + 1], h[8 * i + 2], h[8 * i + 3]);
      cudaFree(dbgp);
      A.dbg = nullptr;
    }
    cudaEventRecord(B.ev[2], st);
    nvtxRangePop();
    NvtxRange nv_gram("combine + Eq. (7)");
    if (getenv("MCH_PCG_TIMING") && B.on2d) {
      char tag[64];
      snprintf(tag, sizeof tag, "level %d variant %d", level, B.variant);
      pcg2d_phase_dump(tag);
    }
    if (level >= 2 && B.fused3) CKC(c, launch_fine3d_combine(A, B.max_comb, st));
    else if (level >= 2) CKC(c, launch_combine(A, B.th_f, st));
    if (B.fused3 && A.f == nullptr && (nr == 4 || nr == 8)) CKC(c, launch_gram3_kp(A, st));
    else CKC(c, launch_gram(A, 256, st));
    cudaEventRecord(B.ev[3], st);
    CKC(c, cudaMemcpyAsync(B.h_flags, c->flags.ptr, sizeof(int) * nmp, cudaMemcpyDeviceToHost, st));
    CKC(c, cudaMemcpyAsync(B.h_iters, c->iters.ptr, sizeof(int) * nmp * nr, cudaMemcpyDeviceToHost, st));
    CKC(c, cudaMemcpyAsync(B.h_relres, c->relres.ptr, sizeof(double) * nmp * nr, cudaMemcpyDeviceToHost, st));
    CKC(c, cudaMemcpyAsync(B.h_diag, c->diag.ptr, sizeof(double) * nmp * nr * 4, cudaMemcpyDeviceToHost, st));
    // batches share the scratch: a later batch may only start after this one's results are read
    if (multi) CKC(c, cudaStreamSynchronize(st));
  }
  // exchange step (i): the parents of S_level go to the ranks whose children of
  // later levels read them (Eq. 11), grouped point-to-point NCCL transfers of whole pool slots
  cudaEventRecord(c->ev[4], st);
  if (c->comm && level < c->p.levels && !c->shard.xfer[level].empty()) {
    NvtxRange nv_x("parent exchange (NCCL)");
    const NcclApi* nc_ = c->nccl;
    ncclResult_t nr_ = nc_->GroupStart();
    for (const auto& x : c->shard.xfer[level]) {
      if (nr_ != ncclSuccess) break;
      int64_t len = 0, offp = c->pool_off[x[0]];
      {
        const MacroHost& pm = pl.all[x[0]];
        len = c->n_rhs;
        for (int d = 0; d < D; d++) len *= (pm.hi[d] - pm.lo[d] + 1);
      }
      if (x[1] == c->p.rank) nr_ = nc_->Send(c->pool + offp, (size_t)len, ncclFloat64, (int)x[2], c->comm, st);
      else if (x[2] == c->p.rank) nr_ = nc_->Recv(c->pool + offp, (size_t)len, ncclFloat64, (int)x[1], c->comm, st);
      if (x[1] == c->p.rank || x[2] == c->p.rank) S.bytes_comm += 8.0 * (double)len;
    }
    const ncclResult_t ge = nc_->GroupEnd();
    if (nr_ == ncclSuccess) nr_ = ge;
    if (nr_ != ncclSuccess) return fail(c, MCH_ENCCL, std::string("parent exchange: ") + nc_->GetErrorString(nr_));
    S.launches += 1;
  }
  cudaEventRecord(c->ev[5], st);
  CKC(c, cudaEventSynchronize(c->ev[5]));
  {
    float tc = 0;
    cudaEventElapsedTime(&tc, c->ev[4], c->ev[5]);
    S.ms_comm = tc;
  }
  float ms_setup = 0, ms_pcg = 0, ms_gram = 0, ms_tr = 0;
  for (size_t bi = 0; bi < batches.size(); bi++) {
    LevelBatch& B = *batches[bi];
    float t1 = 0, t2 = 0, t3 = 0;
    cudaEventElapsedTime(&t1, B.ev[0], B.ev[1]);
    cudaEventElapsedTime(&t2, B.ev[1], B.ev[2]);
    cudaEventElapsedTime(&t3, B.ev[2], B.ev[3]);
    ms_setup += t1; ms_pcg += t2; ms_gram += t3;
    float t4 = 0;
    cudaEventElapsedTime(&t4, B.ev[4], B.ev[5]);
    ms_tr += t4;
    S.transport_units += B.tr_units;
    S.transport_flops += B.tr_flops;
    for (int i = 0; i < B.nmp; i++) {
      const MacroHost& m = pl.all[B.mps[i]];
      if (B.h_flags[i] & 4) S.rank_deficient++;  // k_pinv truncated eigenvalues (reading R20)
      if ((B.h_flags[i] & 16) && getenv("MCH_PINV_STATS_PRINT"))
        fprintf(stderr, "[pinv] level %d macropoint %d: Jacobi eigen-solver (rank not certified by the direct form)\n", level, i);
      if ((B.h_flags[i] >> 8) && getenv("MCH_PINV_STATS_PRINT") && i < 4)
        fprintf(stderr, "[pinv] level %d macropoint %d sweeps %d\n", level, i, B.h_flags[i] >> 8);
      if (B.h_flags[i] & 8) {
        char buf[200];
        snprintf(buf, sizeof buf, "dependent constraint rows at macropoint (%d,%d,%d): the banded projector of "
                 "large oversampling does not handle reading R20", m.k[0], m.k[1], m.k[2]);
        return fail(c, MCH_ERANK, buf);
      }
      if (B.h_flags[i] & 1) {
        char buf[200];
        snprintf(buf, sizeof buf, "continuum absent from K_p of macropoint (%d,%d,%d)", m.k[0], m.k[1], m.k[2]);
        return fail(c, MCH_ERANK, buf);
      }
      const int64_t ln = B.ln[i], lc = B.lc[i];
      int mx = 0;
      bool bad = false;
      int badr = 0;
      for (int r = 0; r < nr; r++) {
        const int it = B.h_iters[i * nr + r];
        if (B.h_diag[(i * nr + r) * 4 + 3] != 0.0 || it >= c->p.max_iter) { bad = true; badr = r; }
        S.iters_total += it;
        mx = std::max(mx, it);
        S.relres_max = std::max(S.relres_max, B.h_relres[i * nr + r]);
        S.pcg_bytes += 8.0 * 6.0 * (double)ln * it;
        S.node_iters += (double)ln * it;
      }
      S.iters_max = std::max<int64_t>(S.iters_max, mx);
      S.unknowns_level += ln;
      S.cells_level += lc;
      const double Dn = (level == 1) ? 1.0 : ((D == 2) ? 5.0 : 19.0);
      S.pcg_bytes += 8.0 * Dn * (double)lc * mx;
      if (bad) {
        const double* dg = &B.h_diag[(i * nr + badr) * 4];
        char buf[320];
        snprintf(buf, sizeof buf,
                 "PCG did not converge at level %d macropoint (%d,%d,%d) rhs %d: %s after %d iterations, "
                 "relres %.3e (rz %.3e, ref %.3e, floor %.3e)",
                 level, m.k[0], m.k[1], m.k[2], badr, dg[3] != 0.0 ? "breakdown" : "iteration cap",
                 B.h_iters[i * nr + badr], B.h_relres[i * nr + badr], dg[0], dg[1], dg[2]);
        return fail(c, MCH_ENOCONV, buf);
      }
    }
    S.macropoints += B.nmp;
    S.problems += (int64_t)B.nmp * nr;
  }
  float tt = 0;
  cudaEventElapsedTime(&tt, c->ev[0], c->ev[5]);
  S.ms_total = tt;
  S.ms_setup = ms_setup;
  S.ms_pcg = ms_pcg;
  S.ms_gram = ms_gram;
  S.ms_transport = ms_tr;
  c->solved = level;
  return MCH_OK;
}

extern "C" int mch_set_medium(mch_ctx* c, const double* kappa, const uint8_t* ids, int on_dev) {
  if (!c) return MCH_EINVAL;
  if (!kappa || !ids) return fail(c, MCH_EINVAL, "NULL argument");
  const int64_t n = c->p.n;
  const int64_t cells = (c->D == 2) ? n * n : n * n * n;
  const cudaMemcpyKind kind = on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  CKC(c, cudaMemcpyAsync(c->kappa, kappa, cells * sizeof(double), kind, c->st));
  CKC(c, cudaMemcpyAsync(c->ids, ids, cells, kind, c->st));
  // validation on the device (no host pass over the inputs), one pinned flag read back
  if (!c->h_bad) CKC(c, cudaMallocHost(&c->h_bad, sizeof(int)));
  if (!c->d_bad) CKC(c, dev_alloc(&c->al, (void**)&c->d_bad, sizeof(int)));
  CKC(c, cudaMemsetAsync(c->d_bad, 0, sizeof(int), c->st));
  CKC(c, launch_validate(c->kappa, c->ids, cells, c->N, c->d_bad, c->st));
  CKC(c, cudaMemcpyAsync(c->h_bad, c->d_bad, sizeof(int), cudaMemcpyDeviceToHost, c->st));
  CKC(c, cudaStreamSynchronize(c->st));
  c->solved = 0;
  c->medium_ok = (*c->h_bad == 0);
  if (!c->medium_ok) return fail(c, MCH_EINVAL, "kappa must be positive and finite; ids < num_continua");
  return MCH_OK;
}

extern "C" int mch_reset(mch_ctx* c) {
  if (!c) return MCH_EINVAL;
  c->solved = 0;
  return MCH_OK;
}

extern "C" int mch_effective_coeffs(mch_ctx* c, double* out, size_t out_len, int out_on_device) {
  if (!c || !out) return MCH_EINVAL;
  if (c->solved != c->p.levels) return fail(c, MCH_EORDER, "coefficients need all levels solved");
  const size_t need = c->plan.all.size() * (size_t)c->n_rhs * c->n_rhs;
  if (out_len < need) return fail(c, MCH_EINVAL, "out_len too small");
  const double* src = c->G;
  if (c->comm) {  // exchange step (ii): non-owned entries are exactly 0, so the sum is exact
    CKC(c, c->Gall.ensure(need * sizeof(double)));
    const ncclResult_t r = c->nccl->AllReduce(c->G, c->Gall.ptr, need, ncclFloat64, ncclSum, c->comm, c->st);
    if (r != ncclSuccess) return fail(c, MCH_ENCCL, std::string("coefficient all-reduce: ") + c->nccl->GetErrorString(r));
    src = c->Gall.as<double>();
  }
  CKC(c, cudaMemcpyAsync(out, src, need * sizeof(double),
                         out_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c->st));
  CKC(c, cudaStreamSynchronize(c->st));
  return MCH_OK;
}

extern "C" int mch_set_source(mch_ctx* c, const double* f, int on_dev) {
  if (!c) return MCH_EINVAL;
  if (c->solved != 0) return fail(c, MCH_EORDER, "set the source before solving level 1 (or after mch_reset)");
  if (!f) {
    c->has_source = false;
    return MCH_OK;
  }
  const int64_t n = c->p.n;
  const int64_t cells = (c->D == 2) ? n * n : n * n * n;
  if (!on_dev)
    for (int64_t i = 0; i < cells; i++)
      if (!std::isfinite(f[i])) return fail(c, MCH_EINVAL, "source must be finite");
  const size_t nb = c->plan.all.size() * (size_t)c->N;
  CKC(c, c->fsrc.ensure(cells * sizeof(double)));
  CKC(c, c->bload.ensure(nb * sizeof(double)));
  CKC(c, cudaMemcpyAsync(c->fsrc.ptr, f, cells * sizeof(double), on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c->st));
  CKC(c, cudaMemsetAsync(c->bload.ptr, 0, nb * sizeof(double), c->st));
  CKC(c, cudaStreamSynchronize(c->st));
  c->has_source = true;
  return MCH_OK;
}

extern "C" int mch_load_vectors(mch_ctx* c, double* out, size_t out_len, int out_on_device) {
  if (!c || !out) return MCH_EINVAL;
  if (!c->has_source) return fail(c, MCH_EINVAL, "no source set (mch_set_source)");
  if (c->solved != c->p.levels) return fail(c, MCH_EORDER, "load vectors need all levels solved");
  const size_t need = c->plan.all.size() * (size_t)c->N;
  if (out_len < need) return fail(c, MCH_EINVAL, "out_len too small");
  const void* bsrc = c->bload.ptr;
  if (c->comm) {
    CKC(c, c->ball.ensure(need * sizeof(double)));
    const ncclResult_t r = c->nccl->AllReduce(c->bload.ptr, c->ball.ptr, need, ncclFloat64, ncclSum, c->comm, c->st);
    if (r != ncclSuccess) return fail(c, MCH_ENCCL, std::string("load all-reduce: ") + c->nccl->GetErrorString(r));
    bsrc = c->ball.ptr;
  }
  CKC(c, cudaMemcpyAsync(out, bsrc, need * sizeof(double),
                         out_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c->st));
  CKC(c, cudaStreamSynchronize(c->st));
  return MCH_OK;
}

extern "C" int mch_macro_solve(mch_ctx* c, const double* G, const double* b, int inputs_on_device, double* U,
                               size_t U_len, int out_on_device, double rtol, int max_iter, int* iters) {
  if (!c || !U) return MCH_EINVAL;
  if (c->p.layout != MCH_LAYOUT_BLOCK)
    return fail(c, MCH_EINVAL, "the macro solve needs the block-centred layout (PAPER.md:199: block midpoints)");
  const int D = c->D, N = c->N, nr = c->n_rhs;
  const int64_t M = c->p.M;
  int64_t nodes = 1;
  for (int i = 0; i < D; i++) nodes *= M + 1;
  const size_t P = c->plan.all.size();
  if (U_len < (size_t)(nodes * N)) return fail(c, MCH_EINVAL, "U_len too small");
  if ((G == nullptr) != (b == nullptr)) return fail(c, MCH_EINVAL, "pass both G and b, or neither");
  if (rtol <= 0.0) rtol = 1e-12;
  if (max_iter <= 0) max_iter = 100000;
  const double* dG = G;
  const double* db = b;
  if (!G) {
    if (c->p.world > 1) return fail(c, MCH_EINVAL, "world > 1: pass the all-reduced coefficients and loads");
    if (!c->has_source) return fail(c, MCH_EINVAL, "no source set (mch_set_source)");
    if (c->solved != c->p.levels) return fail(c, MCH_EORDER, "the macro solve needs all levels solved");
    dG = c->G;
    db = c->bload.as<double>();
  } else if (!inputs_on_device) {
    CKC(c, c->mG.ensure(P * nr * nr * sizeof(double)));
    CKC(c, c->mb.ensure(P * N * sizeof(double)));
    CKC(c, cudaMemcpyAsync(c->mG.ptr, G, P * nr * nr * sizeof(double), cudaMemcpyHostToDevice, c->st));
    CKC(c, cudaMemcpyAsync(c->mb.ptr, b, P * N * sizeof(double), cudaMemcpyHostToDevice, c->st));
    dG = c->mG.as<double>();
    db = c->mb.as<double>();
  }
  double* dU = U;
  if (!out_on_device) {
    CKC(c, c->mU.ensure(nodes * N * sizeof(double)));
    dU = c->mU.as<double>();
  }
  CKC(c, c->mws.ensure(macro_workspace_doubles(D, N, M) * sizeof(double)));
  CKC(c, c->mres.ensure(2 * sizeof(double)));
  if (!c->h_mit) CKC(c, cudaMallocHost(&c->h_mit, sizeof(int)));
  if (!c->h_mrel) CKC(c, cudaMallocHost(&c->h_mrel, sizeof(double)));
  int* d_it = reinterpret_cast<int*>(c->mres.as<double>() + 1);
  CKC(c, launch_macro_pcg(D, N, M, dG, db, dU, c->mws.as<double>(), rtol, max_iter, d_it, c->mres.as<double>(), c->st));
  c->launches += 1;
  if (!out_on_device)
    CKC(c, cudaMemcpyAsync(U, dU, nodes * N * sizeof(double), cudaMemcpyDeviceToHost, c->st));
  CKC(c, cudaMemcpyAsync(c->h_mit, d_it, sizeof(int), cudaMemcpyDeviceToHost, c->st));
  CKC(c, cudaMemcpyAsync(c->h_mrel, c->mres.ptr, sizeof(double), cudaMemcpyDeviceToHost, c->st));
  CKC(c, cudaStreamSynchronize(c->st));
  if (iters) *iters = *c->h_mit;
  if (!(*c->h_mrel <= rtol)) {
    char buf[160];
    snprintf(buf, sizeof buf, "macro PCG: relative residual %.3e after %d iterations", *c->h_mrel, *c->h_mit);
    return fail(c, MCH_ENOCONV, buf);
  }
  return MCH_OK;
}

extern "C" int mch_fine_solve(mch_ctx* c, const double* f, int f_on_device, double* u, size_t u_len, int u_on_device,
                              double rtol, int max_iter, int* iters) {
  if (!c || !f || !u) return c ? fail(c, MCH_EINVAL, "NULL argument") : MCH_EINVAL;
  const int D = c->D;
  const int64_t n = c->p.n;
  int64_t cells = 1, nn = 1;
  for (int i = 0; i < D; i++) {
    cells *= n;
    nn *= n + 1;
  }
  if (u_len < (size_t)nn) return fail(c, MCH_EINVAL, "u_len too small");
  if (rtol <= 0.0) rtol = 1e-10;
  if (max_iter <= 0) max_iter = 1000000;
  if (!f_on_device)
    for (int64_t i = 0; i < cells; i++)
      if (!std::isfinite(f[i])) return fail(c, MCH_EINVAL, "source must be finite");
  const double* df = f;
  if (!f_on_device) {
    CKC(c, c->ff.ensure(cells * sizeof(double)));
    CKC(c, cudaMemcpyAsync(c->ff.ptr, f, cells * sizeof(double), cudaMemcpyHostToDevice, c->st));
    df = c->ff.as<double>();
  }
  const int grid = fine_grid_size(D);
  CKC(c, c->fws.ensure(fine_workspace_doubles(D, n, grid) * sizeof(double)));
  CKC(c, c->fbar.ensure(4 * sizeof(unsigned) + 2 * sizeof(double)));
  if (!c->h_mit) CKC(c, cudaMallocHost(&c->h_mit, sizeof(int)));
  if (!c->h_mrel) CKC(c, cudaMallocHost(&c->h_mrel, sizeof(double)));
  unsigned* bar = reinterpret_cast<unsigned*>(c->fbar.ptr);
  int* d_it = reinterpret_cast<int*>(bar + 2);
  double* d_rel = reinterpret_cast<double*>(bar + 4);
  CKC(c, launch_fine_pcg(D, n, c->kappa, df, c->fws.as<double>(), bar, grid, rtol, max_iter, d_it, d_rel, c->st));
  c->launches += 1;
  CKC(c, cudaMemcpyAsync(u, c->fws.ptr, nn * sizeof(double), u_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                         c->st));
  CKC(c, cudaMemcpyAsync(c->h_mit, d_it, sizeof(int), cudaMemcpyDeviceToHost, c->st));
  CKC(c, cudaMemcpyAsync(c->h_mrel, d_rel, sizeof(double), cudaMemcpyDeviceToHost, c->st));
  CKC(c, cudaStreamSynchronize(c->st));
  if (iters) *iters = *c->h_mit;
  if (!(*c->h_mrel <= rtol)) {
    char buf[160];
    snprintf(buf, sizeof buf, "fine PCG: relative residual %.3e after %d iterations", *c->h_mrel, *c->h_mit);
    return fail(c, MCH_ENOCONV, buf);
  }
  return MCH_OK;
}

extern "C" int mch_fine_block_averages(mch_ctx* c, const double* u, int u_on_device, double* out, size_t out_len,
                                       int out_on_device) {
  if (!c || !u || !out) return c ? fail(c, MCH_EINVAL, "NULL argument") : MCH_EINVAL;
  const int D = c->D, N = c->N;
  const int64_t n = c->p.n;
  int64_t nn = 1;
  for (int i = 0; i < D; i++) nn *= n + 1;
  const HostPlan& pl = c->plan;
  const int64_t P = (int64_t)pl.all.size();
  if (out_len < (size_t)(P * N)) return fail(c, MCH_EINVAL, "out_len too small");
  std::vector<int> kb(6 * P, 0);
  for (int64_t m = 0; m < P; m++)
    for (int d = 0; d < 3; d++) {
      const int64_t a = (int64_t)pl.all[m].k[d] * pl.c - pl.coff(), b = a + pl.c;  // K_p
      kb[6 * m + d] = (d < D) ? (int)std::max<int64_t>(0, a) : 0;
      kb[6 * m + 3 + d] = (d < D) ? (int)std::min<int64_t>(n, b) : 1;
    }
  CKC(c, c->fkbox.ensure(kb.size() * sizeof(int)));
  CKC(c, cudaMemcpyAsync(c->fkbox.ptr, kb.data(), kb.size() * sizeof(int), cudaMemcpyHostToDevice, c->st));
  const double* du = u;
  if (!u_on_device) {
    CKC(c, c->fu.ensure(nn * sizeof(double)));
    CKC(c, cudaMemcpyAsync(c->fu.ptr, u, nn * sizeof(double), cudaMemcpyHostToDevice, c->st));
    du = c->fu.as<double>();
  }
  double* dout = out;
  if (!out_on_device) {
    CKC(c, c->fout.ensure(P * N * sizeof(double)));
    dout = c->fout.as<double>();
  }
  CKC(c, launch_fine_block_avg(D, du, c->ids, c->fkbox.as<int>(), P, n, N, dout, c->st));
  c->launches += 1;
  if (!out_on_device)
    CKC(c, cudaMemcpyAsync(out, dout, P * N * sizeof(double), cudaMemcpyDeviceToHost, c->st));
  CKC(c, cudaStreamSynchronize(c->st));
  return MCH_OK;
}

extern "C" int mch_num_macropoints(const mch_ctx* c, int level, int64_t* count) {
  if (!c || !count || level < 1 || level > c->p.levels) return MCH_EINVAL;
  *count = (int64_t)c->plan.S[level].size();
  return MCH_OK;
}

extern "C" int mch_level_macropoints(const mch_ctx* c, int level, int64_t* out, size_t cap) {
  if (!c || !out || level < 1 || level > c->p.levels) return MCH_EINVAL;
  const std::vector<int64_t>& Sl = c->plan.S[level];
  if (cap < Sl.size()) return MCH_EINVAL;
  for (size_t i = 0; i < Sl.size(); i++) out[i] = Sl[i];
  return MCH_OK;
}

extern "C" int mch_local_solution(mch_ctx* c, int64_t mp, int rhs, double* out, size_t out_len, int64_t ext[3]) {
  if (!c || !out || mp < 0 || mp >= (int64_t)c->plan.all.size() || rhs < 0 || rhs >= c->n_rhs)
    return c ? fail(c, MCH_EINVAL, "bad macropoint/rhs") : MCH_EINVAL;
  const MacroHost& m = c->plan.all[mp];
  if (c->pool_off[mp] < 0) return fail(c, MCH_EINVAL, "local solution not kept (use keep_all)");
  if (m.level > c->solved) return fail(c, MCH_EORDER, "level not solved yet");
  int64_t fn = 1;
  for (int d = 0; d < 3; d++) {
    const int64_t e = (d < c->D) ? (m.hi[d] - m.lo[d] + 1) : 1;
    if (ext) ext[d] = e;
    fn *= e;
  }
  if (out_len < (size_t)fn) return fail(c, MCH_EINVAL, "out_len too small");
  CKC(c, cudaMemcpyAsync(out, c->pool + c->pool_off[mp] + (int64_t)rhs * fn, fn * sizeof(double),
                         cudaMemcpyDefault, c->st));
  CKC(c, cudaStreamSynchronize(c->st));
  return MCH_OK;
}

extern "C" int mch_get_level_stats(const mch_ctx* c, int level, mch_level_stats* out) {
  if (!c || !out || level < 1 || level > c->p.levels) return MCH_EINVAL;
  *out = c->stats[level];
  return MCH_OK;
}

extern "C" int mch_level_iterations(const mch_ctx* c, int level, int32_t* out, size_t cap) {
  if (!c || !out || level < 1 || level > c->p.levels) return MCH_EINVAL;
  if (level > c->solved || (int)c->lplans.size() <= level) return MCH_EORDER;
  size_t total = 0;
  for (const auto& B : c->lplans[level]) total += (size_t)B->nmp * c->n_rhs;
  if (total > cap) return MCH_EINVAL;
  for (const auto& B : c->lplans[level])
    for (int i = 0; i < B->nmp; i++)
      memcpy(out + (size_t)B->lexpos[i] * c->n_rhs, B->h_iters + (size_t)i * c->n_rhs, c->n_rhs * sizeof(int32_t));
  return MCH_OK;
}

// ---- checkpoint / resume (include/mch.h) ------------------------------------------------------
namespace {
struct CkptHeader {
  char magic[8];  // "MCHCKPT1"
  int32_t d, num_continua, levels, eta, oversample, interp, layout, keep_all, rank, world, solved, has_source;
  int64_t n, M, pool_len, g_len, b_len;
  uint64_t medium;
};

int medium_fingerprint(mch_ctx* c, uint64_t* out) {
  const int64_t n = c->p.n, cells = (c->D == 2) ? n * n : n * n * n;
  unsigned long long* d = nullptr;
  CKC(c, dev_alloc(&c->al, (void**)&d, sizeof(unsigned long long)));
  cudaError_t e = cudaMemsetAsync(d, 0, sizeof(unsigned long long), c->st);
  if (e == cudaSuccess) e = launch_fingerprint(c->kappa, c->ids, cells, d, c->st);
  unsigned long long h = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, c->st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->st);
  dev_free(&c->al, d);
  CKC(c, e);
  *out = h;
  return MCH_OK;
}

CkptHeader ckpt_header(const mch_ctx* c) {
  CkptHeader h{};
  memcpy(h.magic, "MCHCKPT1", 8);
  h.d = c->p.d; h.num_continua = c->p.num_continua; h.levels = c->p.levels; h.eta = c->p.eta;
  h.oversample = c->p.oversample; h.interp = c->p.interp; h.layout = c->p.layout; h.keep_all = c->p.keep_all;
  h.rank = c->p.rank; h.world = c->p.world; h.solved = c->solved; h.has_source = c->has_source ? 1 : 0;
  h.n = c->p.n; h.M = c->p.M; h.pool_len = c->pool_len;
  h.g_len = (int64_t)c->plan.all.size() * c->n_rhs * c->n_rhs;
  h.b_len = c->has_source ? (int64_t)c->plan.all.size() * c->N : 0;
  return h;
}

// device array <-> file through a pinned staging buffer (64 MB pieces)
int ckpt_stream(mch_ctx* c, FILE* f, double* dev, int64_t len, bool save, double* stage, int64_t cap) {
  for (int64_t o = 0; o < len; o += cap) {
    const int64_t m = std::min(cap, len - o);
    if (save) {
      CKC(c, cudaMemcpyAsync(stage, dev + o, m * sizeof(double), cudaMemcpyDeviceToHost, c->st));
      CKC(c, cudaStreamSynchronize(c->st));
      if (fwrite(stage, sizeof(double), (size_t)m, f) != (size_t)m) return fail(c, MCH_EINVAL, "checkpoint: write failed");
    } else {
      if (fread(stage, sizeof(double), (size_t)m, f) != (size_t)m) return fail(c, MCH_EINVAL, "checkpoint: file truncated");
      CKC(c, cudaMemcpyAsync(dev + o, stage, m * sizeof(double), cudaMemcpyHostToDevice, c->st));
      CKC(c, cudaStreamSynchronize(c->st));
    }
  }
  return MCH_OK;
}

int ckpt_run(mch_ctx* c, const char* path, bool save) {
  if (!c || !path) return MCH_EINVAL;
  if (!c->medium_ok) return fail(c, MCH_EINVAL, "checkpoint: the context holds no valid medium");
  uint64_t fp = 0;
  if (int rc = medium_fingerprint(c, &fp)) return rc;
  FILE* f = fopen(path, save ? "wb" : "rb");
  if (!f) return fail(c, MCH_EINVAL, std::string("checkpoint: cannot open ") + path);
  CkptHeader h = ckpt_header(c);
  h.medium = fp;
  int rc = MCH_OK;
  if (save) {
    if (fwrite(&h, sizeof(h), 1, f) != 1) rc = fail(c, MCH_EINVAL, "checkpoint: write failed");
  } else {
    CkptHeader g{};
    if (fread(&g, sizeof(g), 1, f) != 1 || memcmp(g.magic, "MCHCKPT1", 8) != 0) {
      rc = fail(c, MCH_EINVAL, "checkpoint: not a checkpoint file");
    } else {
      const int solved = g.solved, src = g.has_source;
      const int64_t bl = g.b_len;
      g.solved = h.solved; g.has_source = h.has_source; g.b_len = h.b_len;  // state, not layout
      if (memcmp(&g, &h, sizeof(h)) != 0)
        rc = fail(c, MCH_EINVAL, (g.medium != h.medium) ? "checkpoint: the medium differs from the one it was taken on"
                                                        : "checkpoint: parameters differ from the context's");
      else if (solved < 0 || solved > c->p.levels || (src != 0) != c->has_source)
        rc = fail(c, MCH_EINVAL, "checkpoint: solved level out of range, or source set on one side only");
      h.solved = solved;
      h.b_len = bl;
    }
  }
  double* stage = nullptr;
  const int64_t cap = (int64_t)8 << 20;
  if (rc == MCH_OK && cudaMallocHost(&stage, cap * sizeof(double)) != cudaSuccess) rc = fail(c, MCH_ENOMEM, "checkpoint: staging buffer");
  if (rc == MCH_OK) rc = ckpt_stream(c, f, c->pool, h.pool_len, save, stage, cap);
  if (rc == MCH_OK) rc = ckpt_stream(c, f, c->G, h.g_len, save, stage, cap);
  if (rc == MCH_OK && h.b_len > 0) rc = ckpt_stream(c, f, c->bload.as<double>(), h.b_len, save, stage, cap);
  if (stage) cudaFreeHost(stage);
  if (fclose(f) != 0 && rc == MCH_OK && save) rc = fail(c, MCH_EINVAL, "checkpoint: close failed");
  if (rc == MCH_OK && !save) c->solved = h.solved;
  return rc;
}
}  // namespace

extern "C" int mch_checkpoint_save(mch_ctx* c, const char* path) { return ckpt_run(c, path, true); }
extern "C" int mch_checkpoint_load(mch_ctx* c, const char* path, int* solved_levels) {
  const int rc = ckpt_run(c, path, false);
  if (rc == MCH_OK && solved_levels) *solved_levels = c->solved;
  return rc;
}

extern "C" int mch_pool_info(const mch_ctx* c, double** pool, int64_t* len) {
  if (!c) return MCH_EINVAL;
  if (pool) *pool = c->pool;
  if (len) *len = c->pool_len;
  return MCH_OK;
}

extern "C" int mch_pool_slot(const mch_ctx* c, int64_t mp, int64_t* offset, int64_t* length) {
  if (!c || mp < 0 || mp >= (int64_t)c->plan.all.size()) return MCH_EINVAL;
  const MacroHost& m = c->plan.all[mp];
  int64_t fn = 1;
  for (int d = 0; d < c->D; d++) fn *= (m.hi[d] - m.lo[d] + 1);
  if (offset) *offset = c->pool_off[mp];
  if (length) *length = (c->pool_off[mp] >= 0) ? fn * c->n_rhs : 0;
  return MCH_OK;
}

extern "C" int mch_coeffs_device(const mch_ctx* c, double** G) {
  if (!c || !G) return MCH_EINVAL;
  *G = c->G;
  return MCH_OK;
}

extern "C" const char* mch_last_error(const mch_ctx* c) {
  return c ? c->err.c_str() : g_create_error.c_str();
}

extern "C" void mch_destroy(mch_ctx* c) {
  if (!c) return;
  if (c->st) cudaStreamSynchronize(c->st);
  else cudaDeviceSynchronize();
  dev_free(&c->al, c->kappa);
  dev_free(&c->al, c->ids);
  dev_free(&c->al, c->pool);
  dev_free(&c->al, c->G);
  c->lplans.clear();
  if (c->h_bad) cudaFreeHost(c->h_bad);
  if (c->h_mit) cudaFreeHost(c->h_mit);
  if (c->h_mrel) cudaFreeHost(c->h_mrel);
  if (c->d_bad) dev_free(&c->al, c->d_bad);
  for (DevBuf* b : c->bufs()) b->release();
  // (LevelBatch buffers are released by lplans.clear() above)
  if (c->events)
    for (int i = 0; i < 8; i++) cudaEventDestroy(c->ev[i]);
  if (c->st2) cudaStreamDestroy(c->st2);
  delete c;
}

// ------------------------------------------------------------------------------------------
// multi-GPU plumbing
extern "C" int mch_comm_id(void* id, size_t id_len) {
  if (!id || id_len < sizeof(ncclUniqueId)) return fail(nullptr, MCH_EINVAL, "id buffer too small (128 bytes)");
  std::string err;
  const NcclApi* api = nccl_api(err);
  if (!api) return fail(nullptr, MCH_ENCCL, err);
  ncclUniqueId u;
  const ncclResult_t r = api->GetUniqueId(&u);
  if (r != ncclSuccess) return fail(nullptr, MCH_ENCCL, api->GetErrorString(r));
  memcpy(id, &u, sizeof(u));
  return MCH_OK;
}

extern "C" int mch_comm_init(void** comm, int world, int rank, const void* id, size_t id_len) {
  if (!comm || !id || id_len < sizeof(ncclUniqueId) || world < 1 || rank < 0 || rank >= world)
    return fail(nullptr, MCH_EINVAL, "bad communicator arguments");
  std::string err;
  const NcclApi* api = nccl_api(err);
  if (!api) return fail(nullptr, MCH_ENCCL, err);
  ncclUniqueId u;
  memcpy(&u, id, sizeof(u));
  ncclComm_t cm = nullptr;
  const ncclResult_t r = api->CommInitRank(&cm, world, u, rank);
  if (r != ncclSuccess) return fail(nullptr, MCH_ENCCL, api->GetErrorString(r));
  *comm = cm;
  return MCH_OK;
}

extern "C" int mch_comm_destroy(void* comm) {
  if (!comm) return MCH_OK;
  std::string err;
  const NcclApi* api = nccl_api(err);
  if (!api) return fail(nullptr, MCH_ENCCL, err);
  const ncclResult_t r = api->CommDestroy(reinterpret_cast<ncclComm_t>(comm));
  return r == ncclSuccess ? MCH_OK : fail(nullptr, MCH_ENCCL, api->GetErrorString(r));
}

extern "C" int mch_shard_plan(const mch_params* prm, int level, int64_t* owned, size_t owned_cap, int64_t* n_owned,
                              int64_t* xfers, size_t xfer_cap, int64_t* n_xfers) {
  if (!prm) return fail(nullptr, MCH_EINVAL, "NULL params");
  mch_params p = *prm;
  if (p.d != 2 && p.d != 3) return fail(nullptr, MCH_EINVAL, "d must be 2 or 3");
  if (p.oversample < 1) p.oversample = 1;
  if (p.world < 1) { p.world = 1; p.rank = 0; }
  if (p.rank < 0 || p.rank >= p.world) return fail(nullptr, MCH_EINVAL, "bad rank/world");
  if (level < 1 || level > p.levels) return fail(nullptr, MCH_EINVAL, "bad level");
  HostPlan pl;
  pl.D = p.d; pl.n = p.n; pl.M = p.M; pl.L = p.levels; pl.eta = p.eta; pl.l = p.oversample;
  pl.interp = p.interp; pl.layout = p.layout;
  std::string perr;
  const int rc = pl.build(perr);
  if (rc != 0) return fail(nullptr, rc == -8 ? MCH_EPLAN : MCH_EDIVISIBILITY, perr);
  ShardPlan sp;
  shard_build(pl, p.world, sp);
  int64_t k = 0;
  for (size_t i = 0; i < pl.S[level].size(); i++)
    if (sp.owner[level][i] == p.rank) {
      if (owned && (size_t)k < owned_cap) owned[k] = pl.S[level][i];
      k++;
    }
  if (n_owned) *n_owned = k;
  if (owned && (size_t)k > owned_cap) return fail(nullptr, MCH_EINVAL, "owned_cap too small");
  const auto& xf = sp.xfer[level];
  if (n_xfers) *n_xfers = (int64_t)xf.size();
  if (xfers) {
    if (xf.size() > xfer_cap) return fail(nullptr, MCH_EINVAL, "xfer_cap too small");
    for (size_t i = 0; i < xf.size(); i++)
      for (int j = 0; j < 3; j++) xfers[3 * i + j] = xf[i][j];
  }
  return MCH_OK;
}
