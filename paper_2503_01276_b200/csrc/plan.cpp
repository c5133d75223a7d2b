// Host planner: macrogrid hierarchy, windows and parents.
//
// Vertex layout (default, reading R1): x_p = H k, k in {0..M}^d.
//  T_n = {k : k_i = 0 mod eta^(L-n)}                    (readings R1/R7)
// Block layout (NEXT-1, the paper's Figures 2-3): x_p = (k + 1/2) H,
//  k in {0..M-1}^d, T_n = {k : k_i = r_n mod eta^(L-n)}; each coarse block of size eta^(L-n) H
//  keeps the T_{n+1} block closest to its centre (ties: the smaller index), r_L = 0.
// Both:
//  S_1 = T_1, S_n = T_n \ T_{n-1}                       (Eq. 10)
//  R_p^+ = x_p +- (l+1/2)H clipped, K_p = x_p +- H/2    (reading R2)
//  parents of p in S_n: the T_{n-1} lattice points bracketing x_p per coordinate, d-linear
//  weights (one-sided: the single point, weight 1), sum c_t = 1 (Eq. 11, PAPER.md:379-389;
//  reading R10); a parent whose window does not cover the child's window after the local
//  shift is dropped per coordinate and its weight moved to the opposite parent (reading R9).
//  interp = 1 (NEXT-1): the single nearest S_1 point whose window covers the
//  child's, weight 1 (ties: the smaller coordinate).
#include "plan.h"

#include <cstdio>
#include <cstdlib>

static int64_t ipow(int64_t b, int e) {
  int64_t r = 1;
  while (e-- > 0) r *= b;
  return r;
}

int HostPlan::level_of(const int* k) const {
  for (int lev = 1; lev <= L; lev++) {
    const int64_t s = ipow(eta, L - lev);
    bool on = true;
    for (int i = 0; i < D; i++) on = on && (k[i] % s == r[lev]);
    if (on) return lev;
  }
  return L;
}

// 2 x fine-cell coordinate of x_p along one dimension
int64_t HostPlan::origin2(int k) const { return 2 * (int64_t)k * c + (layout == 1 ? c : 0); }

// NEXT-4: with interp 2 a child is assigned to its nearest S_1 point, at most
// eta^(L-1) H / 2 away per coordinate, and the level-1 windows are enlarged by that much so they
// contain the windows of all their children (no extrapolation of phi_t is needed)
int HostPlan::lwin(int level) const { return (interp == 2 && level == 1) ? l + (int)(ipow(eta, L - 1) / 2) : l; }

void HostPlan::window(const int* k, int* lo, int* hi) const {
  const int64_t w2 = (2 * lwin(level_of(k)) + 1) * c;
  for (int i = 0; i < 3; i++) {
    if (i >= D) { lo[i] = 0; hi[i] = 1; continue; }
    const int64_t a = (origin2(k[i]) - w2) / 2, b = (origin2(k[i]) + w2) / 2;
    lo[i] = (int)(a < 0 ? 0 : a);
    hi[i] = (int)(b > n ? n : b);
  }
}

bool HostPlan::covers(int t, int k) const {
  const int64_t w2 = (2 * l + 1) * c;
  auto rng = [&](int v, int64_t& a, int64_t& b) {
    const int64_t o = origin2(v);
    a = o - w2;
    b = o + w2;
    if (a < 0) a = 0;
    if (b > 2 * n) b = 2 * n;
    a -= o;
    b -= o;
  };
  int64_t ak, bk, at, bt;
  rng(k, ak, bk);
  rng(t, at, bt);
  return at <= ak && bt >= bk;
}

// lattice points of T_lev bracketing coordinate k: returns count (1 or 2), points, weights
int HostPlan::bracket(int k, int lev, int* t, double* w) const {
  const int64_t s = ipow(eta, L - lev);
  const int64_t rr = r[lev];
  if (k % s == rr) {
    t[0] = k;
    w[0] = 1.0;
    return 1;
  }
  const int64_t a = k - ((k - rr) % s + s) % s, b = a + s;
  const bool ha = a >= 0, hb = b < mv;
  if (ha && hb) {
    const double wb = (double)(k - a) / (double)s;
    t[0] = (int)a; w[0] = 1.0 - wb;
    t[1] = (int)b; w[1] = wb;
    return 2;
  }
  t[0] = (int)(ha ? a : b);
  w[0] = 1.0;
  return 1;
}

int HostPlan::build(std::string& err) {
  if (n % M) { err = "M must divide n"; return -2; }
  c = n / M;
  const int64_t eL = ipow(eta, L - 1);
  // both layouts: the coarsest level mesh has >= 2 elements across every subcell
  if (c % 2) { err = "H/(2h) must be an integer"; return -2; }
  if ((c / 2) % eL) { err = "H/(2 h eta^(L-1)) must be an integer"; return -2; }
  if (M % eL) { err = "eta^(L-1) must divide M"; return -2; }
  mv = (layout == 0) ? M + 1 : M;
  r.assign(L + 1, 0);
  if (layout == 1) {
    for (int lev = L - 1; lev >= 1; lev--) {
      const int64_t s = ipow(eta, L - lev), s1 = ipow(eta, L - lev - 1);
      int64_t best = r[lev + 1];
      double bd = 1e300;
      for (int j = 0; j < eta; j++) {  // closest to the coarse centre s/2, ties: smaller j
        const int64_t v = r[lev + 1] + j * s1;
        const double dd = (v + 0.5 > 0.5 * s) ? (v + 0.5 - 0.5 * s) : (0.5 * s - v - 0.5);
        if (dd < bd) { bd = dd; best = v; }
      }
      r[lev] = best;
    }
  }
  int64_t total = 1;
  for (int i = 0; i < D; i++) total *= mv;
  all.assign(total, MacroHost());
  S.assign(L + 1, {});
  for (int64_t lin = 0; lin < total; lin++) {
    MacroHost& m = all[lin];
    int64_t rem = lin;
    for (int i = 0; i < 3; i++) {
      if (i < D) { m.k[i] = (int)(rem % mv); rem /= mv; } else m.k[i] = 0;
    }
    m.lin = lin;
    m.level = level_of(m.k);
    window(m.k, m.lo, m.hi);
    S[m.level].push_back(lin);
  }
  // parents
  for (int64_t lin = 0; lin < total; lin++) {
    MacroHost& m = all[lin];
    m.npar = 0;
    if (m.level == 1) continue;
    const int plev = (interp >= 1) ? 1 : m.level - 1;
    int cand[3][2], ncand[3];
    double wc[3][2];
    for (int i = 0; i < D; i++) {
      int t[2];
      double w[2];
      const int nb = bracket(m.k[i], plev, t, w);
      int nk = 0;
      bool keep[2] = {false, false};
      for (int j = 0; j < nb; j++) keep[j] = (interp == 2) ? true : covers(t[j], m.k[i]);
      if (interp >= 1) {  // nearest covering point, ties: the smaller coordinate (t[0] < t[1])
        int best = -1;
        for (int j = 0; j < nb; j++)
          if (keep[j] && (best < 0 || std::abs(t[j] - m.k[i]) < std::abs(t[best] - m.k[i]))) best = j;
        if (best >= 0) { cand[i][0] = t[best]; wc[i][0] = 1.0; nk = 1; }
      } else {
        for (int j = 0; j < nb; j++)
          if (keep[j]) { cand[i][nk] = t[j]; wc[i][nk] = (keep[0] && (nb == 1 || keep[1])) ? w[j] : 1.0; nk++; }
      }
      if (nk == 0) {
        char buf[160];
        snprintf(buf, sizeof buf, "no covering parent for macropoint (%d,%d,%d)", m.k[0], m.k[1], m.k[2]);
        err = buf;
        return -8;
      }
      ncand[i] = nk;
    }
    for (int i = D; i < 3; i++) { cand[i][0] = 0; wc[i][0] = 1.0; ncand[i] = 1; }
    if (interp == 2) {  // the enlarged parent window must contain the child's (physical coordinates)
      int t3[3] = {cand[0][0], cand[1][0], cand[2][0]}, plo[3], phi[3];
      window(t3, plo, phi);
      for (int i = 0; i < D; i++)
        if (plo[i] > m.lo[i] || phi[i] < m.hi[i]) {
          char buf[160];
          snprintf(buf, sizeof buf, "parent window does not contain macropoint (%d,%d,%d)", m.k[0], m.k[1], m.k[2]);
          err = buf;
          return -8;
        }
    }
    for (int cz = 0; cz < ncand[2]; cz++)
      for (int cy = 0; cy < ncand[1]; cy++)
        for (int cx = 0; cx < ncand[0]; cx++) {
          const int t[3] = {cand[0][cx], cand[1][cy], cand[2][cz]};
          int64_t tl = 0;
          for (int i = D - 1; i >= 0; i--) tl = tl * mv + t[i];
          m.par_lin[m.npar] = tl;
          m.par_w[m.npar] = wc[0][cx] * wc[1][cy] * wc[2][cz];
          m.npar++;
        }
  }
  return 0;
}
