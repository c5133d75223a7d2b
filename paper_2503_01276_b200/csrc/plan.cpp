// Host planner: vertex macrogrid hierarchy, windows and parents.
//
//  T_n = {k in {0..M}^d : k_i = 0 mod eta^(L-n)}       (readings R1/R7)
//  S_1 = T_1, S_n = T_n \ T_{n-1}                       (Eq. 10)
//  R_p^+ = x_p +- (l+1/2)H clipped, K_p = x_p +- H/2    (reading R2)
//  parents of p in S_n: corners of the T_{n-1} cell containing x_p, d-linear weights,
//  sum c_t = 1 (Eq. 11; reading R10); a parent whose window does not
//  cover the child's window after the local shift is dropped per coordinate and its
//  weight moved to the opposite parent (reading R9).
//  interp = 1 (NEXT-1): the single nearest S_1 point whose window covers the
//  child's, weight 1 (ties: the smaller coordinate).
#include "plan.h"

#include <cstdio>

static int64_t ipow(int64_t b, int e) {
  int64_t r = 1;
  while (e-- > 0) r *= b;
  return r;
}

int HostPlan::level_of(const int* k) const {
  for (int lev = 1; lev <= L; lev++) {
    const int64_t s = ipow(eta, L - lev);
    bool on = true;
    for (int i = 0; i < D; i++) on = on && (k[i] % s == 0);
    if (on) return lev;
  }
  return L;
}

void HostPlan::window(const int* k, int* lo, int* hi) const {
  const int64_t half = (2 * l + 1) * c / 2;
  for (int i = 0; i < 3; i++) {
    if (i >= D) { lo[i] = 0; hi[i] = 1; continue; }
    int64_t a = k[i] * c - half, b = k[i] * c + half;
    lo[i] = (int)(a < 0 ? 0 : a);
    hi[i] = (int)(b > n ? n : b);
  }
}

bool HostPlan::covers(int t, int k) const {
  const int64_t half = (2 * l + 1) * c / 2;
  auto rng = [&](int v, int64_t& a, int64_t& b) {
    a = v * c - half;
    b = v * c + half;
    if (a < 0) a = 0;
    if (b > n) b = n;
    a -= v * c;
    b -= v * c;
  };
  int64_t ak, bk, at, bt;
  rng(k, ak, bk);
  rng(t, at, bt);
  return at <= ak && bt >= bk;
}

int HostPlan::build(std::string& err) {
  if (n % M) { err = "M must divide n"; return -2; }
  c = n / M;
  if (c % 2) { err = "H/(2h) must be an integer"; return -2; }
  const int64_t eL = ipow(eta, L - 1);
  if ((c / 2) % eL) { err = "H/(2 h eta^(L-1)) must be an integer"; return -2; }
  if (M % eL) { err = "eta^(L-1) must divide M"; return -2; }
  const int64_t V = M + 1;
  int64_t total = 1;
  for (int i = 0; i < D; i++) total *= V;
  all.assign(total, MacroHost());
  S.assign(L + 1, {});
  for (int64_t lin = 0; lin < total; lin++) {
    MacroHost& m = all[lin];
    int64_t r = lin;
    for (int i = 0; i < 3; i++) {
      if (i < D) { m.k[i] = (int)(r % V); r /= V; } else m.k[i] = 0;
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
    if (interp == 1) {  // nearest covering S_1 point per dimension (Euclidean distance is separable)
      const int64_t s1 = ipow(eta, L - 1);
      int t[3] = {0, 0, 0};
      for (int i = 0; i < D; i++) {
        const int ki = m.k[i];
        const int a = (int)((ki / s1) * s1), b = (int)(a + s1);
        const bool ca = covers(a, ki), cb = (ki != a) && covers(b, ki);
        if (!ca && !cb) {
          char buf[160];
          snprintf(buf, sizeof buf, "no covering parent for macropoint (%d,%d,%d)", m.k[0], m.k[1], m.k[2]);
          err = buf;
          return -8;
        }
        t[i] = (ca && (!cb || ki - a <= b - ki)) ? a : b;  // tie: the smaller coordinate
      }
      int64_t tl = 0;
      for (int i = D - 1; i >= 0; i--) tl = tl * V + t[i];
      m.par_lin[0] = tl;
      m.par_w[0] = 1.0;
      m.npar = 1;
      continue;
    }
    const int64_t s = ipow(eta, L - m.level + 1);
    int cand[3][2], ncand[3];
    double wc[3][2];
    for (int i = 0; i < D; i++) {
      const int ki = m.k[i];
      if (ki % s == 0) {
        cand[i][0] = ki; wc[i][0] = 1.0; ncand[i] = 1;
      } else {
        const int a = (int)((ki / s) * s), b = (int)(a + s);
        const double wb = (double)(ki - a) / (double)s;
        int nk = 0;
        const bool ca = covers(a, ki), cb = covers(b, ki);
        if (ca) { cand[i][nk] = a; wc[i][nk] = cb ? 1.0 - wb : 1.0; nk++; }
        if (cb) { cand[i][nk] = b; wc[i][nk] = ca ? wb : 1.0; nk++; }
        if (nk == 0) {
          char buf[160];
          snprintf(buf, sizeof buf, "no covering parent for macropoint (%d,%d,%d)", m.k[0], m.k[1], m.k[2]);
          err = buf;
          return -8;
        }
        ncand[i] = nk;
      }
    }
    for (int i = D; i < 3; i++) { cand[i][0] = 0; wc[i][0] = 1.0; ncand[i] = 1; }
    for (int cz = 0; cz < ncand[2]; cz++)
      for (int cy = 0; cy < ncand[1]; cy++)
        for (int cx = 0; cx < ncand[0]; cx++) {
          const int t[3] = {cand[0][cx], cand[1][cy], cand[2][cz]};
          int64_t tl = 0;
          for (int i = D - 1; i >= 0; i--) tl = tl * V + t[i];
          m.par_lin[m.npar] = tl;
          m.par_w[m.npar] = wc[0][cx] * wc[1][cy] * wc[2][cz];
          m.npar++;
        }
  }
  return 0;
}
