#pragma once
#include <cstdint>
#include <string>
#include <vector>

struct MacroHost {
  int k[3] = {0, 0, 0};
  int level = 1;
  int64_t lin = 0;
  int lo[3] = {0, 0, 0}, hi[3] = {1, 1, 1};  // window fine cells [lo, hi)
  int npar = 0;
  int64_t par_lin[8] = {0};
  double par_w[8] = {0};
};

struct HostPlan {
  int D = 2, L = 1, eta = 2, l = 1;
  int interp = 0;  // 0: d-linear on T_{n-1} (R10); 1: nearest covering S_1 point, weight 1;
                   // 2: nearest S_1 point in physical coordinates, enlarged level-1 windows (NEXT-4)
  int layout = 0;  // 0: vertex-centred (R1); 1: block-centred (paper Figs. 2-3)
  int64_t n = 0, M = 0, c = 0;
  int64_t mv = 0;          // macropoints per dimension: M+1 (vertex) or M (block)
  std::vector<int64_t> r;  // r[lev]: T_lev = {k : k_i = r[lev] mod eta^(L-lev)}
  std::vector<MacroHost> all;             // by lexicographic index
  std::vector<std::vector<int64_t>> S;    // S[level] = indices, lexicographic
  int build(std::string& err);
  int level_of(const int* k) const;
  void window(const int* k, int* lo, int* hi) const;
  int lwin(int level) const;  // oversampling layers of a level's windows (l; level 1 of interp 2: l + eta^(L-1)/2)
  bool covers(int t, int k) const;
  int64_t origin2(int k) const;
  int bracket(int k, int lev, int* t, double* w) const;
  int64_t coff() const { return layout == 0 ? c / 2 : 0; }  // subcell of fine cell f: (f + coff) / c
};
