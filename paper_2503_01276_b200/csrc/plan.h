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
  int interp = 0;  // 0: d-linear on T_{n-1} (R10); 1: nearest covering S_1 point, weight 1
  int64_t n = 0, M = 0, c = 0;
  std::vector<MacroHost> all;             // by lexicographic index
  std::vector<std::vector<int64_t>> S;    // S[level] = indices, lexicographic
  int build(std::string& err);
  int level_of(const int* k) const;
  void window(const int* k, int* lo, int* hi) const;
  bool covers(int t, int k) const;
};
