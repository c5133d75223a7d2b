// Helpers shared by the 3D PCG kernels (pcg3d.cu, pcg3d_cl.cu): warp sums, subcell slots and the
// per-node element sides of a window dimension.
#pragma once
#include "device_common.cuh"

namespace pcg3d {

__device__ __forceinline__ double wsum0(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(FULLMASK, v, o);
  return __shfl_sync(FULLMASK, v, 0);
}

// subcell slot of the cell e of a grid of cell size s (in fine cells) along one dimension
__device__ __forceinline__ int slot3(const LevelArgs& A, const ProbDesc& P, int dim, int e, int s) {
  return fdiv(P.lo[dim] + e * s + A.coff, A.inv_c) - P.k[dim] + A.l;
}
__device__ __forceinline__ int slot3(const LevelArgs& A, const ProbDesc& P, int dim, int e) {
  return slot3(A, P, dim, e, A.s);
}

// The elements on the two sides of a node along one dimension (side 0: cell X-1, side 1: cell X)
// are grouped by subcell: pm = 3 if both exist in different subcells (keys k0, k1); pm = 1 if
// they share a subcell or only the lower one exists (all weight stored on side 0, key k0);
// pm = 2 if only the upper one exists (side 1, key k1).
struct Sides {
  int pm, k0, k1;
};
__device__ __forceinline__ Sides sides_of(const LevelArgs& A, const ProbDesc& P, int dim, int X, int ncd,
                                          int cs) {
  Sides s;
  const bool lo = X >= 1, up = X < ncd;
  const int sl = lo ? slot3(A, P, dim, X - 1, cs) : -1, su = up ? slot3(A, P, dim, X, cs) : -1;
  if (lo && up && sl != su) {
    s.pm = 3; s.k0 = sl; s.k1 = su;
  } else if (lo) {
    s.pm = 1; s.k0 = sl; s.k1 = sl;
  } else {
    s.pm = 2; s.k0 = su; s.k1 = su;
  }
  return s;
}
__device__ __forceinline__ Sides sides_of(const LevelArgs& A, const ProbDesc& P, int dim, int X, int ncd) {
  return sides_of(A, P, dim, X, ncd, A.s);
}

}  // namespace pcg3d
using namespace pcg3d;
