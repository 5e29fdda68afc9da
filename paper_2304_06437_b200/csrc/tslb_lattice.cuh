// Compile-time velocity sets for the sm_100a kernels.
//
// Same ordering contract as the reference (lattice.hpp:17-22, 23-75): rest
// first, then axis vectors, then diagonals, the two members of every opposite
// pair adjacent (a, a^1 for a >= 1 when a is odd). D3Q27 is new (no reference
// code); its weights are the standard 8/27, 2/27, 1/54, 1/216 and it keeps the
// D3Q19 order for its first 19 directions.
//
// Everything here is constexpr so that, after the per-direction loops are
// unrolled with `unroll<q>`, every c_a component, weight and sign test folds
// into the instruction stream (the reference's for_each_dir, lattice.hpp:
// 252-257, does the same on the CPU).
#pragma once

#include <cstdint>
#include <utility>

namespace tslb_cuda {

enum LatticeId : int { kD2Q9 = 0, kD3Q19 = 1, kD3Q27 = 2 };

struct D2Q9 {
  static constexpr int id = kD2Q9, dim = 2, q = 9;
  static constexpr int c[q][3] = {{0, 0, 0},  {1, 0, 0},  {-1, 0, 0},
                                  {0, 1, 0},  {0, -1, 0}, {1, 1, 0},
                                  {-1, -1, 0}, {1, -1, 0}, {-1, 1, 0}};
  static constexpr long tw[q][2] = {{4, 9},  {1, 9},  {1, 9},  {1, 9}, {1, 9},
                                    {1, 36}, {1, 36}, {1, 36}, {1, 36}};
  static constexpr long bw[q][2] = {{-4, 27}, {2, 27},  {2, 27},
                                    {2, 27},  {2, 27},  {5, 108},
                                    {5, 108}, {5, 108}, {5, 108}};
};

struct D3Q19 {
  static constexpr int id = kD3Q19, dim = 3, q = 19;
  static constexpr int c[q][3] = {
      {0, 0, 0},   {1, 0, 0},  {-1, 0, 0}, {0, 1, 0},  {0, -1, 0},
      {0, 0, 1},   {0, 0, -1}, {1, 1, 0},  {-1, -1, 0}, {1, -1, 0},
      {-1, 1, 0},  {1, 0, 1},  {-1, 0, -1}, {1, 0, -1}, {-1, 0, 1},
      {0, 1, 1},   {0, -1, -1}, {0, 1, -1}, {0, -1, 1}};
  static constexpr long tw[q][2] = {
      {1, 3},  {1, 18}, {1, 18}, {1, 18}, {1, 18}, {1, 18}, {1, 18},
      {1, 36}, {1, 36}, {1, 36}, {1, 36}, {1, 36}, {1, 36}, {1, 36},
      {1, 36}, {1, 36}, {1, 36}, {1, 36}, {1, 36}};
  static constexpr long bw[q][2] = {
      {-1, 3}, {1, 18}, {1, 18}, {1, 18}, {1, 18}, {1, 18}, {1, 18},
      {1, 36}, {1, 36}, {1, 36}, {1, 36}, {1, 36}, {1, 36}, {1, 36},
      {1, 36}, {1, 36}, {1, 36}, {1, 36}, {1, 36}};
};

struct D3Q27 {
  static constexpr int id = kD3Q27, dim = 3, q = 27;
  static constexpr int c[q][3] = {
      {0, 0, 0},   {1, 0, 0},   {-1, 0, 0},  {0, 1, 0},   {0, -1, 0},
      {0, 0, 1},   {0, 0, -1},  {1, 1, 0},   {-1, -1, 0}, {1, -1, 0},
      {-1, 1, 0},  {1, 0, 1},   {-1, 0, -1}, {1, 0, -1},  {-1, 0, 1},
      {0, 1, 1},   {0, -1, -1}, {0, 1, -1},  {0, -1, 1},  {1, 1, 1},
      {-1, -1, -1}, {1, 1, -1}, {-1, -1, 1}, {1, -1, 1},  {-1, 1, -1},
      {-1, 1, 1},  {1, -1, -1}};
  static constexpr long tw[q][2] = {
      {8, 27},  {2, 27},  {2, 27},  {2, 27},  {2, 27},  {2, 27},  {2, 27},
      {1, 54},  {1, 54},  {1, 54},  {1, 54},  {1, 54},  {1, 54},  {1, 54},
      {1, 54},  {1, 54},  {1, 54},  {1, 54},  {1, 54},  {1, 216}, {1, 216},
      {1, 216}, {1, 216}, {1, 216}, {1, 216}, {1, 216}, {1, 216}};
  // Not in the reference: D3Q19's B on rest/axis/face diagonals, zero on the
  // corners; satisfies sum B = cs2, sum B c = 0, sum B cc = cs2 I.
  static constexpr long bw[q][2] = {
      {-1, 3}, {1, 18}, {1, 18}, {1, 18}, {1, 18}, {1, 18}, {1, 18},
      {1, 36}, {1, 36}, {1, 36}, {1, 36}, {1, 36}, {1, 36}, {1, 36},
      {1, 36}, {1, 36}, {1, 36}, {1, 36}, {1, 36}, {0, 1},  {0, 1},
      {0, 1},  {0, 1},  {0, 1},  {0, 1},  {0, 1},  {0, 1}};
};

/// Per-direction constants of lattice L, all compile-time.
template <class L, int A>
struct Dir {
  static constexpr int x = L::c[A][0], y = L::c[A][1], z = L::c[A][2];
  static constexpr int opp = (A == 0) ? 0 : ((A & 1) ? A + 1 : A - 1);
  static constexpr int norm2 = x * x + y * y + z * z;
  template <typename S>
  __host__ __device__ static constexpr S t() {
    return S(L::tw[A][0]) / S(L::tw[A][1]);
  }
  template <typename S>
  __host__ __device__ static constexpr S b() {
    return S(L::bw[A][0]) / S(L::bw[A][1]);
  }
};

/// Compile-time loop: f(std::integral_constant<int, A>) for A = 0..N-1.
template <class F, int... A>
__host__ __device__ __forceinline__ void unroll_impl(
    F&& f, std::integer_sequence<int, A...>) {
  (f(std::integral_constant<int, A>{}), ...);
}
template <int N, class F>
__host__ __device__ __forceinline__ void unroll(F&& f) {
  unroll_impl(f, std::make_integer_sequence<int, N>{});
}

/// c_a . v with the sign folding of the reference's dot_c
/// (collision.hpp:49-59): start from zero, add or subtract per component.
template <int CX, int CY, int CZ, typename S>
__host__ __device__ __forceinline__ S dot_c(S x, S y, S z) {
  S s = S(0);
  if constexpr (CX == 1) s += x;
  if constexpr (CX == -1) s -= x;
  if constexpr (CY == 1) s += y;
  if constexpr (CY == -1) s -= y;
  if constexpr (CZ == 1) s += z;
  if constexpr (CZ == -1) s -= z;
  return s;
}

}  // namespace tslb_cuda
