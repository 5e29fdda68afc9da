// Register-resident node algebra of the regularised (Hermite-projected)
// collision, shared by every kernel.
//
// Bit-parity contract: each expression keeps the reference's operand order
// and parenthesisation (collision.hpp:63-127), and the whole library is
// compiled with --fmad=false so no multiply-add is contracted. Instantiated
// with S = double for the single-fluid path (the reference always does
// node-local single-fluid arithmetic in double, kernels.hpp:38-42) and with
// S = T for the two-fluid path (multicomponent.hpp:334-378).
#pragma once

#include "tslb_lattice.cuh"

namespace tslb_cuda {

template <typename S>
struct NodeMoments {
  S rho, ux, uy, uz, usq15, pxx, pyy, pzz, pxy2, pxz2, pyz2, trcs2;
};

template <typename S>
__host__ __device__ __forceinline__ S cs2() {
  return S(1) / S(3);
}

/// prepare_node (collision.hpp:72-89)
template <typename S>
__host__ __device__ __forceinline__ NodeMoments<S> prepare_node(
    S rho, S ux, S uy, S uz, S pxx, S pyy, S pzz, S pxy, S pxz, S pyz) {
  NodeMoments<S> m;
  m.rho = rho;
  m.ux = ux;
  m.uy = uy;
  m.uz = uz;
  m.usq15 = S(1.5) * (ux * ux + uy * uy + uz * uz);
  m.pxx = pxx;
  m.pyy = pyy;
  m.pzz = pzz;
  m.pxy2 = pxy + pxy;
  m.pxz2 = pxz + pxz;
  m.pyz2 = pyz + pyz;
  m.trcs2 = cs2<S>() * (pxx + pyy + pzz);
  return m;
}

/// equilibrium_dir (collision.hpp:93-99)
template <class L, int A, typename S>
__host__ __device__ __forceinline__ S equilibrium(const NodeMoments<S>& m) {
  using d = Dir<L, A>;
  constexpr S t = d::template t<S>();
  const S cu = dot_c<d::x, d::y, d::z>(m.ux, m.uy, m.uz);
  return t * (m.rho + S(3) * cu + S(4.5) * cu * cu - m.usq15);
}

/// regularized_dir (collision.hpp:104-119): (t/2cs^4) Q_a : Pi^neq with the
/// contraction reduced to sign picks of the stress components.
template <class L, int A, typename S>
__host__ __device__ __forceinline__ S regularized(const NodeMoments<S>& m) {
  using d = Dir<L, A>;
  constexpr S t = d::template t<S>();
  S s = S(0);
  if constexpr (d::x != 0) s += m.pxx;
  if constexpr (d::y != 0) s += m.pyy;
  if constexpr (d::z != 0) s += m.pzz;
  if constexpr (d::x * d::y == 1) s += m.pxy2;
  if constexpr (d::x * d::y == -1) s -= m.pxy2;
  if constexpr (d::x * d::z == 1) s += m.pxz2;
  if constexpr (d::x * d::z == -1) s -= m.pxz2;
  if constexpr (d::y * d::z == 1) s += m.pyz2;
  if constexpr (d::y * d::z == -1) s -= m.pyz2;
  constexpr S t45 = t * S(4.5);
  return t45 * (s - m.trcs2);
}

/// post_collision_dir (collision.hpp:123-127)
template <class L, int A, typename S>
__host__ __device__ __forceinline__ S post_collision(const NodeMoments<S>& m,
                                                    S om1) {
  return equilibrium<L, A, S>(m) + om1 * regularized<L, A, S>(m);
}

/// bounce_correction (kernels.hpp:129-134): 6 t_a (c_a . u_wall)
template <class L, int A, typename S>
__host__ __device__ __forceinline__ S bounce_correction(S wx, S wy, S wz) {
  using d = Dir<L, A>;
  constexpr S t = d::template t<S>();
  constexpr S t6 = S(6) * t;
  return t6 * dot_c<d::x, d::y, d::z>(wx, wy, wz);
}

}  // namespace tslb_cuda
