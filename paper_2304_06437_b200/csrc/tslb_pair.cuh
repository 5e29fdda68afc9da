// Shared device helpers of the box-geometry stream-collide kernels:
// vector moves, and the opposite-pair / seed-free forms of the collision
// (exact rewrites, see tslb_streamcoll_vec.cu header for the argument).
#pragma once

#include <type_traits>

#include "tslb_collision.cuh"
#include "tslb_domain.cuh"

namespace tslb_cuda {

// VX consecutive scalars moved as one aligned access of VX * sizeof(T) bytes
template <typename T, int VX>
struct alignas(sizeof(T) * VX) Pack {
  T v[VX];
};

template <typename T, int VX>
struct Vec {
  __device__ static void load(const T* p, T (&o)[VX]) {
    const Pack<T, VX> pk = *reinterpret_cast<const Pack<T, VX>*>(p);
#pragma unroll
    for (int e = 0; e < VX; ++e) o[e] = pk.v[e];
  }
  __device__ static void st(T* p, const T (&v)[VX]) {
    Pack<T, VX> pk;
#pragma unroll
    for (int e = 0; e < VX; ++e) pk.v[e] = v[e];
    *reinterpret_cast<Pack<T, VX>*>(p) = pk;
  }
};


// c . u without the +0 seed (sign of a zero result may differ; see header)
template <int CX, int CY, int CZ, typename C>
__device__ __forceinline__ C dot_noseed(C x, C y, C z) {
  C s;
  bool first = true;
  auto add = [&](int c, C v) {
    if (c == 0) return;
    if (first) {
      s = c > 0 ? v : -v;
      first = false;
    } else {
      s = c > 0 ? s + v : s - v;
    }
  };
  add(CX, x);
  add(CY, y);
  add(CZ, z);
  return s;
}

template <class L, typename C>
__device__ __forceinline__ C post_rest(const NodeMoments<C>& m, C om1) {
  constexpr C t = Dir<L, 0>::template t<C>();
  // rho + 3*(+0) + (4.5*(+0))*(+0) == rho for rho != -0
  const C e = t * (m.rho - m.usq15);
  return e + om1 * regularized<L, 0, C>(m);
}

// regularized_dir and c . u without the +0 seeds of the reference's loops.
// Exactness: a seed only ever changes the SIGN OF A ZERO intermediate, and
// sign-of-zero differences survive +, -, * only as sign-of-zero differences.
// The regularised term r is finally added to the equilibrium part
// ea = t ((rho + 3cu + 4.5cu^2) - usq15), which is never -0.0 unless
// rho == -0.0 (x + y == -0 needs both operands -0 under round-to-nearest);
// so ea + r is bit-identical whether r is +0 or -0, and likewise
// rho + 3cu for cu = +-0. Callers guarantee rho != -0.0 (moments from a
// +0-seeded sum), see tslb_streamcoll_vec.cu / tslb_mstep.cu.
template <class L, int A, typename S>
__device__ __forceinline__ S regularized_noseed(const NodeMoments<S>& m) {
  using d = Dir<L, A>;
  constexpr S t45 = d::template t<S>() * S(4.5);
  S s;
  bool first = true;
  auto add = [&](bool on, int sign, S v) {
    if (!on) return;
    if (first) {
      s = sign > 0 ? v : -v;
      first = false;
    } else {
      s = sign > 0 ? s + v : s - v;
    }
  };
  add(d::x != 0, 1, m.pxx);
  add(d::y != 0, 1, m.pyy);
  add(d::z != 0, 1, m.pzz);
  add(d::x * d::y != 0, d::x * d::y, m.pxy2);
  add(d::x * d::z != 0, d::x * d::z, m.pxz2);
  add(d::y * d::z != 0, d::y * d::z, m.pyz2);
  if (first) s = S(0);
  return t45 * (s - m.trcs2);
}

// Post-collision values of the pair (A, A+1 = opp(A)), A odd: Q_a : Pi^neq
// is shared by a and opp(a), and c_opp . u = -(c_a . u) exactly.
template <class L, int A, typename C>
__device__ __forceinline__ void post_pair(const NodeMoments<C>& m, C om1,
                                          C& out_a, C& out_b) {
  using d = Dir<L, A>;
  constexpr C t = d::template t<C>();
  const C cu = dot_noseed<d::x, d::y, d::z, C>(m.ux, m.uy, m.uz);
  const C c3 = C(3) * cu;
  const C q = C(4.5) * cu * cu;
  const C ea = t * (m.rho + c3 + q - m.usq15);
  const C eb = t * (m.rho - c3 + q - m.usq15);
  const C r = om1 * regularized_noseed<L, A, C>(m);
  out_a = ea + r;
  out_b = eb + r;
}

// One direction, seed-free (same exactness argument)
template <class L, int A, typename C>
__device__ __forceinline__ C post_single(const NodeMoments<C>& m, C om1) {
  using d = Dir<L, A>;
  constexpr C t = d::template t<C>();
  const C cu = dot_noseed<d::x, d::y, d::z, C>(m.ux, m.uy, m.uz);
  const C e = t * (m.rho + C(3) * cu + C(4.5) * cu * cu - m.usq15);
  return e + om1 * regularized_noseed<L, A, C>(m);
}

// ---------------------------------------------------------------------------
// fp32 node arithmetic (the opt-in tolerance mode): the same
// regularised collision in fused multiply-adds with the node constants
// folded -- f_a = t (rho - 1.5 u^2) + 3t c.u + 4.5t (c.u)^2
// + (1 - omega) 4.5t (Q_a : Pi^neq - cs2 tr Pi). Every single-fluid kernel
// takes these forms when C = float (mstep, mstep2d, F1 vector / scalar,
// collide, ghost push), so the schedules agree bit for bit with each other;
// the reference parity of fp64 node math and the two-fluid kernels (which
// compute in T as the reference does) never go through them.
template <class L, int A>
__device__ __forceinline__ float reg_arg(const NodeMoments<float>& m) {
  using d = Dir<L, A>;
  float s = 0.0f;
  bool first = true;
  auto add = [&](bool on, int sign, float v) {
    if (!on) return;
    if (first) {
      s = sign > 0 ? v : -v;
      first = false;
    } else {
      s = sign > 0 ? s + v : s - v;
    }
  };
  add(d::x != 0, 1, m.pxx);
  add(d::y != 0, 1, m.pyy);
  add(d::z != 0, 1, m.pzz);
  add(d::x * d::y != 0, d::x * d::y, m.pxy2);
  add(d::x * d::z != 0, d::x * d::z, m.pxz2);
  add(d::y * d::z != 0, d::y * d::z, m.pyz2);
  return first ? -m.trcs2 : s - m.trcs2;
}

template <class L, int A>
__device__ __forceinline__ float fast_post(const NodeMoments<float>& m, float om1) {
  using d = Dir<L, A>;
  constexpr float t = d::template t<float>();
  const float tbase = t * (m.rho - m.usq15);
  const float k = om1 * (4.5f * t);
  if constexpr (d::x == 0 && d::y == 0 && d::z == 0) return fmaf(k, reg_arg<L, A>(m), tbase);
  const float cu = dot_noseed<d::x, d::y, d::z, float>(m.ux, m.uy, m.uz);
  const float e = fmaf((4.5f * t) * cu, cu, fmaf(3.0f * t, cu, tbase));
  return fmaf(k, reg_arg<L, A>(m), e);
}

template <class L, int A>
__device__ __forceinline__ void fast_pair(const NodeMoments<float>& m, float om1, float& out_a, float& out_b) {
  using d = Dir<L, A>;
  constexpr float t = d::template t<float>();
  const float tbase = t * (m.rho - m.usq15);
  const float k = om1 * (4.5f * t);
  const float cu = dot_noseed<d::x, d::y, d::z, float>(m.ux, m.uy, m.uz);
  const float h = (4.5f * t) * cu;
  const float r = reg_arg<L, A>(m);
  out_a = fmaf(k, r, fmaf(h, cu, fmaf(3.0f * t, cu, tbase)));
  out_b = fmaf(k, r, fmaf(h, cu, fmaf(-3.0f * t, cu, tbase)));
}

// the single-fluid entry points: fp32 node math -> the fused forms, fp64 ->
// the exact rewrites above (post_rest / post_pair / post_single)
template <class L, int A, typename C>
__device__ __forceinline__ C sf_post(const NodeMoments<C>& m, C om1) {
  if constexpr (std::is_same_v<C, float>) return fast_post<L, A>(m, om1);
  else if constexpr (A == 0) return post_rest<L, C>(m, om1);
  else return post_single<L, A, C>(m, om1);
}
template <class L, int A, typename C>
__device__ __forceinline__ void sf_pair(const NodeMoments<C>& m, C om1, C& out_a, C& out_b) {
  if constexpr (std::is_same_v<C, float>) fast_pair<L, A>(m, om1, out_a, out_b);
  else post_pair<L, A, C>(m, om1, out_a, out_b);
}
// the reference-order single direction (post_collision) for fp64 node math;
// the fused form for fp32
template <class L, int A, typename C>
__device__ __forceinline__ C sf_post_ref(const NodeMoments<C>& m, C om1) {
  if constexpr (std::is_same_v<C, float>) return fast_post<L, A>(m, om1);
  else return post_collision<L, A, C>(m, om1);
}

// Bounce of direction A at node fi: f[opp][fi] = T(C(out) - 6 t (c.u_wall))
// with u_wall summed in T over the crossed wall faces in axis order.
template <class L, int A, typename T, typename C>
__device__ __forceinline__ T bounce_value(const Dom& d, T out, bool cross_x,
                                          bool cross_y, bool cross_z) {
  using dd = Dir<L, A>;
  T wx = T(0), wy = T(0), wz = T(0);
  auto add = [&](int face) {
    wx += T(d.uw[face][0]);
    wy += T(d.uw[face][1]);
    wz += T(d.uw[face][2]);
  };
  if (cross_x) add(dd::x > 0 ? XMax : XMin);
  if (cross_y) add(dd::y > 0 ? YMax : YMin);
  if (cross_z) add(dd::z > 0 ? ZMax : ZMin);
  return T(C(out) - bounce_correction<L, A, C>(C(wx), C(wy), C(wz)));
}

}  // namespace tslb_cuda
