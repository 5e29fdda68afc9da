// The moment sums of compute_moments (kernels.hpp:74-107) over q gathered
// populations, in two bit-identical forms.
//
// Reference form: ten double accumulators seeded with +0, each population
// added or subtracted in direction order -- 91 additions for D3Q19.
//
// Pair form (fp32 storage, double accumulation only): if every value is
// exact on one common grid and every partial sum fits 53 bits, all those
// additions are EXACT, so the sums equal the exact linear combinations and
// may be formed in any order. With s_a = f_a + f_opp and d_a = f_a - f_opp
// per opposite pair:
//   j_k  = sum over pairs (c_k(a) d_a),   P_kk = sum over pairs with c_k != 0 of s_a,
//   P_kl = sum over pairs (c_k c_l s_a),  rho  = f_0 + P_xx + sum over pairs with c_x == 0 of s_a
// -- 50 additions for D3Q19 (27 fewer ops than the reference's 77 seed-free
// ones, 41 fewer than its 91).
//
// Exactness condition (checked per node, on the fp32 values): M < m * 2^24,
// M = max |f_a|, m = min |f_a|. Every fp32 value x is a multiple of
// 2^(floor(log2 m) - 23) (normal x >= m by its own exponent; subnormals by
// 2^-149), and every partial sum is bounded by sum |f_a| <= q M < 2^(emax+6)
// with emax <= floor(log2 m) + 24, i.e. it needs at most 53 bits. Zeros
// (m = 0), infinities (M = inf) and NaNs (max.NaN propagates) fail the
// check and take the reference form. Signed zeros agree: with no zero
// operand, a zero partial sum only arises as x + (-x) = +0 in either form,
// and no -0 can ever be produced. Over LB populations (f_a ~ t_a rho) the
// check passes everywhere; the reference form remains the fallback.
#pragma once

#include <type_traits>

#include "tslb_collision.cuh"
#include "tslb_domain.cuh"
#include "tslb_lattice.cuh"

namespace tslb_cuda {

template <typename C>
struct MSums {
  C r, jx, jy, jz, pxx, pyy, pzz, pxy, pxz, pyz;
};

/// compute_moments' accumulation order (kernels.hpp:74-107)
template <class L, typename T, typename C>
__device__ __forceinline__ MSums<C> msums_reference(const T (&v)[L::q]) {
  MSums<C> s{0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  unroll<L::q>([&](auto A) {
    constexpr int a = decltype(A)::value;
    using dd = Dir<L, a>;
    const C fa = C(v[a]);
    s.r += fa;
    if constexpr (dd::x == 1) s.jx += fa;
    if constexpr (dd::x == -1) s.jx -= fa;
    if constexpr (dd::y == 1) s.jy += fa;
    if constexpr (dd::y == -1) s.jy -= fa;
    if constexpr (dd::z == 1) s.jz += fa;
    if constexpr (dd::z == -1) s.jz -= fa;
    if constexpr (dd::x != 0) s.pxx += fa;
    if constexpr (dd::y != 0) s.pyy += fa;
    if constexpr (dd::z != 0) s.pzz += fa;
    if constexpr (dd::x * dd::y == 1) s.pxy += fa;
    if constexpr (dd::x * dd::y == -1) s.pxy -= fa;
    if constexpr (dd::x * dd::z == 1) s.pxz += fa;
    if constexpr (dd::x * dd::z == -1) s.pxz -= fa;
    if constexpr (dd::y * dd::z == 1) s.pyz += fa;
    if constexpr (dd::y * dd::z == -1) s.pyz -= fa;
  });
  return s;
}

namespace msums_detail {
// acc (+|-)= v, the first term initialises (no seed)
template <int SIGN, typename C>
__device__ __forceinline__ void acc(C& a, bool& first, C v) {
  if (first) {
    a = SIGN > 0 ? v : -v;
    first = false;
  } else {
    a = SIGN > 0 ? a + v : a - v;
  }
}
}  // namespace msums_detail

/// Incremental moment sums, one opposite pair at a time (step<0> takes the
/// rest population, step<a> for odd a the pair (a, a + 1)), so a kernel can
/// spread the reduction of one plane over the collision of another. PAIRS:
/// the pair form (exact only under the range condition); else the reference
/// order -- which visits the directions in the same ascending order, so
/// consuming pairs in order reproduces msums_reference exactly.
template <class L, typename T, typename C, bool PAIRS>
struct MAcc {
  MSums<C> s{0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  bool fr = false, fjx = true, fjy = true, fjz = true, fxx = true, fyy = true, fzz = true, fxy = true,
       fxz = true, fyz = true;

  template <int A>
  __device__ __forceinline__ void ref1(C fa) {
    using dd = Dir<L, A>;
    s.r += fa;
    if constexpr (dd::x == 1) s.jx += fa;
    if constexpr (dd::x == -1) s.jx -= fa;
    if constexpr (dd::y == 1) s.jy += fa;
    if constexpr (dd::y == -1) s.jy -= fa;
    if constexpr (dd::z == 1) s.jz += fa;
    if constexpr (dd::z == -1) s.jz -= fa;
    if constexpr (dd::x != 0) s.pxx += fa;
    if constexpr (dd::y != 0) s.pyy += fa;
    if constexpr (dd::z != 0) s.pzz += fa;
    if constexpr (dd::x * dd::y == 1) s.pxy += fa;
    if constexpr (dd::x * dd::y == -1) s.pxy -= fa;
    if constexpr (dd::x * dd::z == 1) s.pxz += fa;
    if constexpr (dd::x * dd::z == -1) s.pxz -= fa;
    if constexpr (dd::y * dd::z == 1) s.pyz += fa;
    if constexpr (dd::y * dd::z == -1) s.pyz -= fa;
  }

  template <int A>
  __device__ __forceinline__ void step(const T (&v)[L::q]) {
    using msums_detail::acc;
    if constexpr (A == 0) {
      if constexpr (PAIRS) s.r = C(v[0]);
      else ref1<0>(C(v[0]));
    } else if constexpr (!PAIRS) {
      ref1<A>(C(v[A]));
      ref1<A + 1>(C(v[A + 1]));
    } else {
      using dd = Dir<L, A>;
      const C fa = C(v[A]), fb = C(v[A + 1]);
      const C sp = fa + fb, dm = fa - fb;
      if constexpr (dd::x != 0) {
        acc<dd::x>(s.jx, fjx, dm);
        acc<1>(s.pxx, fxx, sp);
      } else {
        acc<1>(s.r, fr, sp);
      }
      if constexpr (dd::y != 0) {
        acc<dd::y>(s.jy, fjy, dm);
        acc<1>(s.pyy, fyy, sp);
      }
      if constexpr (dd::z != 0) {
        acc<dd::z>(s.jz, fjz, dm);
        acc<1>(s.pzz, fzz, sp);
      }
      if constexpr (dd::x * dd::y != 0) acc<dd::x * dd::y>(s.pxy, fxy, sp);
      if constexpr (dd::x * dd::z != 0) acc<dd::x * dd::z>(s.pxz, fxz, sp);
      if constexpr (dd::y * dd::z != 0) acc<dd::y * dd::z>(s.pyz, fyz, sp);
    }
  }

  __device__ __forceinline__ void all(const T (&v)[L::q]) {
    unroll<L::q>([&](auto A) {
      constexpr int a = decltype(A)::value;
      if constexpr (a == 0 || (a & 1)) step<a>(v);
    });
  }

  __device__ __forceinline__ MSums<C> finish() {
    if constexpr (PAIRS) {
      s.r = s.r + s.pxx;
      if (fjz) s.jz = s.pzz = s.pxz = s.pyz = C(0);  // (2-D lattices: never read)
      if (fxy) s.pxy = C(0);
    }
    return s;
  }
};

/// the pair form (exact only under the range condition, see header)
template <class L, typename T, typename C>
__device__ __forceinline__ MSums<C> msums_pairs(const T (&v)[L::q]) {
  MAcc<L, T, C, true> a;
  a.all(v);
  return a.finish();
}

/// the pair form is used (fp32 storage, double accumulation) unless a node
/// fails the range check
template <typename T, typename C>
__host__ __device__ constexpr bool msums_pair_form() {
#ifdef TSLB_MSUMS_REF  // (measurement switch: the reference form only)
  return false;
#else
  return std::is_same_v<T, float> && std::is_same_v<C, double>;
#endif
}

/// M < m * 2^24 over |v| (false for zeros, infinities, NaNs): three-input
/// |.| min / max (FMNMX3) as a tree of depth 3 for q <= 27; .NaN makes a NaN
/// win the max
namespace msums_detail {
__device__ __forceinline__ float amax3(float a, float b, float c) {
  float r;
  asm("max.NaN.abs.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ float amin3(float a, float b, float c) {
  float r;
  asm("min.abs.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
// reduce N values level by level, three at a time: ceil((N - 1) / 2)
// FMNMX3 in depth ceil(log3 N) (19 -> 7 -> 3 -> 1: 9 instructions)
template <int N, bool MAX>
__device__ __forceinline__ float red3(const float* v) {
  if constexpr (N == 1) {
    return MAX ? amax3(v[0], v[0], v[0]) : amin3(v[0], v[0], v[0]);
  } else {
    constexpr int M = (N + 2) / 3;  // values after this level
    float w[M];
#pragma unroll
    for (int g = 0; g < M; ++g) {
      const int a = 3 * g, b = min(3 * g + 1, N - 1), c = min(3 * g + 2, N - 1);
      if (3 * g + 1 >= N) w[g] = v[a];  // a lone leftover moves up unchanged
      else w[g] = MAX ? amax3(v[a], v[b], v[c]) : amin3(v[a], v[b], v[c]);
    }
    if constexpr (M == 1) return w[0];
    else return red3<M, MAX>(w);
  }
}
}  // namespace msums_detail

template <int Q>
__device__ __forceinline__ bool msums_exact(const float (&v)[Q]) {
  const float mx = msums_detail::red3<Q, true>(v);
  const float mn = msums_detail::red3<Q, false>(v);
  return mx < mn * 16777216.0f;
}

/// (fp64 storage: the pair form never applies)
template <int Q>
__device__ __forceinline__ bool msums_exact(const double (&)[Q]) {
  return false;
}

/// compute_moments' sums, bit-identical to msums_reference; fp32 storage
/// with double accumulation takes the pair form when it is exact. fp32 node
/// arithmetic (the tolerance mode) always takes the pair form in 3-D (every
/// 3-D kernel computes the moments here, so the schedules agree bit for bit).
template <class L, typename T, typename C>
__device__ __forceinline__ MSums<C> msums(const T (&v)[L::q]) {
  if constexpr (std::is_same_v<C, float> && L::dim == 3) return msums_pairs<L, T, C>(v);
  if constexpr (msums_pair_form<T, C>()) {
    // (check first: computing the pair sums speculatively and redoing them
    // on failure measured slower, 33.1 vs 33.9 GLUPS -- more registers)
    if (msums_exact<L::q>(v)) return msums_pairs<L, T, C>(v);
  }
  return msums_reference<L, T, C>(v);
}

/// compute_moments' finishing arithmetic (kernels.hpp:96-106): the body
/// force shift, then rho, j and Pi^neq = P - cs2 rho I - j j rounded to T.
/// fp32 node arithmetic in 3-D fuses the products (tolerance mode, as msums).
template <class L, typename T, typename C, class Put>
__device__ __forceinline__ void moment_tail(const Dom& d, MSums<C> s, const Put& put) {
  if constexpr (L::dim == 3) force_shift<C>(d, s.jx, s.jy, s.jz);
  else { C z0 = 0; force_shift<C>(d, s.jx, s.jy, z0); }
  const C c3 = cs2<C>();
  put(0, T(s.r));
  put(1, T(s.jx));
  put(2, T(s.jy));
  if constexpr (L::dim == 3) {
    put(3, T(s.jz));
    if constexpr (std::is_same_v<C, float>) {
      const float cr = fmaf(-c3, s.r, 0.0f);
      put(4, T(fmaf(-s.jx, s.jx, s.pxx + cr)));
      put(5, T(fmaf(-s.jy, s.jy, s.pyy + cr)));
      put(6, T(fmaf(-s.jz, s.jz, s.pzz + cr)));
      put(7, T(fmaf(-s.jx, s.jy, s.pxy)));
      put(8, T(fmaf(-s.jx, s.jz, s.pxz)));
      put(9, T(fmaf(-s.jy, s.jz, s.pyz)));
    } else {
      put(4, T(s.pxx - c3 * s.r - s.jx * s.jx));
      put(5, T(s.pyy - c3 * s.r - s.jy * s.jy));
      put(6, T(s.pzz - c3 * s.r - s.jz * s.jz));
      put(7, T(s.pxy - s.jx * s.jy));
      put(8, T(s.pxz - s.jx * s.jz));
      put(9, T(s.pyz - s.jy * s.jz));
    }
  } else {
    put(3, T(s.pxx - c3 * s.r - s.jx * s.jx));
    put(4, T(s.pyy - c3 * s.r - s.jy * s.jy));
    put(5, T(s.pxy - s.jx * s.jy));
  }
}

}  // namespace tslb_cuda
