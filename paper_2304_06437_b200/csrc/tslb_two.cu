// Two-component colour-gradient kernels for sm_100a.
//
//   k_cg_moments     color_moments          multicomponent.hpp:55-119
//   k_cg_gradient    gradient_and_nci       multicomponent.hpp:154-242
//   k_cg_prepare     prepare_stress         multicomponent.hpp:271-309
//   k_cg_streamcoll  stream_collide_recolor multicomponent.hpp:315-401
//                    (optionally with prepare_stress folded into its
//                    prologue: the hot schedule is 3 kernels per step)
//
// All arithmetic in T, as in the reference; with --fmad=false and IEEE
// div/sqrt the results are bit-identical for float and double storage.
// NCI flags are set-only byte stores of the value 1 -- concurrent writers
// store the same byte, so the result is launch-shape independent, mirroring
// the reference's relaxed atomic_ref stores (multicomponent.hpp:233-236).
#include <cuda_pipeline.h>

#include <cstdint>

#include "tslb_collision.cuh"
#include "tslb_domain.cuh"
#include "tslb_kernels.h"
#include "tslb_pair.cuh"

namespace tslb_cuda {

#ifndef TSLB_BX2
#define TSLB_BX2 256
#endif
constexpr int BX2 = TSLB_BX2;  // threads per block = x nodes per block (-DTSLB_BX2: measurements)
// the domain as the row-tiled two-fluid launches see it (x blocks of BX2)
inline Dom dx2(const Dom& d) {
  Dom x = d;
  x.xblocks = (d.nx + BX2 - 1) / BX2;
  return x;
}

template <typename T>
struct TF {
  T *rho_r, *rho_b, *rho, *mom, *pin, *phi, *grad;
  uint8_t* flag;
};

// base pointer of every population array of both species (kernel
// parameters, read through the constant cache): a push then costs one
// 32-bit index and one wide multiply-add for its address instead of a
// running 64-bit pointer per species and direction
template <typename T>
struct PopBases {
  T* r[27];
  T* b[27];
};

template <typename T>
__host__ PopBases<T> pop_bases(T* fr, T* fb, const Dom& d, int q) {
  PopBases<T> p{};
  for (int a = 0; a < q; ++a) {
    p.r[a] = fr + int64_t(a) * d.fstride;
    p.b[a] = fb + int64_t(a) * d.fstride;
  }
  return p;
}

template <typename T>
__host__ TF<T> tf_of(const TwoFields& s) {
  return TF<T>{static_cast<T*>(s.rho_r), static_cast<T*>(s.rho_b),
               static_cast<T*>(s.rho),   static_cast<T*>(s.mom),
               static_cast<T*>(s.pin),   static_cast<T*>(s.phi),
               static_cast<T*>(s.grad),  s.flag};
}

// ---------------------------------------------------------------------------
template <class L, typename T>
__global__ void __launch_bounds__(BX2)
    k_cg_moments(Dom d, const T* __restrict__ fr, const T* __restrict__ fb,
                 TF<T> s, const uint8_t* __restrict__ solid) {
  int i, j, k;
  if (!node_coords<BX2>(d, i, j, k)) return;
  const int64_t fi = fidx(d, i, j, k);
  const int64_t mi = midx(d, i, j, k);
  s.flag[mi] = 0;
  if (solid[fi]) return;
  T rr = 0, rb = 0;
  T r = 0, jx = 0, jy = 0, jz = 0, pxx = 0, pyy = 0, pzz = 0, pxy = 0,
    pxz = 0, pyz = 0;
  unroll<L::q>([&](auto A) {
    constexpr int a = decltype(A)::value;
    using dd = Dir<L, a>;
    const T fra = __ldg(fr + a * d.fstride + fi);
    const T fba = __ldg(fb + a * d.fstride + fi);
    const T ga = fra + fba;
    rr += fra;
    rb += fba;
    r += ga;
    if constexpr (dd::x == 1) jx += ga;
    if constexpr (dd::x == -1) jx -= ga;
    if constexpr (dd::y == 1) jy += ga;
    if constexpr (dd::y == -1) jy -= ga;
    if constexpr (dd::z == 1) jz += ga;
    if constexpr (dd::z == -1) jz -= ga;
    if constexpr (dd::x != 0) pxx += ga;
    if constexpr (dd::y != 0) pyy += ga;
    if constexpr (dd::z != 0) pzz += ga;
    if constexpr (dd::x * dd::y == 1) pxy += ga;
    if constexpr (dd::x * dd::y == -1) pxy -= ga;
    if constexpr (dd::x * dd::z == 1) pxz += ga;
    if constexpr (dd::x * dd::z == -1) pxz -= ga;
    if constexpr (dd::y * dd::z == 1) pyz += ga;
    if constexpr (dd::y * dd::z == -1) pyz -= ga;
  });
  const int64_t ms = d.mstride;
  s.rho_r[mi] = rr;
  s.rho_b[mi] = rb;
  s.rho[mi] = r;
  s.phi[mi] = (rr - rb) / r;
  s.mom[mi] = jx;
  s.mom[ms + mi] = jy;
  if constexpr (L::dim == 3) {
    s.mom[2 * ms + mi] = jz;
    s.pin[mi] = pxx;
    s.pin[ms + mi] = pyy;
    s.pin[2 * ms + mi] = pzz;
    s.pin[3 * ms + mi] = pxy;
    s.pin[4 * ms + mi] = pxz;
    s.pin[5 * ms + mi] = pyz;
  } else {
    s.pin[mi] = pxx;
    s.pin[ms + mi] = pyy;
    s.pin[2 * ms + mi] = pxy;
  }
}

// ---------------------------------------------------------------------------
// Neighbour (pull) lookup with the reference's rule: wall or solid
// neighbours read phi(x) itself (multicomponent.hpp:178-186).
__device__ __forceinline__ bool nb_index(const Dom& d,
                                         const uint8_t* __restrict__ solid,
                                         int cx, int cy, int cz, int i, int j,
                                         int k, int64_t& mi_out) {
  int tc[3] = {i + cx, j + cy, k + cz};
  const int nd[3] = {d.nx, d.ny, d.nz};
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    if (tc[ax] < 0 || tc[ax] >= nd[ax]) {
      const int face = 2 * ax + (tc[ax] < 0 ? 0 : 1);
      if (d.mode[face] != kWrap) return false;
      tc[ax] = tc[ax] < 0 ? tc[ax] + nd[ax] : tc[ax] - nd[ax];
    }
  }
  if (solid[fidx(d, tc[0], tc[1], tc[2])]) return false;
  mi_out = midx(d, tc[0], tc[1], tc[2]);
  return true;
}

template <class L, typename T>
__global__ void __launch_bounds__(BX2)
    k_cg_gradient(Dom d, TF<T> s, const uint8_t* __restrict__ solid,
                  const uint32_t* __restrict__ slow, ColorParamsDev cp) {
  int i, j, k;
  if (!node_coords<BX2>(d, i, j, k)) return;
  const int64_t fi = fidx(d, i, j, k);
  const int64_t mi = midx(d, i, j, k);
  if (solid[fi]) return;
  const uint32_t sm = slow[mi];
  const T phi0 = s.phi[mi];
  T gx = 0, gy = 0, gz = 0;
  unroll<L::q>([&](auto A) {
    constexpr int a = decltype(A)::value;
    using dd = Dir<L, a>;
    if constexpr (a > 0) {
      T pn;
      if ((sm >> a) & 1u) {
        int64_t t;
        pn = nb_index(d, solid, dd::x, dd::y, dd::z, i, j, k, t) ? s.phi[t]
                                                                 : phi0;
      } else {
        const int64_t off = int64_t(dd::x) +
                            int64_t(d.nx) * (int64_t(dd::y) + int64_t(d.ny) * dd::z);
        pn = s.phi[mi + off];
      }
      constexpr T w = dd::template t<T>();
      const T tp = w * pn;
      if constexpr (dd::x == 1) gx += tp;
      if constexpr (dd::x == -1) gx -= tp;
      if constexpr (dd::y == 1) gy += tp;
      if constexpr (dd::y == -1) gy -= tp;
      if constexpr (dd::z == 1) gz += tp;
      if constexpr (dd::z == -1) gz -= tp;
    }
  });
  const int64_t ms = d.mstride;
  s.grad[mi] = T(3) * gx;
  s.grad[ms + mi] = T(3) * gy;
  if constexpr (L::dim == 3) s.grad[2 * ms + mi] = T(3) * gz;

  // near-contact scan (multicomponent.hpp:202-238), only when enabled
  const T bulk_cut = T(-1) + T(cp.eps_bulk);
  if (T(cp.nci_strength) != T(0) && phi0 < bulk_cut) {
    unroll<L::q>([&](auto A) {
      constexpr int a = decltype(A)::value;
      using dd = Dir<L, a>;
      if constexpr (a > 0 && dd::opp > a) {
        int64_t hit_p = 0, hit_m = 0;
        bool found_p = false, found_m = false;
        int ci = i, cj = j, ck = k;
        for (int st = 0; st < cp.nci_reach; ++st) {
          int64_t t;
          if (!nb_index(d, solid, dd::x, dd::y, dd::z, ci, cj, ck, t)) break;
          // advance (wrap) the probe position
          ci += dd::x; cj += dd::y; ck += dd::z;
          if (ci < 0) ci += d.nx; if (ci >= d.nx) ci -= d.nx;
          if (cj < 0) cj += d.ny; if (cj >= d.ny) cj -= d.ny;
          if (ck < 0) ck += d.nz; if (ck >= d.nz) ck -= d.nz;
          if (s.phi[t] >= bulk_cut) {
            hit_p = t;
            found_p = true;
            break;
          }
        }
        if (found_p) {
          ci = i; cj = j; ck = k;
          for (int st = 0; st < cp.nci_reach; ++st) {
            int64_t t;
            if (!nb_index(d, solid, -dd::x, -dd::y, -dd::z, ci, cj, ck, t)) break;
            ci -= dd::x; cj -= dd::y; ck -= dd::z;
            if (ci < 0) ci += d.nx; if (ci >= d.nx) ci -= d.nx;
            if (cj < 0) cj += d.ny; if (cj >= d.ny) cj -= d.ny;
            if (ck < 0) ck += d.nz; if (ck >= d.nz) ck -= d.nz;
            if (s.phi[t] >= bulk_cut) {
              hit_m = t;
              found_m = true;
              break;
            }
          }
          if (found_m) {
            s.flag[hit_p] = 1;
            s.flag[hit_m] = 1;
          }
        }
      }
    });
  }
}

// ---------------------------------------------------------------------------
// prepare_stress body (multicomponent.hpp:249-309) for one node; returns the
// shifted velocity and Pi^neq in registers.
template <class L, typename T>
__device__ __forceinline__ void prepare_node_stress(
    const Dom& d, const TF<T>& s, int64_t mi, T tau, const ColorParamsDev& cp,
    T& ux, T& uy, T& uz, T p[6]) {
  const int64_t ms = d.mstride;
  T F0 = 0, F1 = 0, F2 = 0;
  if (s.flag[mi]) {  // nci_force_at
    const T gx = s.grad[mi];
    const T gy = s.grad[ms + mi];
    const T gz = L::dim == 3 ? s.grad[2 * ms + mi] : T(0);
    const T gn = sqrt(gx * gx + gy * gy + gz * gz);
    if (!(gn <= T(cp.grad_threshold))) {
      const T scale = T(cp.nci_strength) * s.rho_r[mi] / gn;
      F0 = scale * gx;
      F1 = scale * gy;
      F2 = scale * gz;
    }
  }
  ux = s.mom[mi] + tau * F0;
  uy = s.mom[ms + mi] + tau * F1;
  uz = L::dim == 3 ? s.mom[2 * ms + mi] + tau * F2 : T(0);
  const T r = s.rho[mi];
  const T c3 = cs2<T>();
  if constexpr (L::dim == 3) {
    p[0] = s.pin[mi] + (-c3 * r - ux * ux);
    p[1] = s.pin[ms + mi] + (-c3 * r - uy * uy);
    p[2] = s.pin[2 * ms + mi] + (-c3 * r - uz * uz);
    p[3] = s.pin[3 * ms + mi] - ux * uy;
    p[4] = s.pin[4 * ms + mi] - ux * uz;
    p[5] = s.pin[5 * ms + mi] - uy * uz;
  } else {
    p[0] = s.pin[mi] + (-c3 * r - ux * ux);
    p[1] = s.pin[ms + mi] + (-c3 * r - uy * uy);
    p[2] = s.pin[2 * ms + mi] - ux * uy;
  }
}

template <class L, typename T>
__global__ void __launch_bounds__(BX2)
    k_cg_prepare(Dom d, TF<T> s, const uint8_t* __restrict__ solid, T tau,
                 ColorParamsDev cp) {
  int i, j, k;
  if (!node_coords<BX2>(d, i, j, k)) return;
  const int64_t mi = midx(d, i, j, k);
  if (solid[fidx(d, i, j, k)]) return;
  T ux, uy, uz, p[6];
  prepare_node_stress<L, T>(d, s, mi, tau, cp, ux, uy, uz, p);
  const int64_t ms = d.mstride;
  s.mom[mi] = ux;
  s.mom[ms + mi] = uy;
  if constexpr (L::dim == 3) s.mom[2 * ms + mi] = uz;
  constexpr int np = L::dim * (L::dim + 1) / 2;
#pragma unroll
  for (int c = 0; c < np; ++c) s.pin[c * ms + mi] = p[c];
}

// inv_cnorm (multicomponent.hpp:35-48), constants pre-rounded to T exactly as
// T(long double literal) does on the host.
template <typename T, int N2>
__device__ __forceinline__ T inv_cnorm() {
  if constexpr (N2 == 0) return T(0);
  if constexpr (N2 == 1) return T(1);
  if constexpr (N2 == 2) {
    if constexpr (sizeof(T) == 4) return __int_as_float(0x3f3504f3);
    else return __longlong_as_double(0x3fe6a09e667f3bcdLL);
  }
  if constexpr (sizeof(T) == 4) return __int_as_float(0x3f13cd3a);
  else return __longlong_as_double(0x3fe279a74590331cLL);
}

template <class L, typename T, bool FOLD>
__global__ void __launch_bounds__(BX2)
    k_cg_streamcoll(Dom d, T* __restrict__ fr, T* __restrict__ fb, TF<T> s,
                    const uint8_t* __restrict__ solid,
                    const uint32_t* __restrict__ slow, T omega, T tau,
                    ColorParamsDev cp) {
  int i, j, k;
  if (!node_coords<BX2>(d, i, j, k)) return;
  const int64_t fi = fidx(d, i, j, k);
  const int64_t mi = midx(d, i, j, k);
  if (solid[fi]) return;
  const int64_t ms = d.mstride;
  T ux, uy, uz, p[6];
  if constexpr (FOLD) {
    prepare_node_stress<L, T>(d, s, mi, tau, cp, ux, uy, uz, p);
  } else {
    ux = s.mom[mi];
    uy = s.mom[ms + mi];
    uz = L::dim == 3 ? s.mom[2 * ms + mi] : T(0);
    constexpr int np = L::dim * (L::dim + 1) / 2;
#pragma unroll
    for (int c = 0; c < np; ++c) p[c] = s.pin[c * ms + mi];
  }
  const T r = s.rho[mi];
  NodeMoments<T> m;
  if constexpr (L::dim == 3)
    m = prepare_node<T>(r, ux, uy, uz, p[0], p[1], p[2], p[3], p[4], p[5]);
  else
    m = prepare_node<T>(r, ux, uy, T(0), p[0], p[1], T(0), p[2], T(0), T(0));
  const T om1 = T(1) - omega;
  const T pert_coef = T(2.25) * T(cp.sigma) * omega;
  const T rr = s.rho_r[mi];
  const T rb = s.rho_b[mi];
  const T red_frac = rr / r;
  const T rec_amp = T(cp.beta) * (rr * rb / r);
  const T gx = s.grad[mi];
  const T gy = s.grad[ms + mi];
  const T gz = L::dim == 3 ? s.grad[2 * ms + mi] : T(0);
  const T gn = sqrt(gx * gx + gy * gy + gz * gz);
  const bool interface = gn > T(cp.grad_threshold);
  const T pert_amp = interface ? pert_coef * gn : T(0);
  const T inv_gn = interface ? T(1) / gn : T(0);
  const T nhx = gx * inv_gn, nhy = gy * inv_gn, nhz = gz * inv_gn;
  const uint32_t sm = slow[mi];
  const bool linear = cp.linear != 0;
  unroll<L::q>([&](auto A) {
    constexpr int a = decltype(A)::value;
    using dd = Dir<L, a>;
    constexpr T t = dd::template t<T>();
    constexpr T b = dd::template b<T>();
    T g_out = post_collision<L, a, T>(m, om1);
    T fr_out;
    if (interface) {
      const T cn = dot_c<dd::x, dd::y, dd::z>(nhx, nhy, nhz);
      const T shape = !linear ? t * cn * cn - b : t * cn - b;
      g_out += pert_amp * shape;
      fr_out = red_frac * g_out + rec_amp * t * cn * inv_cnorm<T, dd::norm2>();
    } else {
      fr_out = red_frac * g_out;
    }
    const T fb_out = g_out - fr_out;
    if ((sm >> a) & 1u) {
      int tc[3] = {i + dd::x, j + dd::y, k + dd::z};
      const int nd[3] = {d.nx, d.ny, d.nz};
      bool bounce = false;
      T wx = T(0), wy = T(0), wz = T(0);
#pragma unroll
      for (int ax = 0; ax < 3; ++ax) {
        if (tc[ax] < 0 || tc[ax] >= nd[ax]) {
          const int face = 2 * ax + (tc[ax] < 0 ? 0 : 1);
          const int mode = d.mode[face];
          if (mode == kWrap) {
            tc[ax] = tc[ax] < 0 ? tc[ax] + nd[ax] : tc[ax] - nd[ax];
          } else if (mode == kWall) {
            bounce = true;
            wx += T(d.uw[face][0]);
            wy += T(d.uw[face][1]);
            wz += T(d.uw[face][2]);
          }
        }
      }
      int64_t target = 0;
      if (!bounce) {
        target = fidx(d, tc[0], tc[1], tc[2]);
        if (solid[target]) bounce = true;
      }
      if (bounce) {
        const T corr = bounce_correction<L, a, T>(wx, wy, wz);
        const T corr_r = red_frac * corr;
        fr[dd::opp * d.fstride + fi] = fr_out - corr_r;
        fb[dd::opp * d.fstride + fi] = fb_out - (corr - corr_r);
      } else {
        fr[a * d.fstride + target] = fr_out;
        fb[a * d.fstride + target] = fb_out;
      }
    } else {
      const int64_t off = int64_t(dd::x) +
                          int64_t(d.nx) * (int64_t(dd::y) + int64_t(d.ny) * dd::z);
      fr[a * d.fstride + fi + off] = fr_out;
      fb[a * d.fstride + fi + off] = fb_out;
    }
  });
}

// ---------------------------------------------------------------------------
// Box geometries (no solid mask): neighbours and push targets come from the
// node coordinates (face_steps) instead of the classify_nodes slow mask, and
// the regularised collision of opposite directions is shared (post_pair,
// exact for rho != -0: rho here is a +0-seeded sum over g, see
// tslb_pair.cuh). The interface terms keep the reference order per
// direction. Same results, bit for bit, as k_cg_gradient / k_cg_streamcoll.
// grad phi at one node from its neighbours (gradient_and_nci,
// multicomponent.hpp:178-200: wall neighbours take phi(x)); accumulation in
// the reference's direction order
// (neighbours as the node's pointer + a signed 32-bit offset: on z slabs the
// plane below node k = 0 is phi's ghost plane, at a negative offset)
template <class L, typename T, bool WALLS>
__device__ __forceinline__ void gradient_at(const T* __restrict__ phi, int64_t mi, const Steps32& st,
                                            T& gx, T& gy, T& gz) {
  const T* __restrict__ ph = phi + mi;
  const T phi0 = ph[0];
  gx = 0;
  gy = 0;
  gz = 0;
  unroll<L::q>([&](auto A) {
    constexpr int a = decltype(A)::value;
    using dd = Dir<L, a>;
    if constexpr (a > 0) {
      int delta = 0;
      bool wall = false;
      if constexpr (dd::x == 1) { delta += st.dp[0]; wall |= st.bp[0]; }
      if constexpr (dd::x == -1) { delta += st.dm[0]; wall |= st.bm[0]; }
      if constexpr (dd::y == 1) { delta += st.dp[1]; wall |= st.bp[1]; }
      if constexpr (dd::y == -1) { delta += st.dm[1]; wall |= st.bm[1]; }
      if constexpr (dd::z == 1) { delta += st.dp[2]; wall |= st.bp[2]; }
      if constexpr (dd::z == -1) { delta += st.dm[2]; wall |= st.bm[2]; }
      const T pn = (WALLS && wall) ? phi0 : __ldg(ph + delta);
      constexpr T w = dd::template t<T>();
      const T tp = w * pn;
      if constexpr (dd::x == 1) gx += tp;
      if constexpr (dd::x == -1) gx -= tp;
      if constexpr (dd::y == 1) gy += tp;
      if constexpr (dd::y == -1) gy -= tp;
      if constexpr (dd::z == 1) gz += tp;
      if constexpr (dd::z == -1) gz -= tp;
    }
  });
  gx = T(3) * gx;
  gy = T(3) * gy;
  gz = T(3) * gz;
}

template <class L, typename T, bool WALLS>
__global__ void __launch_bounds__(BX2) k_cg_gradient_box(Dom d, TF<T> s) {
  int i, j, k;
  if (!node_coords<BX2>(d, i, j, k)) return;
  const int64_t mi = midx(d, i, j, k);
  T gx, gy, gz;
  gradient_at<L, T, WALLS>(s.phi, mi, face_steps32(d, i, j, k), gx, gy, gz);
  const int64_t ms = d.mstride;
  s.grad[mi] = gx;
  s.grad[ms + mi] = gy;
  if constexpr (L::dim == 3) s.grad[2 * ms + mi] = gz;
}

// Near-contact scan (gradient_and_nci's second half, multicomponent.hpp:
// 202-238) on a box geometry that may be a z slab: a probe that crosses a
// slab face continues into phi's ghost planes (the solver keeps nci_reach of
// them on each side), and a hit there flags the node in the flag buffer's
// matching ghost plane -- the neighbour owning that node ORs it into its own
// flags (k_flag_or). Set-only flags commute, so the merged result equals the
// single-domain scan. Owned flags were cleared by k_cg_moments.
template <class L, typename T>
__global__ void __launch_bounds__(BX2) k_cg_nci_box(Dom d, TF<T> s, ColorParamsDev cp) {
  int i, j, k;
  if (!node_coords<BX2>(d, i, j, k)) return;
  const T bulk_cut = T(-1) + T(cp.eps_bulk);
  if (!(s.phi[midx(d, i, j, k)] < bulk_cut)) return;
  const int nd[3] = {d.nx, d.ny, d.nz};
  // detail::advance (multicomponent.hpp:126-143): wrap periodic axes, stop
  // at walls; slab faces lead into the ghost planes
  auto advance = [&](int cx, int cy, int cz, int (&c)[3]) {
    const int dc[3] = {cx, cy, cz};
    int tc[3];
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      tc[ax] = c[ax] + dc[ax];
      if (tc[ax] < 0 || tc[ax] >= nd[ax]) {
        const int m = d.mode[2 * ax + (tc[ax] < 0 ? 0 : 1)];
        if (m == kWrap) tc[ax] += tc[ax] < 0 ? nd[ax] : -nd[ax];
        else if (m != kGhost) return false;
      }
    }
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) c[ax] = tc[ax];
    return true;
  };
  unroll<L::q>([&](auto A) {
    constexpr int a = decltype(A)::value;
    using dd = Dir<L, a>;
    if constexpr (a > 0 && dd::opp > a) {  // one probe per +-c pair
      int64_t hit_p = 0, hit_m = 0;
      bool found = false;
      int c[3] = {i, j, k};
      for (int st = 0; st < cp.nci_reach; ++st) {
        if (!advance(dd::x, dd::y, dd::z, c)) break;
        const int64_t t = midx(d, c[0], c[1], c[2]);
        if (s.phi[t] >= bulk_cut) {
          hit_p = t;
          found = true;
          break;
        }
      }
      if (!found) return;
      found = false;
      c[0] = i;
      c[1] = j;
      c[2] = k;
      for (int st = 0; st < cp.nci_reach; ++st) {
        if (!advance(-dd::x, -dd::y, -dd::z, c)) break;
        const int64_t t = midx(d, c[0], c[1], c[2]);
        if (s.phi[t] >= bulk_cut) {
          hit_m = t;
          found = true;
          break;
        }
      }
      if (!found) return;
      s.flag[hit_p] = 1;
      s.flag[hit_m] = 1;
    }
  });
}

__global__ void __launch_bounds__(256) k_flag_or(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src,
                                                 int64_t n) {
  const int64_t i = int64_t(blockIdx.x) * 256 + threadIdx.x;
  if (i < n) dst[i] |= src[i];
}

// GRAD: compute grad phi in place from the phi stencil instead of reading
// the gradient arrays (the step's gradient phase folded in; the host
// mirror computes the arrays lazily when they are read)
#ifdef TSLB_CG_MINB
#define TSLB_CG_BOUNDS __launch_bounds__(BX2, TSLB_CG_MINB)
#else
#define TSLB_CG_BOUNDS __launch_bounds__(BX2)
#endif
template <class L, typename T, bool FOLD, bool WALLS, bool GRAD>
__global__ void TSLB_CG_BOUNDS
    k_cg_streamcoll_box(Dom d, const __grid_constant__ PopBases<T> pop, TF<T> s, T omega, T tau,
                        ColorParamsDev cp) {
  int i, j, k;
  if (!node_coords<BX2>(d, i, j, k)) return;
  const int64_t fi = fidx(d, i, j, k);
  const int64_t mi = midx(d, i, j, k);
  const int64_t ms = d.mstride;
  T ux, uy, uz, p[6];
  if constexpr (FOLD) {
    prepare_node_stress<L, T>(d, s, mi, tau, cp, ux, uy, uz, p);
  } else {
    ux = s.mom[mi];
    uy = s.mom[ms + mi];
    uz = L::dim == 3 ? s.mom[2 * ms + mi] : T(0);
    constexpr int np = L::dim * (L::dim + 1) / 2;
#pragma unroll
    for (int c = 0; c < np; ++c) p[c] = s.pin[c * ms + mi];
  }
  const T r = s.rho[mi];
  NodeMoments<T> m;
  if constexpr (L::dim == 3)
    m = prepare_node<T>(r, ux, uy, uz, p[0], p[1], p[2], p[3], p[4], p[5]);
  else
    m = prepare_node<T>(r, ux, uy, T(0), p[0], p[1], T(0), p[2], T(0), T(0));
  const T om1 = T(1) - omega;
  const T pert_coef = T(2.25) * T(cp.sigma) * omega;
  const T rr = s.rho_r[mi];
  const T rb = s.rho_b[mi];
  const T red_frac = rr / r;
  const T rec_amp = T(cp.beta) * (rr * rb / r);
  const Steps32 st = face_steps32(d, i, j, k);
  T gx, gy, gz;
  if constexpr (GRAD) {
    gradient_at<L, T, WALLS>(s.phi, mi, st, gx, gy, gz);
    if constexpr (L::dim == 2) gz = T(0);
  } else {
    gx = s.grad[mi];
    gy = s.grad[ms + mi];
    gz = L::dim == 3 ? s.grad[2 * ms + mi] : T(0);
  }
  const T gn = sqrt(gx * gx + gy * gy + gz * gz);
  const bool interface = gn > T(cp.grad_threshold);
  const T pert_amp = interface ? pert_coef * gn : T(0);
  const T inv_gn = interface ? T(1) / gn : T(0);
  const T nhx = gx * inv_gn, nhy = gy * inv_gn, nhz = gz * inv_gn;
  const bool linear = cp.linear != 0;
  // (a population array holds < 2^32 elements: 32-bit slot indices)
  const uint32_t fi32 = uint32_t(fi);

  // one direction: perturbation + recolouring (reference order), then push
  // or bounce (multicomponent.hpp:340-398). IFACE is the node's interface
  // test, hoisted out of the direction loop (one branch per node).
  auto out = [&](auto A, auto IF, T g_out) {
    constexpr int a = decltype(A)::value;
    constexpr bool IFACE = decltype(IF)::value;
    using dd = Dir<L, a>;
    constexpr T t = dd::template t<T>();
    constexpr T b = dd::template b<T>();
    T fr_out;
    if constexpr (IFACE) {
      const T cn = dot_c<dd::x, dd::y, dd::z>(nhx, nhy, nhz);
      const T shape = !linear ? t * cn * cn - b : t * cn - b;
      g_out += pert_amp * shape;
      fr_out = red_frac * g_out + rec_amp * t * cn * inv_cnorm<T, dd::norm2>();
    } else {
      fr_out = red_frac * g_out;
    }
    const T fb_out = g_out - fr_out;
    int delta = 0;
    bool bounce = false;
    if constexpr (dd::x == 1) { delta += st.dp[0]; bounce |= st.bp[0]; }
    if constexpr (dd::x == -1) { delta += st.dm[0]; bounce |= st.bm[0]; }
    if constexpr (dd::y == 1) { delta += st.dp[1]; bounce |= st.bp[1]; }
    if constexpr (dd::y == -1) { delta += st.dm[1]; bounce |= st.bm[1]; }
    if constexpr (dd::z == 1) { delta += st.dp[2]; bounce |= st.bp[2]; }
    if constexpr (dd::z == -1) { delta += st.dm[2]; bounce |= st.bm[2]; }
    if (WALLS && bounce) {
      T wx = T(0), wy = T(0), wz = T(0);
      auto add = [&](bool crossed, int face) {
        if (crossed) {
          wx += T(d.uw[face][0]);
          wy += T(d.uw[face][1]);
          wz += T(d.uw[face][2]);
        }
      };
      if constexpr (dd::x == 1) add(st.bp[0], XMax);
      if constexpr (dd::x == -1) add(st.bm[0], XMin);
      if constexpr (dd::y == 1) add(st.bp[1], YMax);
      if constexpr (dd::y == -1) add(st.bm[1], YMin);
      if constexpr (dd::z == 1) add(st.bp[2], ZMax);
      if constexpr (dd::z == -1) add(st.bm[2], ZMin);
      const T corr = bounce_correction<L, a, T>(wx, wy, wz);
      const T corr_r = red_frac * corr;
      pop.r[dd::opp][fi32] = fr_out - corr_r;
      pop.b[dd::opp][fi32] = fb_out - (corr - corr_r);
    } else {
      const uint32_t t = fi32 + uint32_t(delta);
      // streaming (evict-first) stores: the populations are read back only
      // by the next step's colour moments, long after L2 has turned over
      // (r02: 5.34 vs 5.36 ms at 512^3)
      __stcs(&pop.r[a][t], fr_out);
      __stcs(&pop.b[a][t], fb_out);
    }
  };
  auto all_dirs = [&](auto IF) {
    unroll<L::q>([&](auto A) {
      constexpr int a = decltype(A)::value;
      if constexpr (a == 0) {
        out(A, IF, post_rest<L, T>(m, om1));
      } else if constexpr (a & 1) {
        T ga, gb;
        post_pair<L, a, T>(m, om1, ga, gb);
        out(A, IF, ga);
        out(std::integral_constant<int, a + 1>{}, IF, gb);
      }
    });
  };
  if (interface) all_dirs(std::true_type{});
  else all_dirs(std::false_type{});
}

// ---------------------------------------------------------------------------
// The whole box step in ONE pass (f_old -> f_new, ping-pong population
// buffers): colour moments + grad phi + prepare_stress + perturbation +
// recolouring + push. A CTA owns a 32 x 8 column tile and marches through
// its z range; the populations of the next plane -- the tile and a one-node
// ring around it, all 2q arrays -- are staged in shared memory by cp.async
// one plane ahead; each tile node reduces its own colour moments (kept in
// registers for the collision of that plane and written to the moment
// arrays, which keep the reference's host-visible values), the ring's phi
// is recomputed from its staged populations, and grad phi is taken from
// three planes of phi in shared memory. Same arithmetic, in the same order,
// as k_cg_moments + k_cg_streamcoll_box: same bits, without the round trip
// of the 52 B of moments per node through HBM (356 instead of 408 B per
// lattice update). Box geometries (nx % 32 == ny % 8 == 0), NCI off, whole
// domains.
__device__ __forceinline__ int wrap_coord2(int g, int n, int lo, int hi) {
  if (g < 0) return lo == kWrap ? g + n : -1;
  if (g >= n) return hi == kWrap ? g - n : -1;
  return g;
}

namespace fused {
constexpr int FX = 32, FY = 8, FT = FX * FY;  // tile, threads
constexpr int FR = FY + 2;                    // staged rows (y halo)
constexpr int FPA = FR * FX + 2 * FR;         // staged elements per array: rows + left / right columns
constexpr int FPX = FX + 2;                   // phi plane width
constexpr int kLz = 64;                       // planes per CTA
template <class L, typename T>
constexpr size_t smem_bytes() {
  return size_t(2) * 2 * L::q * FPA * sizeof(T) + size_t(3) * FR * FPX * sizeof(T);
}
}  // namespace fused

template <class L, typename T, bool WALLS>
__global__ void __launch_bounds__(fused::FT)
    k_cg_fused(Dom d, const __grid_constant__ PopBases<T> src, const __grid_constant__ PopBases<T> dst, TF<T> s,
               T omega, T tau, ColorParamsDev cp) {
  using namespace fused;
  constexpr int Q = L::q, NA = 2 * Q;
  extern __shared__ __align__(16) unsigned char fz_raw[];
  T* stg = reinterpret_cast<T*>(fz_raw);    // [2][NA][FPA]
  T* phs = stg + 2 * NA * FPA;              // [3][FR][FPX]
  const int tid = threadIdx.x, lx = tid & 31, ly = tid >> 5;
  const int x0 = int(blockIdx.x) * FX, y0 = int(blockIdx.y) * FY;
  const int za = int(blockIdx.z) * kLz, zb = min(za + kLz, d.nz);
  const int gx = x0 + lx, gy = y0 + ly;
  const int64_t ms = d.mstride;
  const T om1 = T(1) - omega;
  const T pert_coef = T(2.25) * T(cp.sigma) * omega;
  const bool linear = cp.linear != 0;
  // rows y0-1 .. y0+FY and the columns x0-1, x0+FX (wrapped; -1 beyond a wall)
  auto row_of = [&](int r) { return wrap_coord2(y0 - 1 + r, d.ny, d.mode[YMin], d.mode[YMax]); };
  const int colL = wrap_coord2(x0 - 1, d.nx, d.mode[XMin], d.mode[XMax]);
  const int colR = wrap_coord2(x0 + FX, d.nx, d.mode[XMin], d.mode[XMax]);

  // stage plane z (wrapped; nothing beyond a wall) into buffer b
  auto stage = [&](int z, int b) {
    const int zz = wrap_coord2(z, d.nz, d.mode[ZMin], d.mode[ZMax]);
    if (zz < 0) return;
    T* sb = stg + b * NA * FPA;
    // rows: 16-byte pieces
    constexpr int EP = 16 / int(sizeof(T)), PR = FX / EP;
    for (int t = tid; t < NA * FR * PR; t += FT) {
      const int piece = t % PR, rr = (t / PR) % FR, a = t / (PR * FR);
      const int yy = row_of(rr);
      if (yy < 0) continue;
      const T* g = (a < Q ? src.r[a] : src.b[a - Q]) + (int64_t(yy) * d.nx + int64_t(zz) * d.plane + x0 + EP * piece);
      __pipeline_memcpy_async(sb + a * FPA + rr * FX + EP * piece, g, 16);
    }
    // left / right columns: one element each
    for (int t = tid; t < NA * 2 * FR; t += FT) {
      const int rr = t % FR, side = (t / FR) & 1, a = t / (2 * FR);
      const int yy = row_of(rr), xx = side ? colR : colL;
      if (yy < 0 || xx < 0) continue;
      const T* g = (a < Q ? src.r[a] : src.b[a - Q]) + (int64_t(yy) * d.nx + int64_t(zz) * d.plane + xx);
      __pipeline_memcpy_async(sb + a * FPA + FR * FX + side * FR + rr, g, sizeof(T));
    }
  };
  // colour moments of a staged node (color_moments order, k_cg_moments)
  struct CM {
    T rr, rb, r, jx, jy, jz, pxx, pyy, pzz, pxy, pxz, pyz;
  };
  auto moments_at = [&](const T* sb, int off) {
    CM m{};
    unroll<Q>([&](auto A) {
      constexpr int a = decltype(A)::value;
      using dd = Dir<L, a>;
      const T fra = sb[a * FPA + off];
      const T fba = sb[(Q + a) * FPA + off];
      const T ga = fra + fba;
      m.rr += fra;
      m.rb += fba;
      m.r += ga;
      if constexpr (dd::x == 1) m.jx += ga;
      if constexpr (dd::x == -1) m.jx -= ga;
      if constexpr (dd::y == 1) m.jy += ga;
      if constexpr (dd::y == -1) m.jy -= ga;
      if constexpr (dd::z == 1) m.jz += ga;
      if constexpr (dd::z == -1) m.jz -= ga;
      if constexpr (dd::x != 0) m.pxx += ga;
      if constexpr (dd::y != 0) m.pyy += ga;
      if constexpr (dd::z != 0) m.pzz += ga;
      if constexpr (dd::x * dd::y == 1) m.pxy += ga;
      if constexpr (dd::x * dd::y == -1) m.pxy -= ga;
      if constexpr (dd::x * dd::z == 1) m.pxz += ga;
      if constexpr (dd::x * dd::z == -1) m.pxz -= ga;
      if constexpr (dd::y * dd::z == 1) m.pyz += ga;
      if constexpr (dd::y * dd::z == -1) m.pyz -= ga;
    });
    return m;
  };
  auto phi_sum = [&](const T* sb, int off) {  // (rr - rb) / r of a ring node
    T rr = 0, rb = 0, r = 0;
    unroll<Q>([&](auto A) {
      constexpr int a = decltype(A)::value;
      const T fra = sb[a * FPA + off];
      const T fba = sb[(Q + a) * FPA + off];
      rr += fra;
      rb += fba;
      r += fra + fba;
    });
    return (rr - rb) / r;
  };
  // the ring node this thread reduces (warp 0: row below, warp 1: row above,
  // warp 2: left and right columns incl. corners), -1 for none
  int ring_off = -1, ring_phi = -1;
  if (ly == 0) {
    ring_off = 0 * FX + lx;
    ring_phi = 0 * FPX + lx + 1;
  } else if (ly == 1) {
    ring_off = (FR - 1) * FX + lx;
    ring_phi = (FR - 1) * FPX + lx + 1;
  } else if (ly == 2 && (lx < FR || (lx >= 16 && lx < 16 + FR))) {
    const int side = lx >= 16, rr = lx - 16 * side;
    ring_off = FR * FX + side * FR + rr;
    ring_phi = rr * FPX + (side ? FPX - 1 : 0);
  }
  bool ring_ok = false;
  if (ring_off >= 0) {
    const int rr = ring_off < FR * FX ? ring_off / FX : (ring_off - FR * FX) % FR;
    const bool col = ring_off >= FR * FX;
    const int xx = col ? ((ring_off - FR * FX) / FR ? colR : colL) : 0;
    ring_ok = row_of(rr) >= 0 && xx >= 0;
  }

  // prologue: planes za-1 and za staged; phi(za-1) and phi(za), moments(za)
  stage(za - 1, 0);
  __pipeline_commit();
  stage(za, 1);
  __pipeline_commit();
  CM mc{};
  auto plane_exists = [&](int z) { return wrap_coord2(z, d.nz, d.mode[ZMin], d.mode[ZMax]) >= 0; };
  // the colour moments of the tile node (kept) and phi of the tile and ring
  // nodes of plane z from staging buffer b
  auto reduce_plane = [&](int z, int b, CM& out) {
    const T* sb = stg + b * NA * FPA;
    T* ph = phs + ((z % 3 + 3) % 3) * FR * FPX;
    if (!plane_exists(z)) return;
    out = moments_at(sb, (ly + 1) * FX + lx);
    ph[(ly + 1) * FPX + lx + 1] = (out.rr - out.rb) / out.r;
    if (ring_ok) ph[ring_phi] = phi_sum(sb, ring_off);
  };
  __pipeline_wait_prior(1);
  __syncthreads();
  {
    CM dummy{};
    reduce_plane(za - 1, 0, dummy);
  }
  __syncthreads();  // (buffer 0 is reused for plane za+1)
  stage(za + 1, 0);
  __pipeline_commit();
  __pipeline_wait_prior(1);
  __syncthreads();
  reduce_plane(za, 1, mc);

  for (int z = za; z < zb; ++z) {
    // phi(z) is in shared memory (barrier below), moments(z) in mc;
    // plane z+1 is staged in buffer (z+1-za+1)&1 = (z-za)&1
    const int bn = (z - za) & 1;
    __pipeline_wait_prior(0);
    __syncthreads();
    CM mn{};
    reduce_plane(z + 1, bn, mn);
    __syncthreads();
    // the buffer of plane z (the other one) is free: stage plane z+2
    if (z + 2 <= zb) stage(z + 2, bn ^ 1);
    __pipeline_commit();

    // ---- collide and push plane z (cg_streamcoll_box order)
    const int64_t fi = fidx(d, gx, gy, z);
    const int64_t mi = midx(d, gx, gy, z);
    // the colour moments of f(t) into the host-visible arrays (k_cg_moments)
    s.flag[mi] = 0;
    s.rho_r[mi] = mc.rr;
    s.rho_b[mi] = mc.rb;
    s.rho[mi] = mc.r;
    const T phi0 = (mc.rr - mc.rb) / mc.r;
    s.phi[mi] = phi0;
    s.mom[mi] = mc.jx;
    s.mom[ms + mi] = mc.jy;
    s.mom[2 * ms + mi] = mc.jz;
    s.pin[mi] = mc.pxx;
    s.pin[ms + mi] = mc.pyy;
    s.pin[2 * ms + mi] = mc.pzz;
    s.pin[3 * ms + mi] = mc.pxy;
    s.pin[4 * ms + mi] = mc.pxz;
    s.pin[5 * ms + mi] = mc.pyz;
    // prepare_stress (NCI off: the force is 0)
    const T F0 = 0, F1 = 0, F2 = 0;
    const T ux = mc.jx + tau * F0, uy = mc.jy + tau * F1, uz = mc.jz + tau * F2;
    const T c3 = cs2<T>();
    T p[6];
    p[0] = mc.pxx + (-c3 * mc.r - ux * ux);
    p[1] = mc.pyy + (-c3 * mc.r - uy * uy);
    p[2] = mc.pzz + (-c3 * mc.r - uz * uz);
    p[3] = mc.pxy - ux * uy;
    p[4] = mc.pxz - ux * uz;
    p[5] = mc.pyz - uy * uz;
    const NodeMoments<T> m = prepare_node<T>(mc.r, ux, uy, uz, p[0], p[1], p[2], p[3], p[4], p[5]);
    const T red_frac = mc.rr / mc.r;
    const T rec_amp = T(cp.beta) * (mc.rr * mc.rb / mc.r);
    const Steps32 st = face_steps32(d, gx, gy, z);
    // grad phi from the three phi planes (gradient_at order; a neighbour
    // beyond a wall reads phi(x))
    T gxx = 0, gyy = 0, gzz = 0;
    unroll<Q>([&](auto A) {
      constexpr int a = decltype(A)::value;
      using dd = Dir<L, a>;
      if constexpr (a > 0) {
        bool wall = false;
        if constexpr (dd::x == 1) wall |= st.bp[0];
        if constexpr (dd::x == -1) wall |= st.bm[0];
        if constexpr (dd::y == 1) wall |= st.bp[1];
        if constexpr (dd::y == -1) wall |= st.bm[1];
        if constexpr (dd::z == 1) wall |= st.bp[2];
        if constexpr (dd::z == -1) wall |= st.bm[2];
        const T* ph = phs + (((z + dd::z) % 3 + 3) % 3) * FR * FPX;
        const T pn = (WALLS && wall) ? phi0 : ph[(ly + 1 + dd::y) * FPX + lx + 1 + dd::x];
        constexpr T w = dd::template t<T>();
        const T tp = w * pn;
        if constexpr (dd::x == 1) gxx += tp;
        if constexpr (dd::x == -1) gxx -= tp;
        if constexpr (dd::y == 1) gyy += tp;
        if constexpr (dd::y == -1) gyy -= tp;
        if constexpr (dd::z == 1) gzz += tp;
        if constexpr (dd::z == -1) gzz -= tp;
      }
    });
    gxx = T(3) * gxx;
    gyy = T(3) * gyy;
    gzz = T(3) * gzz;
    const T gn = sqrt(gxx * gxx + gyy * gyy + gzz * gzz);
    const bool interface = gn > T(cp.grad_threshold);
    const T pert_amp = interface ? pert_coef * gn : T(0);
    const T inv_gn = interface ? T(1) / gn : T(0);
    const T nhx = gxx * inv_gn, nhy = gyy * inv_gn, nhz = gzz * inv_gn;
    const uint32_t fi32 = uint32_t(fi);
    auto out = [&](auto A, auto IF, T g_out) {
      constexpr int a = decltype(A)::value;
      constexpr bool IFACE = decltype(IF)::value;
      using dd = Dir<L, a>;
      constexpr T t = dd::template t<T>();
      constexpr T b = dd::template b<T>();
      T fr_out;
      if constexpr (IFACE) {
        const T cn = dot_c<dd::x, dd::y, dd::z>(nhx, nhy, nhz);
        const T shape = !linear ? t * cn * cn - b : t * cn - b;
        g_out += pert_amp * shape;
        fr_out = red_frac * g_out + rec_amp * t * cn * inv_cnorm<T, dd::norm2>();
      } else {
        fr_out = red_frac * g_out;
      }
      const T fb_out = g_out - fr_out;
      int delta = 0;
      bool bounce = false;
      if constexpr (dd::x == 1) { delta += st.dp[0]; bounce |= st.bp[0]; }
      if constexpr (dd::x == -1) { delta += st.dm[0]; bounce |= st.bm[0]; }
      if constexpr (dd::y == 1) { delta += st.dp[1]; bounce |= st.bp[1]; }
      if constexpr (dd::y == -1) { delta += st.dm[1]; bounce |= st.bm[1]; }
      if constexpr (dd::z == 1) { delta += st.dp[2]; bounce |= st.bp[2]; }
      if constexpr (dd::z == -1) { delta += st.dm[2]; bounce |= st.bm[2]; }
      if (WALLS && bounce) {
        T wx = T(0), wy = T(0), wz = T(0);
        auto add = [&](bool crossed, int face) {
          if (crossed) {
            wx += T(d.uw[face][0]);
            wy += T(d.uw[face][1]);
            wz += T(d.uw[face][2]);
          }
        };
        if constexpr (dd::x == 1) add(st.bp[0], XMax);
        if constexpr (dd::x == -1) add(st.bm[0], XMin);
        if constexpr (dd::y == 1) add(st.bp[1], YMax);
        if constexpr (dd::y == -1) add(st.bm[1], YMin);
        if constexpr (dd::z == 1) add(st.bp[2], ZMax);
        if constexpr (dd::z == -1) add(st.bm[2], ZMin);
        const T corr = bounce_correction<L, a, T>(wx, wy, wz);
        const T corr_r = red_frac * corr;
        dst.r[dd::opp][fi32] = fr_out - corr_r;
        dst.b[dd::opp][fi32] = fb_out - (corr - corr_r);
      } else {
        const uint32_t tt = fi32 + uint32_t(delta);
        dst.r[a][tt] = fr_out;
        dst.b[a][tt] = fb_out;
      }
    };
    auto all_dirs = [&](auto IF) {
      unroll<Q>([&](auto A) {
        constexpr int a = decltype(A)::value;
        if constexpr (a == 0) {
          out(A, IF, post_rest<L, T>(m, om1));
        } else if constexpr (a & 1) {
          T ga, gb;
          post_pair<L, a, T>(m, om1, ga, gb);
          out(A, IF, ga);
          out(std::integral_constant<int, a + 1>{}, IF, gb);
        }
      });
    };
    if (interface) all_dirs(std::true_type{});
    else all_dirs(std::false_type{});
    mc = mn;
  }
}

// ---------------------------------------------------------------------------
// device droplet initialiser (initialize_colors, multicomponent.hpp:427-449,
// with the tslb_main droplet profile 0.5 (1 + tanh(R - r)))
template <class L, typename T>
__global__ void __launch_bounds__(BX2)
    k_init_colors(Dom d, T* __restrict__ fr, T* __restrict__ fb,
                  const uint8_t* __restrict__ solid, InitSpec sp) {
  int i, j, k;
  if (!node_coords<BX2>(d, i, j, k)) return;
  const int64_t fi = fidx(d, i, j, k);
  if (solid[fi]) return;
  const double kg = double(k + sp.z0);
  const double dz2 = L::dim == 3 ? (kg - sp.cz) * (kg - sp.cz) : 0.0;
  const double dist = sp.radius - sqrt((i - sp.cx) * (i - sp.cx) +
                                       (j - sp.cy) * (j - sp.cy) + dz2);
  const double prof = 0.5 * (1.0 + tanh(dist / sp.width));
  const T rr = T(prof), rb = T(1.0 - prof);
  const T r = rr + rb;
  const NodeMoments<T> m =
      prepare_node<T>(r, T(0), T(0), T(0), T(0), T(0), T(0), T(0), T(0), T(0));
  const T frac = rr / r;
  unroll<L::q>([&](auto A) {
    constexpr int a = decltype(A)::value;
    const T fe = equilibrium<L, a, T>(m);
    fr[a * d.fstride + fi] = frac * fe;
    fb[a * d.fstride + fi] = fe - frac * fe;
  });
}

// ---------------------------------------------------------------------------
namespace {
inline dim3 grid2(const Dom& d) {
  return row_grid(dx2(d));
}
template <class F>
int with_lat2(int lat, F&& f) {
  switch (lat) {
    case kD2Q9: f(D2Q9{}); return 0;
    case kD3Q19: f(D3Q19{}); return 0;
    case kD3Q27: f(D3Q27{}); return 0;
    default: return 1;
  }
}
}  // namespace

template <typename T>
int launch_cg_moments(int lat, const Dom& d, const T* fr, const T* fb,
                      const TwoFields& s, const uint8_t* solid,
                      cudaStream_t st) {
  return with_lat2(lat, [&](auto L) {
    k_cg_moments<decltype(L), T><<<grid2(d), BX2, 0, st>>>(dx2(d), fr, fb, tf_of<T>(s), solid);
  });
}

template <typename T>
int launch_cg_gradient(int lat, const Dom& d, const TwoFields& s,
                       const uint8_t* solid, const uint32_t* slow,
                       const ColorParamsDev& cp, cudaStream_t st) {
  return with_lat2(lat, [&](auto L) {
    bool walls = false;
    for (int fc = 0; fc < 6; ++fc) walls |= d.mode[fc] == kWall;
    if (!d.has_solid && cp.nci_strength == 0.0 && walls)
      k_cg_gradient_box<decltype(L), T, true><<<grid2(d), BX2, 0, st>>>(dx2(d), tf_of<T>(s));
    else if (!d.has_solid && cp.nci_strength == 0.0)
      k_cg_gradient_box<decltype(L), T, false><<<grid2(d), BX2, 0, st>>>(dx2(d), tf_of<T>(s));
    else
      k_cg_gradient<decltype(L), T><<<grid2(d), BX2, 0, st>>>(dx2(d), tf_of<T>(s), solid, slow, cp);
  });
}

template <typename T>
int launch_cg_prepare_stress(int lat, const Dom& d, const TwoFields& s,
                             const uint8_t* solid, double omega,
                             const ColorParamsDev& cp, cudaStream_t st) {
  const T tau = T(1) / T(omega);
  return with_lat2(lat, [&](auto L) {
    k_cg_prepare<decltype(L), T><<<grid2(d), BX2, 0, st>>>(dx2(d), tf_of<T>(s), solid, tau, cp);
  });
}

template <typename T>
int launch_cg_streamcoll(int lat, const Dom& d, T* fr, T* fb,
                         const TwoFields& s, const uint8_t* solid,
                         const uint32_t* slow, double omega,
                         const ColorParamsDev& cp, int fold_prepare,
                         cudaStream_t st) {
  const T om = T(omega);
  const T tau = T(1) / om;
  return with_lat2(lat, [&](auto L) {
    // the fused step (fold_prepare) reads rho from k_cg_moments, a +0-seeded
    // sum, so the pair rewrite is exact; the standalone phase may see
    // user-written moments and keeps the reference order
    if (!d.has_solid && fold_prepare) {
      bool walls = false;
      for (int fc = 0; fc < 6; ++fc) walls |= d.mode[fc] == kWall;
      if (walls)
        k_cg_streamcoll_box<decltype(L), T, true, true, false>
            <<<grid2(d), BX2, 0, st>>>(dx2(d), pop_bases(fr, fb, d, decltype(L)::q), tf_of<T>(s), om, tau, cp);
      else
        k_cg_streamcoll_box<decltype(L), T, true, false, false>
            <<<grid2(d), BX2, 0, st>>>(dx2(d), pop_bases(fr, fb, d, decltype(L)::q), tf_of<T>(s), om, tau, cp);
      return;
    }
    if (fold_prepare)
      k_cg_streamcoll<decltype(L), T, true>
          <<<grid2(d), BX2, 0, st>>>(dx2(d), fr, fb, tf_of<T>(s), solid, slow, om, tau, cp);
    else
      k_cg_streamcoll<decltype(L), T, false>
          <<<grid2(d), BX2, 0, st>>>(dx2(d), fr, fb, tf_of<T>(s), solid, slow, om, tau, cp);
  });
}

// The step's gradient + prepare_stress + stream_collide_recolor in one
// kernel (box geometries, NCI off). Returns nonzero when not applicable.
template <typename T>
int launch_cg_streamcoll_grad(int lat, const Dom& d, T* fr, T* fb, const TwoFields& s, double omega,
                              const ColorParamsDev& cp, cudaStream_t st) {
  if (d.has_solid || cp.nci_strength != 0.0) return 1;
  const T om = T(omega);
  const T tau = T(1) / om;
  bool walls = false;
  for (int fc = 0; fc < 6; ++fc) walls |= d.mode[fc] == kWall;
  return with_lat2(lat, [&](auto L) {
    if (walls)
      k_cg_streamcoll_box<decltype(L), T, true, true, true>
          <<<grid2(d), BX2, 0, st>>>(dx2(d), pop_bases(fr, fb, d, decltype(L)::q), tf_of<T>(s), om, tau, cp);
    else
      k_cg_streamcoll_box<decltype(L), T, true, false, true>
          <<<grid2(d), BX2, 0, st>>>(dx2(d), pop_bases(fr, fb, d, decltype(L)::q), tf_of<T>(s), om, tau, cp);
  });
}

// The fused one-pass step (k_cg_fused): f_old -> f_new plus the colour
// moment arrays. Returns 1 (nothing launched) where it does not apply.
template <typename T>
int launch_cg_fused(int lat, const Dom& d, const T* fr, const T* fb, T* gr, T* gb, const TwoFields& s,
                    double omega, const ColorParamsDev& cp, cudaStream_t st) {
  using namespace fused;
  if (lat == kD2Q9 || d.has_solid || d.ghost || cp.nci_strength != 0.0) return 1;
  if (d.nx % FX || d.ny % FY || d.k0 != 0 || d.nzr != d.nz) return 1;
  if (d.ny / FY > 65535 || (d.nz + kLz - 1) / kLz > 65535) return 1;
  const T om = T(omega);
  const T tau = T(1) / om;
  bool walls = false;
  for (int fc = 0; fc < 6; ++fc) walls |= d.mode[fc] == kWall;
  const dim3 grid(unsigned(d.nx / FX), unsigned(d.ny / FY), unsigned((d.nz + kLz - 1) / kLz));
  int err = 1;
  auto go = [&](auto L) {
    using Lat = decltype(L);
    constexpr size_t smem = smem_bytes<Lat, T>();
    if constexpr (smem > 227 * 1024) {
      return;
    } else {
      auto kern = walls ? k_cg_fused<Lat, T, true> : k_cg_fused<Lat, T, false>;
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      if (e == cudaSuccess) {
        kern<<<grid, FT, smem, st>>>(d, pop_bases(const_cast<T*>(fr), const_cast<T*>(fb), d, Lat::q),
                                      pop_bases(gr, gb, d, Lat::q), tf_of<T>(s), om, tau, cp);
        e = cudaGetLastError();
      }
      err = e == cudaSuccess ? 0 : -int(e);
    }
  };
  if (lat == kD3Q19) go(D3Q19{});
  else go(D3Q27{});
  return err;
}

bool cg_fused_supported(int lat, const Dom& d, int esz, const ColorParamsDev& cp) {
  using namespace fused;
  if (lat == kD2Q9 || d.has_solid || d.ghost || cp.nci_strength != 0.0) return false;
  if (d.nx % FX || d.ny % FY) return false;
  const size_t q = lat == kD3Q19 ? 19 : 27;
  return size_t(2) * 2 * q * FPA * esz + size_t(3) * FR * FPX * esz <= 227 * 1024;
}

// gradient_and_nci on a box geometry / z slab: the gradient kernel (phi
// stencil through the ghost planes) and the near-contact scan
template <typename T>
int launch_cg_gradient_nci_box(int lat, const Dom& d, const TwoFields& s, const ColorParamsDev& cp,
                               cudaStream_t st) {
  if (d.has_solid) return 1;
  bool walls = false;
  for (int fc = 0; fc < 6; ++fc) walls |= d.mode[fc] == kWall;
  return with_lat2(lat, [&](auto L) {
    if (walls) k_cg_gradient_box<decltype(L), T, true><<<grid2(d), BX2, 0, st>>>(dx2(d), tf_of<T>(s));
    else k_cg_gradient_box<decltype(L), T, false><<<grid2(d), BX2, 0, st>>>(dx2(d), tf_of<T>(s));
    if (T(cp.nci_strength) != T(0)) k_cg_nci_box<decltype(L), T><<<grid2(d), BX2, 0, st>>>(dx2(d), tf_of<T>(s), cp);
  });
}

int launch_flag_or(uint8_t* dst, const uint8_t* src, int64_t n, cudaStream_t st) {
  if (n <= 0) return 0;
  k_flag_or<<<unsigned((n + 255) / 256), 256, 0, st>>>(dst, src, n);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

template <typename T>
int launch_init_colors(int lat, const Dom& d, T* fr, T* fb,
                       const uint8_t* solid, const InitSpec& sp,
                       cudaStream_t st) {
  return with_lat2(lat, [&](auto L) {
    k_init_colors<decltype(L), T><<<grid2(d), BX2, 0, st>>>(dx2(d), fr, fb, solid, sp);
  });
}

#define TSLB_INST2(T)                                                         \
  template int launch_cg_moments<T>(int, const Dom&, const T*, const T*,      \
                                    const TwoFields&, const uint8_t*,         \
                                    cudaStream_t);                            \
  template int launch_cg_gradient<T>(int, const Dom&, const TwoFields&,       \
                                     const uint8_t*, const uint32_t*,         \
                                     const ColorParamsDev&, cudaStream_t);    \
  template int launch_cg_prepare_stress<T>(int, const Dom&, const TwoFields&, \
                                           const uint8_t*, double,            \
                                           const ColorParamsDev&,             \
                                           cudaStream_t);                     \
  template int launch_cg_streamcoll<T>(int, const Dom&, T*, T*,               \
                                       const TwoFields&, const uint8_t*,      \
                                       const uint32_t*, double,               \
                                       const ColorParamsDev&, int,            \
                                       cudaStream_t);                         \
  template int launch_cg_fused<T>(int, const Dom&, const T*, const T*, T*, T*, \
                                  const TwoFields&, double, const ColorParamsDev&, \
                                  cudaStream_t);                              \
  template int launch_cg_streamcoll_grad<T>(int, const Dom&, T*, T*,         \
                                            const TwoFields&, double,         \
                                            const ColorParamsDev&,            \
                                            cudaStream_t);                    \
  template int launch_init_colors<T>(int, const Dom&, T*, T*,                 \
                                     const uint8_t*, const InitSpec&,         \
                                     cudaStream_t);                           \
  template int launch_cg_gradient_nci_box<T>(int, const Dom&, const TwoFields&, \
                                             const ColorParamsDev&, cudaStream_t);
TSLB_INST2(float)
TSLB_INST2(double)
#undef TSLB_INST2

}  // namespace tslb_cuda
