// Single-fluid thread-safe LB kernels for sm_100a (F1 schedule).
//
//   k_moments     reference compute_moments      kernels.hpp:74-107
//   k_streamcoll  reference stream_collide_fused kernels.hpp:154-204
//   k_stream_only reference stream_only          kernels.hpp:219-256
//   k_collide     collide-in-place half of reference_step, kernels.hpp:272-287
//   k_classify    reference classify_nodes       boundary.hpp:61-111
//   k_init_*      device analytic initialisers (throughput runs only)
//
// One CUDA grid = one reference phase; the kernel boundary on a single stream
// replaces WorkerPool's phase barrier (parallel.hpp:60-67). Every slot
// (x, a) has exactly one writer inside k_streamcoll, so the push into the
// single population buffer is race-free exactly as on the CPU, and results
// do not depend on the launch shape.
//
// Arithmetic: double for all node-local math (bit-identical to the reference
// for double AND float storage, given --fmad=false), or -- opt-in "fp32 math"
// mode -- float (tolerance parity).
#include <cstdint>

#include "tslb_collision.cuh"
#include "tslb_domain.cuh"
#include "tslb_kernels.h"
#include "tslb_msums.cuh"
#include "tslb_pair.cuh"

namespace tslb_cuda {

constexpr int BX = 128;  // threads per block along x

// ---------------------------------------------------------------------------
// phase 1: moments
// ---------------------------------------------------------------------------
template <class L, typename T, typename C, bool SOLID>
__global__ void __launch_bounds__(BX) k_moments(Dom d, const T* __restrict__ f,
                                                T* __restrict__ mo,
                                                const uint8_t* __restrict__ solid) {
  int i, j, k;
  if (!node_coords<BX>(d, i, j, k)) return;
  const int64_t fi = fidx(d, i, j, k);
  const int64_t mi = midx(d, i, j, k);
  if constexpr (SOLID) {
    if (solid[fi]) return;
  }
  // compute_moments' sums and finish (tslb_msums.cuh: bit-identical to the
  // reference order for fp64 node math; the same forms as the M kernel)
  T v[L::q];
#pragma unroll
  for (int a = 0; a < L::q; ++a) v[a] = __ldg(f + a * d.fstride + fi);
  const int64_t ms = d.mstride;
  moment_tail<L, T, C>(d, msums<L, T, C>(v), [&](int c, T x) { mo[c * ms + mi] = x; });
}

// load_node_moments (kernels.hpp:109-125)
template <class L, typename T, typename C>
__device__ __forceinline__ NodeMoments<C> load_node(const Dom& d,
                                                    const T* __restrict__ mo,
                                                    int64_t mi) {
  const int64_t ms = d.mstride;
  if constexpr (L::dim == 3) {
    return prepare_node<C>(C(mo[mi]), C(mo[ms + mi]), C(mo[2 * ms + mi]),
                           C(mo[3 * ms + mi]), C(mo[4 * ms + mi]),
                           C(mo[5 * ms + mi]), C(mo[6 * ms + mi]),
                           C(mo[7 * ms + mi]), C(mo[8 * ms + mi]),
                           C(mo[9 * ms + mi]));
  } else {
    return prepare_node<C>(C(mo[mi]), C(mo[ms + mi]), C(mo[2 * ms + mi]), C(0),
                           C(mo[3 * ms + mi]), C(mo[4 * ms + mi]), C(0),
                           C(mo[5 * ms + mi]), C(0), C(0));
  }
}

// Generic (slow-bit) resolution with solids: resolve_push, boundary.hpp:118-144.
// Returns true on bounce; u_wall summed in T over crossed wall faces.
template <typename T>
__device__ __forceinline__ bool resolve_generic(const Dom& d,
                                                const uint8_t* __restrict__ solid,
                                                int cx, int cy, int cz, int i,
                                                int j, int k, int64_t& target,
                                                T& wx, T& wy, T& wz) {
  int tc[3] = {i + cx, j + cy, k + cz};
  const int nd[3] = {d.nx, d.ny, d.nz};
  bool bounce = false;
  wx = T(0);
  wy = T(0);
  wz = T(0);
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    if (tc[ax] < 0 || tc[ax] >= nd[ax]) {
      const int face = 2 * ax + (tc[ax] < 0 ? 0 : 1);
      const int m = d.mode[face];
      if (m == kWrap) {
        tc[ax] = tc[ax] < 0 ? tc[ax] + nd[ax] : tc[ax] - nd[ax];
      } else if (m == kWall) {
        bounce = true;
        wx += T(d.uw[face][0]);
        wy += T(d.uw[face][1]);
        wz += T(d.uw[face][2]);
      }  // kGhost: keep the out-of-slab z, it addresses the ghost plane
    }
  }
  if (bounce) return true;
  const int64_t t = fidx(d, tc[0], tc[1], tc[2]);
  if (solid[t]) return true;
  target = t;
  return false;
}

// ---------------------------------------------------------------------------
// phase 2: fused stream-collide (push)
// ---------------------------------------------------------------------------
template <class L, typename T, typename C, bool SOLID>
__global__ void __launch_bounds__(BX)
    k_streamcoll(Dom d, T* __restrict__ f, const T* __restrict__ mo,
                 const uint8_t* __restrict__ solid,
                 const uint32_t* __restrict__ slow, C om1) {
  int i, j, k;
  if (!node_coords<BX>(d, i, j, k)) return;
  const int64_t fi = fidx(d, i, j, k);
  const int64_t mi = midx(d, i, j, k);
  if constexpr (SOLID) {
    if (solid[fi]) return;
  }
  const NodeMoments<C> m = load_node<L, T, C>(d, mo, mi);
  if constexpr (SOLID) {
    const uint32_t sm = slow[mi];
    unroll<L::q>([&](auto A) {
      constexpr int a = decltype(A)::value;
      using dd = Dir<L, a>;
      const T out = T(sf_post_ref<L, a, C>(m, om1));
      if ((sm >> a) & 1u) {
        int64_t target = 0;
        T wx, wy, wz;
        if (resolve_generic<T>(d, solid, dd::x, dd::y, dd::z, i, j, k, target,
                               wx, wy, wz)) {
          f[dd::opp * d.fstride + fi] =
              T(C(out) - bounce_correction<L, a, C>(C(wx), C(wy), C(wz)));
        } else {
          f[a * d.fstride + target] = out;
        }
      } else {
        constexpr int64_t off_c = dd::x;
        const int64_t off =
            off_c + int64_t(d.nx) * (int64_t(dd::y) + int64_t(d.ny) * dd::z);
        f[a * d.fstride + fi + off] = out;
      }
    });
  } else {
    const Steps st = face_steps(d, i, j, k);
    unroll<L::q>([&](auto A) {
      constexpr int a = decltype(A)::value;
      using dd = Dir<L, a>;
      const T out = T(sf_post_ref<L, a, C>(m, om1));
      int64_t delta = 0;
      bool bounce = false;
      if constexpr (dd::x == 1) { delta += st.dp[0]; bounce |= st.bp[0]; }
      if constexpr (dd::x == -1) { delta += st.dm[0]; bounce |= st.bm[0]; }
      if constexpr (dd::y == 1) { delta += st.dp[1]; bounce |= st.bp[1]; }
      if constexpr (dd::y == -1) { delta += st.dm[1]; bounce |= st.bm[1]; }
      if constexpr (dd::z == 1) { delta += st.dp[2]; bounce |= st.bp[2]; }
      if constexpr (dd::z == -1) { delta += st.dm[2]; bounce |= st.bm[2]; }
      if (bounce) {
        // sum the velocities of every crossed wall face, in T, axis order
        T wx = T(0), wy = T(0), wz = T(0);
        auto add = [&](bool crossed, int face) {
          if (crossed && d.mode[face] == kWall) {
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
        f[dd::opp * d.fstride + fi] =
            T(C(out) - bounce_correction<L, a, C>(C(wx), C(wy), C(wz)));
      } else {
        f[a * d.fstride + fi + delta] = out;
      }
    });
  }
}

// ---------------------------------------------------------------------------
// two-buffer reference step pieces (oracle parity; not on the hot path)
// ---------------------------------------------------------------------------
template <class L, typename T, typename C, bool SOLID>
__global__ void __launch_bounds__(BX)
    k_collide(Dom d, T* __restrict__ f, const T* __restrict__ mo,
              const uint8_t* __restrict__ solid, C om1) {
  int i, j, k;
  if (!node_coords<BX>(d, i, j, k)) return;
  const int64_t fi = fidx(d, i, j, k);
  if constexpr (SOLID) {
    if (solid[fi]) return;
  }
  const NodeMoments<C> m = load_node<L, T, C>(d, mo, midx(d, i, j, k));
  unroll<L::q>([&](auto A) {
    constexpr int a = decltype(A)::value;
    f[a * d.fstride + fi] = T(sf_post_ref<L, a, C>(m, om1));
  });
}

template <class L, typename T, bool SOLID>
__global__ void __launch_bounds__(BX)
    k_stream_only(Dom d, const T* __restrict__ f, T* __restrict__ dst,
                  const uint8_t* __restrict__ solid,
                  const uint32_t* __restrict__ slow) {
  int i, j, k;
  if (!node_coords<BX>(d, i, j, k)) return;
  const int64_t fi = fidx(d, i, j, k);
  if (SOLID && solid[fi]) return;
  const uint32_t sm = SOLID ? slow[midx(d, i, j, k)] : 0xffffffffu;
  unroll<L::q>([&](auto A) {
    constexpr int a = decltype(A)::value;
    using dd = Dir<L, a>;
    const T out = f[a * d.fstride + fi];
    int64_t target = 0;
    T wx, wy, wz;
    if (((sm >> a) & 1u) || !SOLID) {
      if (resolve_generic<T>(d, solid, dd::x, dd::y, dd::z, i, j, k, target, wx,
                             wy, wz)) {
        dst[dd::opp * d.fstride + fi] = T(
            double(out) - bounce_correction<L, a, double>(double(wx), double(wy),
                                                         double(wz)));
      } else {
        dst[a * d.fstride + target] = out;
      }
    } else {
      const int64_t off = int64_t(dd::x) +
                          int64_t(d.nx) * (int64_t(dd::y) + int64_t(d.ny) * dd::z);
      dst[a * d.fstride + fi + off] = out;
    }
  });
}

// ---------------------------------------------------------------------------
// geometry: classify_nodes (boundary.hpp:61-111), bit-exact
// ---------------------------------------------------------------------------
template <class L>
__global__ void __launch_bounds__(BX)
    k_classify(Dom d, const uint8_t* __restrict__ solid,
               uint32_t* __restrict__ slow, unsigned long long* n_fluid) {
  int i, j, k;
  const bool live = node_coords<BX>(d, i, j, k);
  unsigned fluid = 0;
  if (live) {
    const int64_t fi = fidx(d, i, j, k);
    uint32_t mask = 0;
    if (!solid[fi]) {
      fluid = 1;
      const int nd[3] = {d.nx, d.ny, d.nz};
      unroll<L::q>([&](auto A) {
        constexpr int a = decltype(A)::value;
        if constexpr (a > 0) {
          using dd = Dir<L, a>;
          int tc[3] = {i + dd::x, j + dd::y, k + dd::z};
          bool s = false;
#pragma unroll
          for (int ax = 0; ax < 3; ++ax) {
            if (tc[ax] < 0 || tc[ax] >= nd[ax]) {
              s = true;
              tc[ax] = tc[ax] < 0 ? tc[ax] + nd[ax] : tc[ax] - nd[ax];
            }
          }
          if (!s && solid[fidx(d, tc[0], tc[1], tc[2])]) s = true;
          if (s) mask |= (uint32_t(1) << a);
        }
      });
    }
    slow[midx(d, i, j, k)] = mask;
  }
  // warp-aggregated fluid count (integer: order-independent, deterministic)
  const unsigned cnt = __popc(__ballot_sync(0xffffffffu, fluid));
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(n_fluid, (unsigned long long)cnt);
}

// ---------------------------------------------------------------------------
// device analytic initialisers (initialize_regularized pattern,
// kernels.hpp:295-311, with the node state computed on the device)
// ---------------------------------------------------------------------------
// node state of the analytic initialisers (rest, shear, Taylor-Green)
template <class L, typename T>
__device__ __forceinline__ NodeMoments<T> init_state(const InitSpec& s, int i, int j, int k) {
  if (s.kind == kInitState) {  // user node states, already in T
    const T* p = static_cast<const T*>(s.state) + (int64_t(i) + int64_t(s.nx_g) * (int64_t(j) + int64_t(s.ny_g) * k));
    const int64_t q = s.sstride;
    if (!s.spi) {  // rho and u only: the prepare_node(rho, u, 0) of tslb_main.cpp:115-122
      if constexpr (L::dim == 3)
        return prepare_node<T>(p[0], p[q], p[2 * q], p[3 * q], T(0), T(0), T(0), T(0), T(0), T(0));
      else
        return prepare_node<T>(p[0], p[q], p[2 * q], T(0), T(0), T(0), T(0), T(0), T(0), T(0));
    }
    if constexpr (L::dim == 3)
      return prepare_node<T>(p[0], p[q], p[2 * q], p[3 * q], p[4 * q], p[5 * q], p[6 * q], p[7 * q], p[8 * q],
                             p[9 * q]);
    else
      return prepare_node<T>(p[0], p[q], p[2 * q], T(0), p[3 * q], p[4 * q], T(0), p[5 * q], T(0), T(0));
  }
  const double two_pi = 6.283185307179586476925286766559;
  double rho = 1.0, ux = 0.0, uy = 0.0, uz = 0.0;
  const int kg = k + s.z0;
  if (s.kind == kInitShear) {
    ux = s.amp * sin(two_pi * j / s.ny_g);
  } else if (s.kind == kInitTaylorGreen) {
    const double X = two_pi * (i + 0.5) / s.nx_g;
    const double Y = two_pi * (j + 0.5) / s.ny_g;
    const double Z = two_pi * (kg + 0.5) / s.nz_g;
    const double U0 = s.amp;
    if (L::dim == 3) {
      ux = U0 * sin(X) * cos(Y) * cos(Z);
      uy = -U0 * cos(X) * sin(Y) * cos(Z);
      rho = 1.0 + 3.0 * (U0 * U0 / 16.0) * (cos(2 * X) + cos(2 * Y)) *
                      (cos(2 * Z) + 2.0);
    } else {
      ux = U0 * sin(X) * cos(Y);
      uy = -U0 * cos(X) * sin(Y);
      rho = 1.0 + 3.0 * (U0 * U0 / 4.0) * (cos(2 * X) + cos(2 * Y));
    }
  }
  return prepare_node<T>(T(rho), T(ux), T(uy), T(uz), T(0), T(0), T(0), T(0), T(0), T(0));
}

// f(0) = f_eq + f_neq of the node state, in T (initialize_regularized,
// kernels.hpp:295-311)
template <class L, int A, typename T>
__device__ __forceinline__ T init_population(const NodeMoments<T>& m) {
  return equilibrium<L, A, T>(m) + regularized<L, A, T>(m);
}

template <class L, typename T>
__global__ void __launch_bounds__(BX)
    k_init_analytic(Dom d, T* __restrict__ f, const uint8_t* __restrict__ solid,
                    InitSpec s) {
  int i, j, k;
  if (!node_coords<BX>(d, i, j, k)) return;
  const int64_t fi = fidx(d, i, j, k);
  if (solid && solid[fi]) return;
  const NodeMoments<T> m = init_state<L, T>(s, i, j, k);
  unroll<L::q>([&](auto A) {
    constexpr int a = decltype(A)::value;
    f[a * d.fstride + fi] = init_population<L, a, T>(m);
  });
}

// The moments pass of the first step applied to the analytic f(0), without
// storing f(0) (M schedule, box geometries): the populations are formed in
// registers exactly as k_init_analytic stores them and reduced exactly as
// k_moments does (compute_moments, kernels.hpp:74-107).
template <class L, typename T, typename C>
__global__ void __launch_bounds__(BX)
    k_init_moments(Dom d, T* __restrict__ mo, InitSpec s) {
  int i, j, k;
  if (!node_coords<BX>(d, i, j, k)) return;
  const int64_t mi = midx(d, i, j, k);
  const NodeMoments<T> m = init_state<L, T>(s, i, j, k);
  T v[L::q];
  unroll<L::q>([&](auto A) {
    constexpr int a = decltype(A)::value;
    v[a] = init_population<L, a, T>(m);
  });
  const int64_t ms = d.mstride;
  moment_tail<L, T, C>(d, msums<L, T, C>(v), [&](int c, T x) { mo[c * ms + mi] = x; });
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
namespace {

inline dim3 grid_of(const Dom& d) {
  return row_grid(d);
}

template <class F>
int with_lat(int lat, F&& f) {
  switch (lat) {
    case kD2Q9: f(D2Q9{}); return 0;
    case kD3Q19: f(D3Q19{}); return 0;
    case kD3Q27: f(D3Q27{}); return 0;
    default: return 1;
  }
}

}  // namespace

template <typename T>
int launch_moments(int lat, int math, const Dom& d, const T* f, T* mo,
                   const uint8_t* solid, cudaStream_t st) {
  return with_lat(lat, [&](auto L) {
    using Lat = decltype(L);
    if (math == kMathDouble) {
      if (d.has_solid)
        k_moments<Lat, T, double, true><<<grid_of(d), BX, 0, st>>>(d, f, mo, solid);
      else
        k_moments<Lat, T, double, false><<<grid_of(d), BX, 0, st>>>(d, f, mo, solid);
    } else {
      if (d.has_solid)
        k_moments<Lat, T, float, true><<<grid_of(d), BX, 0, st>>>(d, f, mo, solid);
      else
        k_moments<Lat, T, float, false><<<grid_of(d), BX, 0, st>>>(d, f, mo, solid);
    }
  });
}

template <typename T>
int launch_streamcoll(int lat, int math, const Dom& d, T* f, const T* mo,
                      const uint8_t* solid, const uint32_t* slow, double omega,
                      cudaStream_t st) {
  return with_lat(lat, [&](auto L) {
    using Lat = decltype(L);
    // om1 = 1 - double(prm.omega) with omega stored as T (kernels.hpp:160)
    const double om1d = 1.0 - double(T(omega));
    if (math == kMathDouble) {
      if (d.has_solid)
        k_streamcoll<Lat, T, double, true>
            <<<grid_of(d), BX, 0, st>>>(d, f, mo, solid, slow, om1d);
      else
        k_streamcoll<Lat, T, double, false>
            <<<grid_of(d), BX, 0, st>>>(d, f, mo, solid, slow, om1d);
    } else {
      const float om1f = 1.0f - float(omega);
      if (d.has_solid)
        k_streamcoll<Lat, T, float, true>
            <<<grid_of(d), BX, 0, st>>>(d, f, mo, solid, slow, om1f);
      else
        k_streamcoll<Lat, T, float, false>
            <<<grid_of(d), BX, 0, st>>>(d, f, mo, solid, slow, om1f);
    }
  });
}

template <typename T>
int launch_collide(int lat, const Dom& d, T* f, const T* mo,
                   const uint8_t* solid, double omega, cudaStream_t st) {
  return with_lat(lat, [&](auto L) {
    using Lat = decltype(L);
    const double om1 = 1.0 - double(T(omega));
    if (d.has_solid)
      k_collide<Lat, T, double, true><<<grid_of(d), BX, 0, st>>>(d, f, mo, solid, om1);
    else
      k_collide<Lat, T, double, false><<<grid_of(d), BX, 0, st>>>(d, f, mo, solid, om1);
  });
}

template <typename T>
int launch_stream_only(int lat, const Dom& d, const T* f, T* dst,
                       const uint8_t* solid, const uint32_t* slow,
                       cudaStream_t st) {
  return with_lat(lat, [&](auto L) {
    using Lat = decltype(L);
    if (d.has_solid)
      k_stream_only<Lat, T, true><<<grid_of(d), BX, 0, st>>>(d, f, dst, solid, slow);
    else
      k_stream_only<Lat, T, false><<<grid_of(d), BX, 0, st>>>(d, f, dst, solid, slow);
  });
}

int launch_classify(int lat, const Dom& d, const uint8_t* solid,
                    uint32_t* slow, unsigned long long* n_fluid,
                    cudaStream_t st) {
  return with_lat(lat, [&](auto L) {
    using Lat = decltype(L);
    k_classify<Lat><<<grid_of(d), BX, 0, st>>>(d, solid, slow, n_fluid);
  });
}

template <typename T>
int launch_init_analytic(int lat, const Dom& d, T* f, const uint8_t* solid,
                         const InitSpec& s, cudaStream_t st) {
  return with_lat(lat, [&](auto L) {
    using Lat = decltype(L);
    k_init_analytic<Lat, T><<<grid_of(d), BX, 0, st>>>(d, f, solid, s);
  });
}

template <typename T>
int launch_init_moments(int lat, int math, const Dom& d, T* mo, const InitSpec& s, cudaStream_t st) {
  return with_lat(lat, [&](auto L) {
    using Lat = decltype(L);
    if (math == kMathDouble)
      k_init_moments<Lat, T, double><<<grid_of(d), BX, 0, st>>>(d, mo, s);
    else
      k_init_moments<Lat, T, float><<<grid_of(d), BX, 0, st>>>(d, mo, s);
  });
}

#define TSLB_INST(T)                                                          \
  template int launch_init_moments<T>(int, int, const Dom&, T*, const InitSpec&, \
                                      cudaStream_t);                          \
  template int launch_moments<T>(int, int, const Dom&, const T*, T*,          \
                                 const uint8_t*, cudaStream_t);               \
  template int launch_streamcoll<T>(int, int, const Dom&, T*, const T*,       \
                                    const uint8_t*, const uint32_t*, double,  \
                                    cudaStream_t);                            \
  template int launch_collide<T>(int, const Dom&, T*, const T*,               \
                                 const uint8_t*, double, cudaStream_t);       \
  template int launch_stream_only<T>(int, const Dom&, const T*, T*,           \
                                     const uint8_t*, const uint32_t*,         \
                                     cudaStream_t);                           \
  template int launch_init_analytic<T>(int, const Dom&, T*, const uint8_t*,   \
                                       const InitSpec&, cudaStream_t);
TSLB_INST(float)
TSLB_INST(double)
#undef TSLB_INST

}  // namespace tslb_cuda
