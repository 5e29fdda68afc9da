// Vectorised fused stream-collide for box geometries (no solid mask): the
// throughput kernel of the F1 schedule.
//
// Same results, bit for bit, as k_streamcoll / the reference
// stream_collide_fused (kernels.hpp:154-204); what changes is the shape:
//   * each thread owns VX consecutive x nodes (VX = 16 B / sizeof(T)), so the
//     moment loads and population stores are 128-bit and the address
//     arithmetic is paid once per VX nodes;
//   * pushes along c_x = +-1 land one element off the thread's aligned
//     vector: the missing element comes from the neighbour lane by a warp
//     shuffle, and the two ends of each warp's row segment patch their edge
//     element with a scalar store -- every slot still has exactly one writer;
//   * opposite directions share their work: Q_a : Pi^neq is identical for a
//     and opp(a), and c_opp . u = -(c_a . u), so one pair costs ~20 DP ops
//     instead of ~36. These rewrites only change the sign of intermediate
//     zeros, which cannot reach the result unless rho == -0.0; rho from the
//     moments pass is never -0.0 (a +0-seeded sum cannot produce it), and a
//     thread that sees rho == -0.0 (user-written moments) takes the
//     reference-order path instead.
#include <cstdint>

#include "tslb_collision.cuh"
#include "tslb_domain.cuh"
#include "tslb_kernels.h"
#include "tslb_pair.cuh"

namespace tslb_cuda {

constexpr int BXV = 128;

template <class L, typename T, typename C, int VX>
__device__ __forceinline__ void load_moments_vec(const Dom& d,
                                                 const T* __restrict__ mo,
                                                 int64_t mi,
                                                 NodeMoments<C> (&m)[VX]) {
  constexpr int NM = 1 + L::dim + L::dim * (L::dim + 1) / 2;
  T v[NM][VX];
#pragma unroll
  for (int c = 0; c < NM; ++c) Vec<T, VX>::load(mo + c * d.mstride + mi, v[c]);
#pragma unroll
  for (int x = 0; x < VX; ++x) {
    if constexpr (L::dim == 3)
      m[x] = prepare_node<C>(C(v[0][x]), C(v[1][x]), C(v[2][x]), C(v[3][x]), C(v[4][x]),
                             C(v[5][x]), C(v[6][x]), C(v[7][x]), C(v[8][x]), C(v[9][x]));
    else
      m[x] = prepare_node<C>(C(v[0][x]), C(v[1][x]), C(v[2][x]), C(0), C(v[3][x]),
                             C(v[4][x]), C(0), C(v[5][x]), C(0), C(0));
  }
}

struct RowGeom {
  int64_t dyp, dym, dzp, dzm;  // row deltas (wrapped / ghost-shifted)
  bool byp, bym, bzp, bzm;     // y / z step bounces off a wall
  bool xwall_lo, xwall_hi;     // x faces are walls
};

__device__ __forceinline__ RowGeom row_geom(const Dom& d, int j, int k) {
  RowGeom g;
  const int64_t nx = d.nx, pl = d.plane;
  g.dyp = nx;
  g.dym = -nx;
  g.dzp = pl;
  g.dzm = -pl;
  g.byp = g.bym = g.bzp = g.bzm = false;
  if (j == d.ny - 1) {
    if (d.mode[YMax] == kWrap) g.dyp = -nx * (d.ny - 1);
    else if (d.mode[YMax] == kWall) g.byp = true;
  }
  if (j == 0) {
    if (d.mode[YMin] == kWrap) g.dym = nx * (d.ny - 1);
    else if (d.mode[YMin] == kWall) g.bym = true;
  }
  if (k == d.nz - 1) {
    if (d.mode[ZMax] == kWrap) g.dzp = -pl * (d.nz - 1);
    else if (d.mode[ZMax] == kWall) g.bzp = true;
  }
  if (k == 0) {
    if (d.mode[ZMin] == kWrap) g.dzm = pl * (d.nz - 1);
    else if (d.mode[ZMin] == kWall) g.bzm = true;
  }
  g.xwall_lo = d.mode[XMin] == kWall;
  g.xwall_hi = d.mode[XMax] == kWall;
  return g;
}

// Store direction A's VX outputs of this thread. WALLS = false compiles out
// every bounce path (all faces periodic or slab ghosts).
template <class L, int A, typename T, typename C, int VX, bool WALLS>
__device__ __forceinline__ void push_dir(const Dom& d, T* __restrict__ f,
                                         const RowGeom& g, int64_t fi, int i0,
                                         bool seg_start, bool seg_end,
                                         const T (&o)[VX]) {
  using dd = Dir<L, A>;
  T* fa = f + A * d.fstride;
  int64_t dr = 0;
  bool by = false, bz = false;
  if constexpr (dd::y == 1) { dr += g.dyp; by = g.byp; }
  if constexpr (dd::y == -1) { dr += g.dym; by = g.bym; }
  if constexpr (dd::z == 1) { dr += g.dzp; bz = g.bzp; }
  if constexpr (dd::z == -1) { dr += g.dzm; bz = g.bzm; }

  if constexpr (dd::x == 0) {
    if (i0 < 0) return;  // inactive lane
    if constexpr (WALLS) {
      if (by || bz) {
        T b[VX];
#pragma unroll
        for (int v = 0; v < VX; ++v) b[v] = bounce_value<L, A, T, C>(d, o[v], false, by, bz);
        Vec<T, VX>::st(f + dd::opp * d.fstride + fi, b);
        return;
      }
    }
    Vec<T, VX>::st(fa + fi + dr, o);
  } else {
    // x-shifted push. Shuffles run on every lane of the warp (inactive
    // lanes carry dummies and store nothing).
    T carry;
    if constexpr (dd::x == 1) carry = __shfl_up_sync(0xffffffffu, o[VX - 1], 1);
    else carry = __shfl_down_sync(0xffffffffu, o[0], 1);
    if (i0 < 0) return;  // inactive lane
    if constexpr (WALLS) {
      if (by || bz) {
        // the whole row segment bounces (y/z wall); x edges may add their face
        T b[VX];
#pragma unroll
        for (int v = 0; v < VX; ++v) {
          const int x = i0 + v;
          const bool cx = dd::x == 1 ? (x == d.nx - 1 && g.xwall_hi) : (x == 0 && g.xwall_lo);
          b[v] = bounce_value<L, A, T, C>(d, o[v], cx, by, bz);
        }
        Vec<T, VX>::st(f + dd::opp * d.fstride + fi, b);
        return;
      }
    }
    T* base = fa + fi + dr;  // aligned slot of this thread's first node
    if constexpr (dd::x == 1) {
      // targets x0+1 .. x0+VX; aligned vector [x0 .. x0+VX-1] needs x0-1
      if (!seg_start) {
        T v[VX];
        v[0] = carry;
#pragma unroll
        for (int e = 1; e < VX; ++e) v[e] = o[e - 1];
        Vec<T, VX>::st(base, v);
      } else {
#pragma unroll
        for (int e = 1; e < VX; ++e) base[e] = o[e - 1];
      }
      if (seg_end) {
        const int x = i0 + VX;  // target of the last node
        if (x < d.nx) {
          base[VX] = o[VX - 1];
        } else if (WALLS && g.xwall_hi) {
          f[dd::opp * d.fstride + fi + VX - 1] =
              bounce_value<L, A, T, C>(d, o[VX - 1], true, false, false);
        } else {
          base[VX - d.nx] = o[VX - 1];  // periodic wrap to x = 0
        }
      }
    } else {
      // targets x0-1 .. x0+VX-2; aligned vector needs x0+VX from lane+1
      if (!seg_end) {
        T v[VX];
#pragma unroll
        for (int e = 0; e < VX - 1; ++e) v[e] = o[e + 1];
        v[VX - 1] = carry;
        Vec<T, VX>::st(base, v);
      } else {
#pragma unroll
        for (int e = 0; e < VX - 1; ++e) base[e] = o[e + 1];
      }
      if (seg_start) {
        if (i0 > 0) {
          base[-1] = o[0];
        } else if (WALLS && g.xwall_lo) {
          f[dd::opp * d.fstride + fi] = bounce_value<L, A, T, C>(d, o[0], true, false, false);
        } else {
          base[d.nx - 1] = o[0];  // periodic wrap to x = nx-1
        }
      }
    }
  }
}

// All q directions of this thread's VX nodes. EXACT selects the reference
// evaluation order (only needed if some rho is -0.0, see header).
template <class L, typename T, typename C, int VX, bool WALLS, bool EXACT>
__device__ __forceinline__ void all_dirs(const Dom& d, T* __restrict__ f,
                                         const RowGeom& g, int64_t fi, int i0,
                                         bool active, bool seg_start,
                                         bool seg_end,
                                         const NodeMoments<C> (&m)[VX], C om1) {
  unroll<L::q>([&](auto A) {
    constexpr int a = decltype(A)::value;
    if constexpr (a == 0) {
      T o[VX];
#pragma unroll
      for (int x = 0; x < VX; ++x)
        o[x] = EXACT ? T(sf_post_ref<L, 0, C>(m[x], om1)) : T(sf_post<L, 0, C>(m[x], om1));
      if (active) push_dir<L, 0, T, C, VX, WALLS>(d, f, g, fi, i0, seg_start, seg_end, o);
    } else if constexpr (a & 1) {
      T oa[VX], ob[VX];
#pragma unroll
      for (int x = 0; x < VX; ++x) {
        if constexpr (EXACT) {
          oa[x] = T(sf_post_ref<L, a, C>(m[x], om1));
          ob[x] = T(sf_post_ref<L, a + 1, C>(m[x], om1));
        } else {
          C ra, rb;
          sf_pair<L, a, C>(m[x], om1, ra, rb);
          oa[x] = T(ra);
          ob[x] = T(rb);
        }
      }
      push_dir<L, a, T, C, VX, WALLS>(d, f, g, fi, i0, seg_start, seg_end, oa);
      push_dir<L, a + 1, T, C, VX, WALLS>(d, f, g, fi, i0, seg_start, seg_end, ob);
    }
  });
}

// Reference-order path, outlined so it stays out of the hot instruction
// stream (taken only when some rho == -0.0, i.e. user-written moments).
template <class L, typename T, typename C, int VX, bool WALLS>
// Everything is passed by value and the moments are reloaded, so the hot
// path never spills its registers to set up this call.
__device__ __noinline__ void all_dirs_exact(Dom d, T* f, const T* mo, RowGeom g, int64_t mi, int64_t fi,
                                            int i0, bool active, bool seg_start, bool seg_end, C om1) {
  NodeMoments<C> m[VX];
  if (active) {
    load_moments_vec<L, T, C, VX>(d, mo, mi, m);
  } else {
#pragma unroll
    for (int x = 0; x < VX; ++x)
      m[x] = prepare_node<C>(C(1), C(0), C(0), C(0), C(0), C(0), C(0), C(0), C(0), C(0));
  }
  all_dirs<L, T, C, VX, WALLS, true>(d, f, g, fi, i0, active, seg_start, seg_end, m, om1);
}

template <class L, typename T, typename C, int VX, bool WALLS>
__global__ void __launch_bounds__(BXV)
    k_streamcoll_vec(Dom d, T* __restrict__ f, const T* __restrict__ mo, C om1) {
  unsigned xb;
  int j, k;
  row_block(d, xb, j, k);
  int i0 = int((xb * BXV + threadIdx.x) * VX);
  const bool active = i0 < d.nx;
  // active lanes form a prefix of the warp (rows never share a warp)
  const unsigned amask = __ballot_sync(0xffffffffu, active);
  const unsigned lane = threadIdx.x & 31u;
  const bool seg_start = lane == 0;
  const bool seg_end = active && (lane == 31u || !((amask >> (lane + 1)) & 1u));
  const int64_t mi = int64_t(d.nx) * (int64_t(j) + int64_t(d.ny) * k) + (active ? i0 : 0);
  const int64_t fi = mi + int64_t(d.ghost) * d.plane;
  if (!active) i0 = -1;

  NodeMoments<C> m[VX];
  if (active) {
    load_moments_vec<L, T, C, VX>(d, mo, mi, m);
  } else {
#pragma unroll
    for (int x = 0; x < VX; ++x)
      m[x] = prepare_node<C>(C(1), C(0), C(0), C(0), C(0), C(0), C(0), C(0), C(0), C(0));
  }
  bool exact = false;  // rho == -0.0 anywhere: fall back to reference order
#pragma unroll
  for (int x = 0; x < VX; ++x) exact |= (m[x].rho == C(0)) && signbit(m[x].rho);
  const RowGeom g = row_geom(d, j, k);

  if (__any_sync(0xffffffffu, exact))
    all_dirs_exact<L, T, C, VX, WALLS>(d, f, mo, g, mi, fi, i0, active, seg_start, seg_end, om1);
  else
    all_dirs<L, T, C, VX, WALLS, false>(d, f, g, fi, i0, active, seg_start, seg_end, m, om1);
}

// Software-pipelined form: a block walks KZ consecutive planes of its
// (x segment, row j) column and prefetches the next plane's moments into
// registers while the current plane is collided and pushed, so the load
// latency of each warp hides behind its own fp64 work (the fp64 build runs
// at low occupancy: ~90-170 registers per thread).
template <class L, typename T, typename C, int VX, bool WALLS>
__global__ void __launch_bounds__(BXV)
    k_streamcoll_pipe(Dom d, T* __restrict__ f, const T* __restrict__ mo, C om1, int kz) {
  constexpr int NM = 1 + L::dim + L::dim * (L::dim + 1) / 2;
  const int j = int(blockIdx.y);
  const int kb = d.k0 + int(blockIdx.z) * kz;
  const int ke = min(kb + kz, d.k0 + d.nzr);
  int i0 = int((blockIdx.x * BXV + threadIdx.x) * VX);
  const bool active = i0 < d.nx;
  const unsigned amask = __ballot_sync(0xffffffffu, active);
  const unsigned lane = threadIdx.x & 31u;
  const bool seg_start = lane == 0;
  const bool seg_end = active && (lane == 31u || !((amask >> (lane + 1)) & 1u));
  const int64_t mrow = int64_t(d.nx) * j + (active ? i0 : 0);
  if (!active) i0 = -1;

  T cur[NM][VX], nxt[NM][VX];
  auto fetch = [&](T (&buf)[NM][VX], int k) {
    const int64_t mi = mrow + int64_t(k) * d.plane;
#pragma unroll
    for (int c = 0; c < NM; ++c) Vec<T, VX>::load(mo + c * d.mstride + mi, buf[c]);
  };
  if (active) fetch(cur, kb);
#pragma unroll 1
  for (int k = kb; k < ke; ++k) {
    if (active && k + 1 < ke) fetch(nxt, k + 1);
    NodeMoments<C> m[VX];
#pragma unroll
    for (int x = 0; x < VX; ++x) {
      if (!active) {
        m[x] = prepare_node<C>(C(1), C(0), C(0), C(0), C(0), C(0), C(0), C(0), C(0), C(0));
      } else if constexpr (L::dim == 3) {
        m[x] = prepare_node<C>(C(cur[0][x]), C(cur[1][x]), C(cur[2][x]), C(cur[3][x]), C(cur[4][x]),
                               C(cur[5][x]), C(cur[6][x]), C(cur[7][x]), C(cur[8][x]), C(cur[9][x]));
      } else {
        m[x] = prepare_node<C>(C(cur[0][x]), C(cur[1][x]), C(cur[2][x]), C(0), C(cur[3][x]), C(cur[4][x]),
                               C(0), C(cur[5][x]), C(0), C(0));
      }
    }
    bool exact = false;
#pragma unroll
    for (int x = 0; x < VX; ++x) exact |= (m[x].rho == C(0)) && signbit(m[x].rho);
    const RowGeom g = row_geom(d, j, k);
    const int64_t mi = mrow + int64_t(k) * d.plane;
    const int64_t fi = mi + int64_t(d.ghost) * d.plane;
    if (__any_sync(0xffffffffu, exact))
      all_dirs_exact<L, T, C, VX, WALLS>(d, f, mo, g, mi, fi, i0, active, seg_start, seg_end, om1);
    else
      all_dirs<L, T, C, VX, WALLS, false>(d, f, g, fi, i0, active, seg_start, seg_end, m, om1);
#pragma unroll
    for (int c = 0; c < NM; ++c)
#pragma unroll
      for (int x = 0; x < VX; ++x) cur[c][x] = nxt[c][x];
  }
}

// vx: elements per thread (1, 2 or 4 for float; 1 or 2 for double);
// 0 picks the default (full 16-byte vectors for fp32 node math, 8-byte for
// fp64 node math, whose register footprint per node is twice as large).
// kz > 1 selects the software-pipelined kernel (kz planes per block).
template <typename T>
int launch_streamcoll_vec(int lat, int math, const Dom& d0, T* f, const T* mo,
                          double omega, int vx, int kz, cudaStream_t st) {
  if (vx == 0) vx = math == kMathDouble ? 8 / int(sizeof(T)) : 16 / int(sizeof(T));
  if (vx * int(sizeof(T)) > 16 || d0.nx % vx != 0) return 1;
  const double om1d = 1.0 - double(T(omega));
  const float om1f = 1.0f - float(omega);
  auto go = [&](auto L, auto V) {
    using Lat = decltype(L);
    constexpr int VX = decltype(V)::value;
    if constexpr (VX * sizeof(T) <= 16) {
      Dom d = d0;
      d.xblocks = (d.nx / VX + BXV - 1) / BXV;
      bool walls = false;
      for (int fc = 0; fc < 6; ++fc) walls |= d.mode[fc] == kWall;
      const int nzc = kz > 1 ? (d.nzr + kz - 1) / kz : 0;
      if (kz > 1 && d.ny <= 65535 && nzc <= 65535) {
        const dim3 grid(unsigned(d.xblocks), unsigned(d.ny), unsigned(nzc));
        if (math == kMathDouble) {
          if (walls) k_streamcoll_pipe<Lat, T, double, VX, true><<<grid, BXV, 0, st>>>(d, f, mo, om1d, kz);
          else k_streamcoll_pipe<Lat, T, double, VX, false><<<grid, BXV, 0, st>>>(d, f, mo, om1d, kz);
        } else {
          if (walls) k_streamcoll_pipe<Lat, T, float, VX, true><<<grid, BXV, 0, st>>>(d, f, mo, om1f, kz);
          else k_streamcoll_pipe<Lat, T, float, VX, false><<<grid, BXV, 0, st>>>(d, f, mo, om1f, kz);
        }
        return;
      }
      const dim3 grid = row_grid(d);
      if (math == kMathDouble) {
        if (walls) k_streamcoll_vec<Lat, T, double, VX, true><<<grid, BXV, 0, st>>>(d, f, mo, om1d);
        else k_streamcoll_vec<Lat, T, double, VX, false><<<grid, BXV, 0, st>>>(d, f, mo, om1d);
      } else {
        if (walls) k_streamcoll_vec<Lat, T, float, VX, true><<<grid, BXV, 0, st>>>(d, f, mo, om1f);
        else k_streamcoll_vec<Lat, T, float, VX, false><<<grid, BXV, 0, st>>>(d, f, mo, om1f);
      }
    }
  };
  auto by_vx = [&](auto L) {
    if (vx == 1) go(L, std::integral_constant<int, 1>{});
    else if (vx == 2) go(L, std::integral_constant<int, 2>{});
    else go(L, std::integral_constant<int, 4>{});
  };
  switch (lat) {
    case kD2Q9: by_vx(D2Q9{}); return 0;
    case kD3Q19: by_vx(D3Q19{}); return 0;
    case kD3Q27: by_vx(D3Q27{}); return 0;
    default: return 1;
  }
}

template int launch_streamcoll_vec<float>(int, int, const Dom&, float*, const float*, double, int, int, cudaStream_t);
template int launch_streamcoll_vec<double>(int, int, const Dom&, double*, const double*, double, int, int, cudaStream_t);

}  // namespace tslb_cuda
