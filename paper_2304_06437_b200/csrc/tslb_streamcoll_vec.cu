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

constexpr int BXV = 128;

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

// Post-collision values of the pair (A, A+1 = opp(A)), A odd.
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
  const C r = om1 * regularized<L, A, C>(m);  // reference order, shared
  out_a = ea + r;
  out_b = eb + r;
}

template <class L, typename C>
__device__ __forceinline__ C post_rest(const NodeMoments<C>& m, C om1) {
  constexpr C t = Dir<L, 0>::template t<C>();
  // rho + 3*(+0) + (4.5*(+0))*(+0) == rho for rho != -0
  const C e = t * (m.rho - m.usq15);
  return e + om1 * regularized<L, 0, C>(m);
}

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
        o[x] = EXACT ? T(post_collision<L, 0, C>(m[x], om1)) : T(post_rest<L, C>(m[x], om1));
      if (active) push_dir<L, 0, T, C, VX, WALLS>(d, f, g, fi, i0, seg_start, seg_end, o);
    } else if constexpr (a & 1) {
      T oa[VX], ob[VX];
#pragma unroll
      for (int x = 0; x < VX; ++x) {
        if constexpr (EXACT) {
          oa[x] = T(post_collision<L, a, C>(m[x], om1));
          ob[x] = T(post_collision<L, a + 1, C>(m[x], om1));
        } else {
          C ra, rb;
          post_pair<L, a, C>(m[x], om1, ra, rb);
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



// ===========================================================================
// Lean variant: one node per thread, scalar stores at precomputed per-
// direction offsets (interior nodes), everything else through an outlined
// reference-order path. Fewest issued instructions per node, which is what
// bounds the fp64-arithmetic build.
// ===========================================================================
constexpr int BXL = 128;

struct PushOffsets {
  int64_t off[27];  // a * fstride + c_x + nx c_y + nx ny c_z
};

// Reference-order push of one node (any face kind), moments reloaded.
template <class L, typename T, typename C>
__device__ __noinline__ void lean_slow_node(Dom d, T* f, const T* mo, int i, int j, int k, C om1) {
  const int64_t mi = midx(d, i, j, k);
  const int64_t fi = mi + int64_t(d.ghost) * d.plane;
  const int64_t ms = d.mstride;
  NodeMoments<C> m;
  if constexpr (L::dim == 3)
    m = prepare_node<C>(C(mo[mi]), C(mo[ms + mi]), C(mo[2 * ms + mi]), C(mo[3 * ms + mi]), C(mo[4 * ms + mi]),
                        C(mo[5 * ms + mi]), C(mo[6 * ms + mi]), C(mo[7 * ms + mi]), C(mo[8 * ms + mi]),
                        C(mo[9 * ms + mi]));
  else
    m = prepare_node<C>(C(mo[mi]), C(mo[ms + mi]), C(mo[2 * ms + mi]), C(0), C(mo[3 * ms + mi]),
                        C(mo[4 * ms + mi]), C(0), C(mo[5 * ms + mi]), C(0), C(0));
  const int c3[3] = {i, j, k};
  const int nd[3] = {d.nx, d.ny, d.nz};
  const int64_t unit[3] = {1, int64_t(d.nx), d.plane};
  unroll<L::q>([&](auto A) {
    constexpr int a = decltype(A)::value;
    using dd = Dir<L, a>;
    const T out = T(post_collision<L, a, C>(m, om1));
    const int cv[3] = {dd::x, dd::y, dd::z};
    int64_t delta = 0;
    bool bounce = false;
    T wx = T(0), wy = T(0), wz = T(0);
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      if (cv[ax] == 0) continue;
      delta += cv[ax] * unit[ax];
      const int t = c3[ax] + cv[ax];
      if (t < 0 || t >= nd[ax]) {
        const int face = 2 * ax + (t < 0 ? 0 : 1);
        if (d.mode[face] == kWrap) {
          delta -= cv[ax] * int64_t(nd[ax]) * unit[ax];
        } else if (d.mode[face] == kWall) {
          bounce = true;
          wx += T(d.uw[face][0]);
          wy += T(d.uw[face][1]);
          wz += T(d.uw[face][2]);
        }
      }
    }
    if (bounce)
      f[dd::opp * d.fstride + fi] = T(C(out) - bounce_correction<L, a, C>(C(wx), C(wy), C(wz)));
    else
      f[a * d.fstride + fi + delta] = out;
  });
}

template <class L, typename T, typename C>
__global__ void __launch_bounds__(BXL)
    k_streamcoll_lean(Dom d, T* __restrict__ f, const T* __restrict__ mo, C om1, PushOffsets po) {
  int i, j, k;
  if (!node_coords<BXL>(d, i, j, k)) return;
  const int64_t mi = midx(d, i, j, k);
  const int64_t ms = d.mstride;
  const T* p = mo + mi;
  constexpr int NM = 1 + L::dim + L::dim * (L::dim + 1) / 2;
  T v[NM];
#pragma unroll
  for (int c = 0; c < NM; ++c) v[c] = __ldg(p + c * ms);
  const C rho = C(v[0]);
  // nodes whose pushes leave the box through a wrap or a wall face, and the
  // (never produced by the moments pass) rho == -0.0, take the outlined path
  const bool edge = (i == 0 && d.mode[XMin] != kGhost) || (i == d.nx - 1 && d.mode[XMax] != kGhost) ||
                    (j == 0 && d.mode[YMin] != kGhost) || (j == d.ny - 1 && d.mode[YMax] != kGhost) ||
                    (k == 0 && d.mode[ZMin] != kGhost) || (k == d.nz - 1 && d.mode[ZMax] != kGhost);
  if (edge || (rho == C(0) && signbit(rho))) {
    lean_slow_node<L, T, C>(d, f, mo, i, j, k, om1);
    return;
  }
  NodeMoments<C> m;
  if constexpr (L::dim == 3)
    m = prepare_node<C>(rho, C(v[1]), C(v[2]), C(v[3]), C(v[4]), C(v[5]), C(v[6]), C(v[7]), C(v[8]), C(v[9]));
  else
    m = prepare_node<C>(rho, C(v[1]), C(v[2]), C(0), C(v[3]), C(v[4]), C(0), C(v[5]), C(0), C(0));
  T* base = f + (mi + int64_t(d.ghost) * d.plane);
  unroll<L::q>([&](auto A) {
    constexpr int a = decltype(A)::value;
    if constexpr (a == 0) {
      base[po.off[0]] = T(post_rest<L, C>(m, om1));
    } else if constexpr (a & 1) {
      C ra, rb;
      post_pair<L, a, C>(m, om1, ra, rb);
      base[po.off[a]] = T(ra);
      base[po.off[a + 1]] = T(rb);
    }
  });
}

template <typename T>
int launch_streamcoll_lean(int lat, int math, const Dom& d0, T* f, const T* mo, double omega,
                           cudaStream_t st) {
  Dom d = d0;
  d.xblocks = (d.nx + BXL - 1) / BXL;
  const dim3 grid = row_grid(d);
  const double om1d = 1.0 - double(T(omega));
  const float om1f = 1.0f - float(omega);
  auto go = [&](auto L) {
    using Lat = decltype(L);
    PushOffsets po{};
    for (int a = 0; a < Lat::q; ++a)
      po.off[a] = int64_t(a) * d.fstride + Lat::c[a][0] +
                  int64_t(d.nx) * (Lat::c[a][1] + int64_t(d.ny) * Lat::c[a][2]);
    if (math == kMathDouble)
      k_streamcoll_lean<Lat, T, double><<<grid, BXL, 0, st>>>(d, f, mo, om1d, po);
    else
      k_streamcoll_lean<Lat, T, float><<<grid, BXL, 0, st>>>(d, f, mo, om1f, po);
  };
  switch (lat) {
    case kD2Q9: go(D2Q9{}); return 0;
    case kD3Q19: go(D3Q19{}); return 0;
    case kD3Q27: go(D3Q27{}); return 0;
    default: return 1;
  }
}

template int launch_streamcoll_lean<float>(int, int, const Dom&, float*, const float*, double, cudaStream_t);
template int launch_streamcoll_lean<double>(int, int, const Dom&, double*, const double*, double, cudaStream_t);

}  // namespace tslb_cuda

namespace tslb_cuda {

// ===========================================================================
// Row kernel: one CTA owns a whole x row (nx / VX threads, a multiple of 32,
// <= 1024) and walks KZ planes of it. Because the CTA holds the entire row,
// the one-element shift of c_x = +-1 pushes is closed inside the CTA: within
// a warp by a shuffle, across warps through shared memory, and across the
// row ends by the periodic wrap (or, for x walls, by the bounce of the
// opposite direction of the same node). Every population store is therefore
// one aligned VX-wide vector -- no per-lane edge stores, no divergence.
// Rows that touch a wrapped/walled y or z face (block-uniform) take the
// general per-lane path (push_dir). Moments of the next plane are prefetched
// into registers while the current plane is collided.
// ===========================================================================
constexpr int kMaxRowThreads = 512;  // keeps >= 128 registers per thread

struct RowOffsets {
  int64_t off[27];  // (a * fstride + nx c_y + nx ny c_z) * sizeof(T): aligned part of the push
};

// regularized_dir without the +0 seed: identical whenever the first picked
// stress component is nonzero (checked by the caller, see header).
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

template <class L, typename T, typename C, int VX, bool EXACT>
__device__ __forceinline__ void row_outputs(const NodeMoments<C> (&m)[VX], C om1, T (&o)[L::q][VX]) {
  unroll<L::q>([&](auto A) {
    constexpr int a = decltype(A)::value;
#pragma unroll
    for (int x = 0; x < VX; ++x) {
      if constexpr (EXACT) {
        o[a][x] = T(post_collision<L, a, C>(m[x], om1));
      } else if constexpr (a == 0) {
        o[0][x] = T(post_rest<L, C>(m[x], om1));
      } else if constexpr (a & 1) {
        using dd = Dir<L, a>;
        constexpr C t = dd::template t<C>();
        const C cu = dot_noseed<dd::x, dd::y, dd::z, C>(m[x].ux, m[x].uy, m[x].uz);
        const C c3 = C(3) * cu;
        const C qq = C(4.5) * cu * cu;
        const C ea = t * (m[x].rho + c3 + qq - m[x].usq15);
        const C eb = t * (m[x].rho - c3 + qq - m[x].usq15);
        const C r = om1 * regularized_noseed<L, a, C>(m[x]);
        o[a][x] = T(ea + r);
        o[a + 1][x] = T(eb + r);
      }
    }
  });
}

template <class L, typename T, typename C, int VX, bool XWALL>
__global__ void __launch_bounds__(kMaxRowThreads)
    k_streamcoll_row(Dom d, T* __restrict__ f, const T* __restrict__ mo, C om1, int kz, RowOffsets ro) {
  constexpr int NM = 1 + L::dim + L::dim * (L::dim + 1) / 2;
  extern __shared__ unsigned char smem_raw[];
  T* carry_up = reinterpret_cast<T*>(smem_raw);      // [q][nwarps]: lane 31 value, c_x = +1 dirs
  const int nwarps = int(blockDim.x) >> 5;
  T* carry_dn = carry_up + L::q * nwarps;            // [q][nwarps]: lane 0 value, c_x = -1 dirs
  const int j = int(blockIdx.y);
  const int kb = d.k0 + int(blockIdx.z) * kz;
  const int ke = min(kb + kz, d.k0 + d.nzr);
  const int tid = int(threadIdx.x);
  const int lane = tid & 31, warp = tid >> 5;
  const int i0 = tid * VX;
  const int64_t mrow = int64_t(d.nx) * j + i0;
  const bool yedge = (j == 0 && d.mode[YMin] != kGhost) || (j == d.ny - 1 && d.mode[YMax] != kGhost);

  T cur[NM][VX], nxt[NM][VX];
  auto fetch = [&](T (&buf)[NM][VX], int k) {
    const int64_t mi = mrow + int64_t(k) * d.plane;
#pragma unroll
    for (int c = 0; c < NM; ++c) Vec<T, VX>::load(mo + c * d.mstride + mi, buf[c]);
  };
  fetch(cur, kb);
#pragma unroll 1
  for (int k = kb; k < ke; ++k) {
    if (k + 1 < ke) fetch(nxt, k + 1);
    NodeMoments<C> m[VX];
    bool exact = false;
#pragma unroll
    for (int x = 0; x < VX; ++x) {
      if constexpr (L::dim == 3)
        m[x] = prepare_node<C>(C(cur[0][x]), C(cur[1][x]), C(cur[2][x]), C(cur[3][x]), C(cur[4][x]),
                               C(cur[5][x]), C(cur[6][x]), C(cur[7][x]), C(cur[8][x]), C(cur[9][x]));
      else
        m[x] = prepare_node<C>(C(cur[0][x]), C(cur[1][x]), C(cur[2][x]), C(0), C(cur[3][x]), C(cur[4][x]),
                               C(0), C(cur[5][x]), C(0), C(0));
      exact |= (m[x].rho == C(0) && signbit(m[x].rho)) || m[x].pxx == C(0) || m[x].pyy == C(0) ||
               (L::dim == 3 && m[x].pzz == C(0));
    }
    const int64_t mi = mrow + int64_t(k) * d.plane;
    const int64_t fi = mi + int64_t(d.ghost) * d.plane;
    const bool zedge = (k == 0 && d.mode[ZMin] != kGhost) || (k == d.nz - 1 && d.mode[ZMax] != kGhost);
    if (yedge || zedge) {
      // general per-lane path (wrap / wall rows), reference evaluation order
      const RowGeom g = row_geom(d, j, k);
      const bool seg_start = lane == 0;
      const bool seg_end = lane == 31;
      all_dirs<L, T, C, VX, true, true>(d, f, g, fi, i0, true, seg_start, seg_end, m, om1);
      __syncthreads();  // keep the CTA in step (smem reuse below)
    } else {
      T o[L::q][VX];
      if (__syncthreads_or(exact))
        row_outputs<L, T, C, VX, true>(m, om1, o);
      else
        row_outputs<L, T, C, VX, false>(m, om1, o);
      // publish warp-edge values of the x-shifted directions
      unroll<L::q>([&](auto A) {
        constexpr int a = decltype(A)::value;
        if constexpr (Dir<L, a>::x == 1) {
          if (lane == 31) carry_up[a * nwarps + warp] = o[a][VX - 1];
        } else if constexpr (Dir<L, a>::x == -1) {
          if (lane == 0) carry_dn[a * nwarps + warp] = o[a][0];
        }
      });
      __syncthreads();
      unsigned char* rowp = reinterpret_cast<unsigned char*>(f + fi);
      unroll<L::q>([&](auto A) {
        constexpr int a = decltype(A)::value;
        using dd = Dir<L, a>;
        T* dst = reinterpret_cast<T*>(rowp + ro.off[a]);
        if constexpr (dd::x == 0) {
          Vec<T, VX>::st(dst, o[a]);
        } else if constexpr (dd::x == 1) {
          // slot x0 receives node x0 - 1
          T c = __shfl_up_sync(0xffffffffu, o[a][VX - 1], 1);
          if (lane == 0) {
            if (warp > 0) c = carry_up[a * nwarps + warp - 1];
            else if constexpr (XWALL)  // x = 0: bounce of opp(a) at node 0
              c = bounce_value<L, dd::opp, T, C>(d, o[dd::opp][0], true, false, false);
            else c = carry_up[a * nwarps + nwarps - 1];  // periodic: node nx - 1
          }
          T v[VX];
          v[0] = c;
#pragma unroll
          for (int e = 1; e < VX; ++e) v[e] = o[a][e - 1];
          Vec<T, VX>::st(dst, v);
        } else {
          // slot x0 + VX - 1 receives node x0 + VX
          T c = __shfl_down_sync(0xffffffffu, o[a][0], 1);
          if (lane == 31) {
            if (warp < nwarps - 1) c = carry_dn[a * nwarps + warp + 1];
            else if constexpr (XWALL)  // x = nx - 1: bounce of opp(a) at node nx - 1
              c = bounce_value<L, dd::opp, T, C>(d, o[dd::opp][VX - 1], true, false, false);
            else c = carry_dn[a * nwarps];  // periodic: node 0
          }
          T v[VX];
#pragma unroll
          for (int e = 0; e < VX - 1; ++e) v[e] = o[a][e + 1];
          v[VX - 1] = c;
          Vec<T, VX>::st(dst, v);
        }
      });
      __syncthreads();  // carries are rewritten by the next plane
    }
#pragma unroll
    for (int c = 0; c < NM; ++c)
#pragma unroll
      for (int x = 0; x < VX; ++x) cur[c][x] = nxt[c][x];
  }
}

/// Returns 1 (not launched) when the row does not fit one CTA.
template <typename T>
int launch_streamcoll_row(int lat, int math, const Dom& d0, T* f, const T* mo, double omega, int vx, int kz,
                          cudaStream_t st) {
  if (vx == 0) vx = 2;
  if (kz <= 0) kz = 8;
  if (vx * int(sizeof(T)) > 16 || d0.nx % vx != 0) return 1;
  const int threads = d0.nx / vx;
  if (threads % 32 != 0 || threads > kMaxRowThreads || d0.ny > 65535) return 1;
  // x faces: both periodic or both walls (classify rule); only no-slip x
  // walls are folded into the carries, moving x walls use the other kernels
  const bool xwall = d0.mode[XMin] == kWall;
  if (xwall && (d0.uw[XMin][0] != 0 || d0.uw[XMin][1] != 0 || d0.uw[XMin][2] != 0 || d0.uw[XMax][0] != 0 ||
                d0.uw[XMax][1] != 0 || d0.uw[XMax][2] != 0))
    return 1;
  const int nzc = (d0.nzr + kz - 1) / kz;
  if (nzc > 65535) return 1;
  const double om1d = 1.0 - double(T(omega));
  const float om1f = 1.0f - float(omega);
  int rc = 1;
  auto go = [&](auto L, auto V) {
    using Lat = decltype(L);
    constexpr int VX = decltype(V)::value;
    if constexpr (VX * sizeof(T) <= 16) {
      RowOffsets ro{};
      for (int a = 0; a < Lat::q; ++a)
        ro.off[a] = (int64_t(a) * d0.fstride +
                     int64_t(d0.nx) * (Lat::c[a][1] + int64_t(d0.ny) * Lat::c[a][2])) * int64_t(sizeof(T));
      const dim3 grid(1, unsigned(d0.ny), unsigned(nzc));
      const size_t sm = size_t(2) * Lat::q * (threads / 32) * sizeof(T);
      auto launch = [&](auto kern, auto om) {
        kern<<<grid, threads, sm, st>>>(d0, f, mo, om, kz, ro);
        rc = 0;
      };
      if (math == kMathDouble) {
        if (xwall) launch(k_streamcoll_row<Lat, T, double, VX, true>, om1d);
        else launch(k_streamcoll_row<Lat, T, double, VX, false>, om1d);
      } else {
        if (xwall) launch(k_streamcoll_row<Lat, T, float, VX, true>, om1f);
        else launch(k_streamcoll_row<Lat, T, float, VX, false>, om1f);
      }
    }
  };
  auto by_vx = [&](auto L) {
    if (vx == 2) go(L, std::integral_constant<int, 2>{});
    else if (vx == 4) go(L, std::integral_constant<int, 4>{});
  };
  switch (lat) {
    case kD2Q9: by_vx(D2Q9{}); break;
    case kD3Q19: by_vx(D3Q19{}); break;
    case kD3Q27: by_vx(D3Q27{}); break;
    default: return 1;
  }
  return rc;
}

template int launch_streamcoll_row<float>(int, int, const Dom&, float*, const float*, double, int, int, cudaStream_t);
template int launch_streamcoll_row<double>(int, int, const Dom&, double*, const double*, double, int, int,
                                           cudaStream_t);

}  // namespace tslb_cuda
