// Moment-resident single-pass step ("M" schedule) for
// 3-D box geometries (periodic faces and walls, no solid mask).
//
// The F1 schedule (k_moments + k_streamcoll) moves the populations through
// HBM twice per step: 2 (q + 1 + D + np) scalars per lattice update. Here the
// populations never leave the SM: one kernel reads m(t) -- the 1 + D + np
// moment arrays of the pre-step state -- and writes m(t+1):
//
//   1. each node x of the tile (and of a one-node ring around it) rebuilds
//      its post-collision populations pc_a(m(x)) -- the regularised
//      collision of stream_collide_fused, kernels.hpp:154-204, in the
//      reference's operand order -- rounds them to the storage type T and
//      pushes them into the shared-memory slot of x + c_a (bounce-back on
//      walls writes the node's own opposite slot, kernels.hpp:178-199);
//   2. after a barrier, every node of the tile gathers its q slots in
//      direction order and reduces them to m(t+1) exactly as
//      compute_moments does (kernels.hpp:74-107, double accumulation).
//
// So each slot still has exactly one writer, the populations are rounded
// to T exactly where the reference stores them, and the moment sums see the
// same values in the same order: m(t+1) is bit-identical to the moments of
// the reference's f(t+1). The host-visible f(t+1) is never stored; the
// C-ABI materialises it on demand with one stream-collide launch from m(t)
// (the moment arrays the reference leaves behind after a step, solver.hpp:
// 68-69), so every API reads the same bits as after F1.
//
// Shape: a CTA owns a 32 x 8 column tile and marches through LZ planes
// (2.5-D blocking). Moments of plane z+1 are staged with cp.async while
// plane z is collided; slots live in per-direction plane rings sized by the
// direction's c_z (a slot of destination plane d is written while the march
// is at plane d - c_z, or at d for a bounce, and read at plane d + 1), so a
// single __syncthreads per plane orders every write before its read. Pure-z
// and rest directions never leave the thread: they ride a register ring.
// Ring nodes outside the tile (one-node x/y halo, the planes just below and
// above the march) only rebuild the directions that land inside the tile;
// they never bounce (a push that lands in the tile cannot cross a wall).
//
// HBM traffic per lattice update: 2 (1 + D + np) scalars = 80 B (D3Q19 fp32)
// instead of 232 B, plus ~1/LZ of a plane of halo re-reads.
//
// The pair rewrite of the collision (tslb_pair.cuh) differs from the
// reference order only for rho == -0.0; the moments this kernel reads are
// always produced by a +0-seeded sum (k_moments or this kernel), which
// cannot return -0.0, so the rewrite is exact here.
#include <cuda_pipeline.h>

#include <cstdint>

#include "tslb_collision.cuh"
#include "tslb_domain.cuh"
#include "tslb_kernels.h"
#include "tslb_pair.cuh"

namespace tslb_cuda {
namespace mstep {

constexpr int TX = 32;                     // tile width (one warp per row)
constexpr int TY = 8;                      // tile rows (warps per CTA)
constexpr int NT = TX * TY;                // threads = tile columns
constexpr int NH = 2 * TX + 2 * TY + 4;    // halo ring nodes
constexpr int NS = NT + NH;                // staged nodes per plane

template <class L>
__host__ __device__ constexpr bool is_reg(int a) {
  return L::c[a][0] == 0 && L::c[a][1] == 0;
}
// plane-ring depth of slot direction a (see header): 4 for c_z = +1, else 3
template <class L>
__host__ __device__ constexpr int ring_depth(int a) {
  return L::c[a][2] == 1 ? 4 : 3;
}
template <class L>
__host__ __device__ constexpr int slot_base(int a) {
  int s = 0;
  for (int b = 0; b < a; ++b)
    if (!is_reg<L>(b)) s += ring_depth<L>(b);
  return s;
}
template <class L>
__host__ __device__ constexpr int slot_planes() {
  return slot_base<L>(L::q);
}
template <class L>
__host__ __device__ constexpr int n_moments() {
  return 1 + L::dim + L::dim * (L::dim + 1) / 2;
}
template <class L, typename T>
constexpr size_t smem_bytes() {
  return (size_t(slot_planes<L>()) * NT + size_t(2) * n_moments<L>() * NS) * sizeof(T);
}

// coordinate after crossing a face: wrapped (periodic) or -1 (wall: absent)
__device__ __forceinline__ int wrap_coord(int g, int n, int lo, int hi) {
  if (g < 0) return lo == kWrap ? g + n : -1;
  if (g >= n) return hi == kWrap ? g - n : -1;
  return g;
}

// ring offsets (in elements) of destination planes z-1, z, z+1 relative to
// the plane being pushed, for 3- and 4-deep rings
struct Ring {
  int o3[3], o4[3];
  int p3, p4;
  __device__ __forceinline__ void set() {
    o3[0] = (p3 == 0 ? 2 : p3 - 1) * NT;
    o3[1] = p3 * NT;
    o3[2] = (p3 == 2 ? 0 : p3 + 1) * NT;
    o4[0] = ((p4 + 3) & 3) * NT;
    o4[1] = p4 * NT;
    o4[2] = ((p4 + 1) & 3) * NT;
  }
  __device__ __forceinline__ void advance() {
    p3 = p3 == 2 ? 0 : p3 + 1;
    p4 = (p4 + 1) & 3;
    set();
  }
};

template <class L, int A, int DZ, typename T>
__device__ __forceinline__ T* slot(T* sl, const Ring& rg, int lx, int ly) {
  constexpr int base = slot_base<L>(A) * NT;
  const int ro = ring_depth<L>(A) == 4 ? rg.o4[DZ + 1] : rg.o3[DZ + 1];
  return sl + base + ro + ly * TX + lx;
}

template <class L, typename T, typename C>
__device__ __forceinline__ NodeMoments<C> staged_node(const T* s, int node) {
  constexpr int NM = n_moments<L>();
  T v[NM];
#pragma unroll
  for (int c = 0; c < NM; ++c) v[c] = s[c * NS + node];
  if constexpr (L::dim == 3)
    return prepare_node<C>(C(v[0]), C(v[1]), C(v[2]), C(v[3]), C(v[4]), C(v[5]),
                           C(v[6]), C(v[7]), C(v[8]), C(v[9]));
  else
    return prepare_node<C>(C(v[0]), C(v[1]), C(v[2]), C(0), C(v[3]), C(v[4]), C(0),
                           C(v[5]), C(0), C(0));
}

// per-thread wall contact of the tile node (only for WALLS kernels)
struct Contact {
  bool xlo, xhi, ylo, yhi, zlo, zhi;
};

// Output of direction A from a tile node: bounce into its own opposite slot
// or push into the slot of the destination (dropped if outside the tile).
template <class L, int A, typename T, typename C, bool WALLS, int ZC>
__device__ __forceinline__ void emit(const Dom& d, T* sl, const Ring& rg, T (&R)[L::q][3],
                                     int lx, int ly, const Contact& ct, T o) {
  using dd = Dir<L, A>;
  if constexpr (WALLS && ZC == 0) {
    const bool cx = (dd::x == 1 && ct.xhi) || (dd::x == -1 && ct.xlo);
    const bool cy = (dd::y == 1 && ct.yhi) || (dd::y == -1 && ct.ylo);
    const bool cz = (dd::z == 1 && ct.zhi) || (dd::z == -1 && ct.zlo);
    if (cx || cy || cz) {
      const T b = bounce_value<L, A, T, C>(d, o, cx, cy, cz);
      if constexpr (is_reg<L>(dd::opp)) R[dd::opp][1] = b;
      else *slot<L, dd::opp, 0>(sl, rg, lx, ly) = b;
      return;
    }
  }
  if constexpr (is_reg<L>(A)) {
    R[A][1 + dd::z] = o;
  } else {
    const int tx = lx + dd::x, ty = ly + dd::y;
    bool in = true;
    if constexpr (dd::x != 0) in = unsigned(tx) < unsigned(TX);
    if constexpr (dd::y != 0) in = in && unsigned(ty) < unsigned(TY);
    if (in) *slot<L, A, dd::z>(sl, rg, tx, ty) = o;
  }
}

// All directions of a tile node; ZC != 0 (a plane just outside the march)
// keeps only the directions with c_z == ZC.
template <class L, typename T, typename C, bool WALLS, int ZC>
__device__ __forceinline__ void push_tile(const Dom& d, T* sl, const Ring& rg, T (&R)[L::q][3],
                                          int lx, int ly, const Contact& ct,
                                          const NodeMoments<C>& m, C om1) {
  unroll<L::q>([&](auto A) {
    constexpr int a = decltype(A)::value;
    if constexpr (a == 0) {
      if constexpr (ZC == 0) emit<L, 0, T, C, WALLS, ZC>(d, sl, rg, R, lx, ly, ct, T(post_rest<L, C>(m, om1)));
    } else if constexpr (a & 1) {
      constexpr bool ua = ZC == 0 || Dir<L, a>::z == ZC;
      constexpr bool ub = ZC == 0 || Dir<L, a + 1>::z == ZC;
      if constexpr (ua && ub) {
        C ra, rb;
        post_pair<L, a, C>(m, om1, ra, rb);
        emit<L, a, T, C, WALLS, ZC>(d, sl, rg, R, lx, ly, ct, T(ra));
        emit<L, a + 1, T, C, WALLS, ZC>(d, sl, rg, R, lx, ly, ct, T(rb));
      } else if constexpr (ua) {
        emit<L, a, T, C, WALLS, ZC>(d, sl, rg, R, lx, ly, ct, T(post_collision<L, a, C>(m, om1)));
      } else if constexpr (ub) {
        emit<L, a + 1, T, C, WALLS, ZC>(d, sl, rg, R, lx, ly, ct, T(post_collision<L, a + 1, C>(m, om1)));
      }
    }
  });
}

// A halo node at tile-local (hx, hy) on side (SX, SY): only the directions
// pointing into the tile, reference order (no pair partner is needed).
template <class L, typename T, typename C, int SX, int SY, int ZC>
__device__ __forceinline__ void push_halo(T* sl, const Ring& rg, int hx, int hy,
                                          const NodeMoments<C>& m, C om1) {
  unroll<L::q>([&](auto A) {
    constexpr int a = decltype(A)::value;
    using dd = Dir<L, a>;
    constexpr bool use = !is_reg<L>(a) && (SX == 0 || dd::x == -SX) &&
                         (SY == 0 || dd::y == -SY) && (ZC == 0 || dd::z == ZC);
    if constexpr (use) {
      const int tx = hx + dd::x, ty = hy + dd::y;
      bool in = true;
      if constexpr (SX == 0 && dd::x != 0) in = unsigned(tx) < unsigned(TX);
      if constexpr (SY == 0 && dd::y != 0) in = in && unsigned(ty) < unsigned(TY);
      if (in) *slot<L, a, dd::z>(sl, rg, tx, ty) = T(post_collision<L, a, C>(m, om1));
    }
  });
}

template <class L, typename T, typename C, int ZC>
__device__ __forceinline__ void push_ring(T* sl, const Ring& rg, int role, int hx, int hy,
                                          const NodeMoments<C>& m, C om1) {
  switch (role) {
    case 0: push_halo<L, T, C, 0, -1, ZC>(sl, rg, hx, hy, m, om1); break;
    case 1: push_halo<L, T, C, 0, 1, ZC>(sl, rg, hx, hy, m, om1); break;
    case 2: push_halo<L, T, C, -1, 0, ZC>(sl, rg, hx, hy, m, om1); break;
    case 3: push_halo<L, T, C, 1, 0, ZC>(sl, rg, hx, hy, m, om1); break;
    case 4: push_halo<L, T, C, -1, -1, ZC>(sl, rg, hx, hy, m, om1); break;
    case 5: push_halo<L, T, C, 1, -1, ZC>(sl, rg, hx, hy, m, om1); break;
    case 6: push_halo<L, T, C, -1, 1, ZC>(sl, rg, hx, hy, m, om1); break;
    default: push_halo<L, T, C, 1, 1, ZC>(sl, rg, hx, hy, m, om1); break;
  }
}

// compute_moments of one node from its gathered slots (kernels.hpp:74-107;
// same accumulation order and formulae as k_moments)
template <class L, typename T, typename C>
__device__ __forceinline__ void finalize(const Dom& d, T* sl, const Ring& rg, const T (&R)[L::q][3],
                                         int lx, int ly, T* __restrict__ mo, int64_t idx) {
  C r = 0, jx = 0, jy = 0, jz = 0, pxx = 0, pyy = 0, pzz = 0, pxy = 0, pxz = 0, pyz = 0;
  unroll<L::q>([&](auto A) {
    constexpr int a = decltype(A)::value;
    using dd = Dir<L, a>;
    T v;
    if constexpr (is_reg<L>(a)) v = R[a][0];
    else v = *slot<L, a, -1>(sl, rg, lx, ly);
    const C fa = C(v);
    r += fa;
    if constexpr (dd::x == 1) jx += fa;
    if constexpr (dd::x == -1) jx -= fa;
    if constexpr (dd::y == 1) jy += fa;
    if constexpr (dd::y == -1) jy -= fa;
    if constexpr (dd::z == 1) jz += fa;
    if constexpr (dd::z == -1) jz -= fa;
    if constexpr (dd::x != 0) pxx += fa;
    if constexpr (dd::y != 0) pyy += fa;
    if constexpr (dd::z != 0) pzz += fa;
    if constexpr (dd::x * dd::y == 1) pxy += fa;
    if constexpr (dd::x * dd::y == -1) pxy -= fa;
    if constexpr (dd::x * dd::z == 1) pxz += fa;
    if constexpr (dd::x * dd::z == -1) pxz -= fa;
    if constexpr (dd::y * dd::z == 1) pyz += fa;
    if constexpr (dd::y * dd::z == -1) pyz -= fa;
  });
  const C c3 = cs2<C>();
  const int64_t ms = d.mstride;
  mo[idx] = T(r);
  mo[ms + idx] = T(jx);
  mo[2 * ms + idx] = T(jy);
  mo[3 * ms + idx] = T(jz);
  mo[4 * ms + idx] = T(pxx - c3 * r - jx * jx);
  mo[5 * ms + idx] = T(pyy - c3 * r - jy * jy);
  mo[6 * ms + idx] = T(pzz - c3 * r - jz * jz);
  mo[7 * ms + idx] = T(pxy - jx * jy);
  mo[8 * ms + idx] = T(pxz - jx * jz);
  mo[9 * ms + idx] = T(pyz - jy * jz);
}

template <class L, typename T, typename C, bool WALLS>
__global__ void __launch_bounds__(NT, 2)
    k_mstep(Dom d, const T* __restrict__ mi, T* __restrict__ mo, C om1, int lz) {
  static_assert(L::dim == 3, "the M step is 3-D");
  constexpr int NM = n_moments<L>();
  extern __shared__ __align__(16) unsigned char smraw[];
  T* sl = reinterpret_cast<T*>(smraw);
  T* stg = sl + slot_planes<L>() * NT;  // [2][NM][NS] staged moments

  const int tid = threadIdx.x, lx = tid & (TX - 1), ly = tid >> 5;
  const int x0 = int(blockIdx.x) * TX, y0 = int(blockIdx.y) * TY;
  const int za = int(blockIdx.z) * lz, zb = min(za + lz, d.nz);
  const int gx = x0 + lx, gy = y0 + ly;
  const int64_t col = gx + int64_t(d.nx) * gy;

  // halo role of this thread: warp 0 the row below the tile, warp 1 the row
  // above, warps 2/3 the columns left/right, warp 4 the four corners
  int hnode = -1, role = 0, hx = 0, hy = 0;
  if (ly == 0) { hnode = lx; role = 0; hx = lx; hy = -1; }
  else if (ly == 1) { hnode = TX + lx; role = 1; hx = lx; hy = TY; }
  else if (ly == 2 && lx < TY) { hnode = 2 * TX + lx; role = 2; hx = -1; hy = lx; }
  else if (ly == 3 && lx < TY) { hnode = 2 * TX + TY + lx; role = 3; hx = TX; hy = lx; }
  else if (ly == 4 && lx < 4) {
    hnode = 2 * TX + 2 * TY + lx;
    role = 4 + lx;
    hx = (lx & 1) ? TX : -1;
    hy = (lx & 2) ? TY : -1;
  }
  int64_t hcol = 0;
  if (hnode >= 0) {
    const int hgx = wrap_coord(x0 + hx, d.nx, d.mode[XMin], d.mode[XMax]);
    const int hgy = wrap_coord(y0 + hy, d.ny, d.mode[YMin], d.mode[YMax]);
    if (hgx < 0 || hgy < 0) hnode = -1;
    else hcol = hgx + int64_t(d.nx) * hgy;
  }
  Contact ct{};
  if constexpr (WALLS) {
    ct.xlo = gx == 0 && d.mode[XMin] == kWall;
    ct.xhi = gx == d.nx - 1 && d.mode[XMax] == kWall;
    ct.ylo = gy == 0 && d.mode[YMin] == kWall;
    ct.yhi = gy == d.ny - 1 && d.mode[YMax] == kWall;
  }

  auto issue = [&](int z, int buf) {
    const int zz = wrap_coord(z, d.nz, d.mode[ZMin], d.mode[ZMax]);
    if (zz < 0) return;
    T* s = stg + buf * NM * NS;
    const int64_t pl = int64_t(zz) * d.plane;
#pragma unroll
    for (int c = 0; c < NM; ++c)
      __pipeline_memcpy_async(s + c * NS + tid, mi + c * d.mstride + pl + col, sizeof(T));
    if (hnode >= 0) {
#pragma unroll
      for (int c = 0; c < NM; ++c)
        __pipeline_memcpy_async(s + c * NS + NT + hnode, mi + c * d.mstride + pl + hcol, sizeof(T));
    }
  };

  T R[L::q][3];
#pragma unroll
  for (int a = 0; a < L::q; ++a) R[a][0] = R[a][1] = R[a][2] = T(0);
  Ring rg;
  rg.p3 = 0;
  rg.p4 = 0;
  rg.set();
  int buf = 0;

  auto plane = [&](auto ZCc, int z) {
    constexpr int ZC = decltype(ZCc)::value;
    if (ZC != -1) issue(z + 1, buf ^ 1);
    __pipeline_commit();
    __pipeline_wait_prior(1);
    if (wrap_coord(z, d.nz, d.mode[ZMin], d.mode[ZMax]) >= 0) {
      const T* s = stg + buf * NM * NS;
      if constexpr (WALLS) {
        ct.zlo = z == 0 && d.mode[ZMin] == kWall;
        ct.zhi = z == d.nz - 1 && d.mode[ZMax] == kWall;
      }
      const NodeMoments<C> m = staged_node<L, T, C>(s, tid);
      push_tile<L, T, C, WALLS, ZC>(d, sl, rg, R, lx, ly, ct, m, om1);
      if (hnode >= 0) {
        const NodeMoments<C> hm = staged_node<L, T, C>(s, NT + hnode);
        push_ring<L, T, C, ZC>(sl, rg, role, hx, hy, hm, om1);
      }
    }
    __syncthreads();
    if (z - 1 >= za)
      finalize<L, T, C>(d, sl, rg, R, lx, ly, mo, col + int64_t(z - 1) * d.plane);
#pragma unroll
    for (int a = 0; a < L::q; ++a) {
      R[a][0] = R[a][1];
      R[a][1] = R[a][2];
    }
    rg.advance();
    buf ^= 1;
  };

  issue(za - 1, 0);
  __pipeline_commit();
  plane(std::integral_constant<int, 1>{}, za - 1);
#pragma unroll 1
  for (int z = za; z < zb; ++z) plane(std::integral_constant<int, 0>{}, z);
  plane(std::integral_constant<int, -1>{}, zb);
}

}  // namespace mstep

bool mstep_supported(int lat, const Dom& d) {
  return (lat == kD3Q19 || lat == kD3Q27) && !d.has_solid && d.ghost == 0 &&
         d.nx % mstep::TX == 0 && d.ny % mstep::TY == 0;
}

template <typename T>
int launch_mstep(int lat, int math, const Dom& d, const T* mi, T* mo, double omega,
                 int lz, cudaStream_t st) {
  using namespace mstep;
  if (!mstep_supported(lat, d)) return 1;
  if (lz <= 0) lz = 32;
  bool walls = false;
  for (int fc = 0; fc < 6; ++fc) walls |= d.mode[fc] == kWall;
  const dim3 grid(unsigned(d.nx / TX), unsigned(d.ny / TY), unsigned((d.nz + lz - 1) / lz));
  if (grid.y > 65535 || grid.z > 65535) return 1;
  const double om1d = 1.0 - double(T(omega));
  const float om1f = 1.0f - float(omega);
  auto go = [&](auto L, auto kern, auto om1) {
    using Lat = decltype(L);
    constexpr size_t smem = smem_bytes<Lat, T>();
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    kern<<<grid, NT, smem, st>>>(d, mi, mo, om1, lz);
  };
  auto by_lat = [&](auto L) {
    using Lat = decltype(L);
    if (math == kMathDouble) {
      if (walls) go(L, k_mstep<Lat, T, double, true>, om1d);
      else go(L, k_mstep<Lat, T, double, false>, om1d);
    } else {
      if (walls) go(L, k_mstep<Lat, T, float, true>, om1f);
      else go(L, k_mstep<Lat, T, float, false>, om1f);
    }
  };
  if (lat == kD3Q19) by_lat(D3Q19{});
  else by_lat(D3Q27{});
  return 0;
}

template int launch_mstep<float>(int, int, const Dom&, const float*, float*, double, int, cudaStream_t);
template int launch_mstep<double>(int, int, const Dom&, const double*, double*, double, int, cudaStream_t);

}  // namespace tslb_cuda
