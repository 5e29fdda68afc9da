// Moment-resident single-pass step ("M" schedule) for
// 3-D grids: periodic faces, walls, slab ghost faces and (SOLID kernels)
// solid masks.
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
// (2.5-D blocking). The moments of plane z+1 -- all 1+D+np arrays of the
// tile plus the rows just below and above it -- arrive by ONE TMA tensor
// load (cp.async.bulk.tensor, 4-D box, mbarrier completion) while plane z
// is collided; the x-halo columns and wrapped rows come in by cp.async.
// Slots live in per-direction plane rings sized by the direction's c_z (a
// slot of destination plane d is written while the march is at plane
// d - c_z, or at d for a bounce, and read after the march passed d): two
// barriers per plane, or one with rings a plane deeper (SL<L, 1>). Pure-z
// and rest directions never leave the thread: they ride a register ring.
// Solid masks (SOLID): per-node solid bits (k_solid_bits) ride along with
// the moments; solid nodes push nothing and carry their moments through,
// a push towards a solid node is a bounce (see emit).
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
#include <cuda.h>
#include <cuda_pipeline.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "tslb_collision.cuh"
#include "tslb_domain.cuh"
#include "tslb_kernels.h"
#include "tslb_msums.cuh"
#include "tslb_pair.cuh"
#include "tslb_store16.cuh"
#include "tslb_async.cuh"

namespace tslb_cuda {

// encoded tensor maps of the moment buffers used as M-step inputs
struct MstepMaps {
  struct Entry {
    CUtensorMap map;
    const void* base = nullptr;
    int64_t key[5] = {0, 0, 0, 0, 0};
  } e[3];  // the two moment buffers (ping-pong) and the slab ghost planes
  int next = 0;
};
void free_mstep_maps(MstepMaps* m) { delete m; }

namespace mstep {

constexpr int TX = 32;                     // tile width (one warp per row)
#ifndef TSLB_TY
#define TSLB_TY 8
#endif
constexpr int TY = TSLB_TY;                // tile rows (warps per CTA; -DTSLB_TY: measurements)
constexpr int NT = TX * TY;                // threads = tile columns
constexpr int NH = 2 * TX + 2 * (TY + 2);  // halo ring nodes (x columns include the corners)
constexpr int TR = TY + 2;                 // staged tile rows (with y halo)
constexpr int TC = TR * TX;                // staged elements per moment array
// planes marched per CTA: the march re-reads one halo plane below and above
// per column, so longer columns amortise it; s28 sweep at 1024^3 (fp64 math,
// same box): 32 / 64 / 128 / 256 / 512 -> 33.3 / 33.9 / 34.1 / 34.1-34.2 /
// 33.7 GLUPS, D3Q27 channel 64 / 128 / 256 -> 20.56 / 20.61 / 20.73; fp32
// node math 64 / 128 -> 44.1-44.3 / 44.9
constexpr int kDefaultLz = 128;

template <class L>
__host__ __device__ constexpr bool is_reg(int a) {
  return L::c[a][0] == 0 && L::c[a][1] == 0;
}
// Lattice L with the slot-ring variant RD: 0 = two barriers per plane
// (rings 2 / 3 deep, least shared memory), 1 = one barrier per plane (rings
// 3 / 4 deep: a slot of plane d may then be rewritten only after every warp
// has passed the NEXT plane's barrier).
template <class B, int RD>
struct SL : B {
  static constexpr int rd = RD;
};
// plane-ring depth of slot direction a: (3 for c_z = +1, else 2) + rd
template <class L>
__host__ __device__ constexpr int ring_depth(int a) {
  return (L::c[a][2] == 1 ? 3 : 2) + L::rd;
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
__host__ __device__ constexpr size_t align128(size_t b) { return (b + 127) / 128 * 128; }

// dynamic shared memory: [tile buf 0 | tile buf 1 | wstg 0 | wstg 1 | slots | mbarriers]
template <class L, typename T, bool SOLID = false, typename TM = T>
struct Smem {
  static constexpr size_t tile = align128(size_t(n_moments<L>()) * TC * sizeof(TM));
  // one copy of the ring per halo task half (see push_ring)
  static constexpr size_t wstg = align128(size_t(n_moments<L>()) * 2 * NH * sizeof(typename MStore<TM>::W));
  static constexpr size_t slots = size_t(slot_planes<L>()) * NT * sizeof(T);
  // solid geometries: the per-node solid bits of the tile and of the halo
  // ring (cp.async, double buffered) -- [2][NT + 2 NH] u32
  static constexpr size_t bits = SOLID ? align128(size_t(2) * (NT + 2 * NH) * 4) : 0;
  static constexpr size_t off_wstg = 2 * tile;
  static constexpr size_t off_slots = off_wstg + 2 * wstg;
  static constexpr size_t off_bits = align128(off_slots + slots);
  static constexpr size_t off_bar = align128(off_bits + bits);
  static constexpr size_t total = off_bar + 2 * sizeof(uint64_t);
};

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

// coordinate after crossing a face: wrapped (periodic) or -1 (wall: absent)
__device__ __forceinline__ int wrap_coord(int g, int n, int lo, int hi) {
  if (g < 0) return lo == kWrap ? g + n : -1;
  if (g >= n) return hi == kWrap ? g - n : -1;
  return g;
}

// Where the moments of plane z (possibly outside [0, nz)) come from:
// 0 nowhere (beyond a wall), 1 an owned plane zz (wrapped if periodic),
// 2 the slab ghost plane zz (0 below, 1 above) received from a neighbour.
__device__ __forceinline__ int plane_src(const Dom& d, int z, int& zz) {
  if (z >= 0 && z < d.nz) {
    zz = z;
    return 1;
  }
  const int face = z < 0 ? ZMin : ZMax;
  if (d.mode[face] == kWrap) {
    zz = z < 0 ? z + d.nz : z - d.nz;
    return 1;
  }
  if (d.mode[face] == kGhost) {
    zz = z < 0 ? 0 : 1;
    return 2;
  }
  return 0;
}

// Shared-memory slot accesses as single instructions: 32-bit shared
// address + compile-time byte offset; the guarded store is one predicated
// st.shared (the compiler otherwise wraps each guarded store in a
// reconvergence region).
template <typename T>
struct Shm;
template <>
struct Shm<float> {
  template <int OFF>
  __device__ static __forceinline__ void st(uint32_t a, float v) {
    asm volatile("st.shared.f32 [%0+%2], %1;" ::"r"(a), "f"(v), "n"(OFF) : "memory");
  }
  template <int OFF>
  __device__ static __forceinline__ void st_if(uint32_t a, float v, bool p) {
    asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q st.shared.f32 [%0+%3], %1;\n}" ::"r"(a), "f"(v),
                 "r"(int(p)), "n"(OFF)
                 : "memory");
  }
  template <int OFF>
  __device__ static __forceinline__ float ld(uint32_t a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1+%2];" : "=f"(v) : "r"(a), "n"(OFF) : "memory");
    return v;
  }
};
template <>
struct Shm<double> {
  template <int OFF>
  __device__ static __forceinline__ void st(uint32_t a, double v) {
    asm volatile("st.shared.f64 [%0+%2], %1;" ::"r"(a), "d"(v), "n"(OFF) : "memory");
  }
  template <int OFF>
  __device__ static __forceinline__ void st_if(uint32_t a, double v, bool p) {
    asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q st.shared.f64 [%0+%3], %1;\n}" ::"r"(a), "d"(v),
                 "r"(int(p)), "n"(OFF)
                 : "memory");
  }
  template <int OFF>
  __device__ static __forceinline__ double ld(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1+%2];" : "=d"(v) : "r"(a), "n"(OFF) : "memory");
    return v;
  }
};

// Slot addressing. Each thread keeps the shared addresses of its own
// column's slot in the ring planes of destination planes z-1, z, z+1
// relative to the plane being pushed, for the shallow (DA) and deep (DA+1)
// rings; a push by (dx, dy) is then that address plus a compile-time offset.
template <class L, typename T>
struct Ring {
  static constexpr int DA = 2 + L::rd, DB = DA + 1;
  static constexpr uint32_t P = NT * sizeof(T);
  // qa[k] = address of ring plane (p + k - 1) mod DA: qa[0] holds destination
  // plane z-1, qa[1] plane z, qa[2 mod DA] plane z+1; advancing the march
  // rotates the array (register renames, no index arithmetic)
  uint32_t qa[DA], qb[DB];
  __device__ __forceinline__ void init(uint32_t own) {
#pragma unroll
    for (int k = 0; k < DA; ++k) qa[k] = own + uint32_t((k - 1 + DA) % DA) * P;
#pragma unroll
    for (int k = 0; k < DB; ++k) qb[k] = own + uint32_t((k - 1 + DB) % DB) * P;
  }
  __device__ __forceinline__ void advance() {
    const uint32_t ta = qa[0], tb = qb[0];
#pragma unroll
    for (int k = 0; k + 1 < DA; ++k) qa[k] = qa[k + 1];
    qa[DA - 1] = ta;
#pragma unroll
    for (int k = 0; k + 1 < DB; ++k) qb[k] = qb[k + 1];
    qb[DB - 1] = tb;
  }
};

// byte offset of direction A's slot shifted by (DX, DY) from the own column
template <class L, int A, int DX, int DY, typename T>
__host__ __device__ constexpr int slot_off() {
  return int((slot_base<L>(A) * NT + DY * TX + DX) * int(sizeof(T)));
}
template <class L, int A, int DZ, typename T>
__device__ __forceinline__ uint32_t ring_addr(const Ring<L, T>& rg) {
  constexpr int DA = Ring<L, T>::DA, DB = Ring<L, T>::DB;
  if constexpr (ring_depth<L>(A) == DB) return rg.qb[((DZ + 1) % DB + DB) % DB];
  else return rg.qa[((DZ + 1) % DA + DA) % DA];
}

template <class L, typename TM, typename C>
__device__ __forceinline__ NodeMoments<C> node_at(const TM* s, int stride) {
  constexpr int NM = n_moments<L>();
  C v[NM];
#pragma unroll
  for (int c = 0; c < NM; ++c) v[c] = C(MStore<TM>::dec(c, s[c * stride]));
  return prepare_node<C>(v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7], v[8], v[9]);
}

// a lane-fetched halo node: staged words (MStore<TM>::W), `sel` picks the
// half of a 2-byte element inside its aligned 4-byte word
template <class L, typename TM, typename C>
__device__ __forceinline__ NodeMoments<C> staged_at(const typename MStore<TM>::W* s, int stride, int sel) {
  constexpr int NM = n_moments<L>();
  C v[NM];
#pragma unroll
  for (int c = 0; c < NM; ++c) v[c] = C(MStore<TM>::dec(c, MStore<TM>::pick(s[c * stride], sel)));
  return prepare_node<C>(v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7], v[8], v[9]);
}

// per-thread wall contact of the tile node (only for WALLS kernels) and,
// for solid geometries, its solid bits (bit a: the push target of
// direction a is solid; bit 31: the node itself is solid)
struct Contact {
  bool xlo, xhi, ylo, yhi, zlo, zhi;
  uint32_t sb;
};
constexpr uint32_t kSelfSolid = 1u << 31;

// Output of direction A from a tile node: bounce into its own opposite slot
// or push into the slot of the destination (dropped if outside the tile).
template <class L, int A, typename T, typename C, bool WALLS, bool SOLID, int ZC>
__device__ __forceinline__ void emit(const Dom& d, const Ring<L, T>& rg, T (&R)[L::q][3],
                                     int lx, int ly, const Contact& ct, T o) {
  using dd = Dir<L, A>;
  if constexpr ((WALLS || SOLID) && ZC == 0) {
    // wall faces crossed (resolve_push, boundary.hpp:118-144), else a solid
    // target: both bounce into the node's own opposite slot
    const bool cx = WALLS && ((dd::x == 1 && ct.xhi) || (dd::x == -1 && ct.xlo));
    const bool cy = WALLS && ((dd::y == 1 && ct.yhi) || (dd::y == -1 && ct.ylo));
    const bool cz = WALLS && ((dd::z == 1 && ct.zhi) || (dd::z == -1 && ct.zlo));
    if (cx || cy || cz) {  // (spatially coherent: a branch)
      const T b = bounce_value<L, A, T, C>(d, o, cx, cy, cz);
      if constexpr (is_reg<L>(dd::opp)) R[dd::opp][1] = b;
      else Shm<T>::template st<slot_off<L, dd::opp, 0, 0, T>()>(ring_addr<L, dd::opp, 0>(rg), b);
      return;
    }
    if constexpr (SOLID) {
      // solid target, no wall crossed: the bounce is o itself (the wall
      // correction of u_w = 0 is +0 and o - (+0) == o for every o). The
      // scattered pattern is handled without branches: a predicated store
      // into the own opposite slot, and the regular push below also runs
      // (it lands in the solid target's slot, which is never reduced)
      const bool cs = (ct.sb >> A) & 1u;
      if constexpr (is_reg<L>(dd::opp)) R[dd::opp][1] = cs ? o : R[dd::opp][1];
      else Shm<T>::template st_if<slot_off<L, dd::opp, 0, 0, T>()>(ring_addr<L, dd::opp, 0>(rg), o, cs);
    }
  }
  if constexpr (is_reg<L>(A)) {
    R[A][1 + dd::z] = o;
  } else {
    const int tx = lx + dd::x, ty = ly + dd::y;
    bool in = true;
    if constexpr (dd::x != 0) in = unsigned(tx) < unsigned(TX);
    if constexpr (dd::y != 0) in = in && unsigned(ty) < unsigned(TY);
    if constexpr (dd::x == 0 && dd::y == 0) {
      Shm<T>::template st<slot_off<L, A, 0, 0, T>()>(ring_addr<L, A, dd::z>(rg), o);
    } else {
      Shm<T>::template st_if<slot_off<L, A, dd::x, dd::y, T>()>(ring_addr<L, A, dd::z>(rg), o, in);
    }
  }
}

// All directions of a tile node; ZC != 0 (a plane just outside the march)
// keeps only the directions with c_z == ZC.
template <class L, typename T, typename C, bool WALLS, bool SOLID, int ZC>
__device__ __forceinline__ void push_tile(const Dom& d, const Ring<L, T>& rg, T (&R)[L::q][3],
                                          int lx, int ly, const Contact& ct,
                                          const NodeMoments<C>& m, C om1) {
  unroll<L::q>([&](auto A) {
    constexpr int a = decltype(A)::value;
    if constexpr (a == 0) {
      if constexpr (ZC == 0) emit<L, 0, T, C, WALLS, SOLID, ZC>(d, rg, R, lx, ly, ct, T(sf_post<L, 0, C>(m, om1)));
    } else if constexpr (a & 1) {
      constexpr bool ua = ZC == 0 || Dir<L, a>::z == ZC;
      constexpr bool ub = ZC == 0 || Dir<L, a + 1>::z == ZC;
      if constexpr (ua && ub) {
        C ra, rb;
        sf_pair<L, a, C>(m, om1, ra, rb);
        emit<L, a, T, C, WALLS, SOLID, ZC>(d, rg, R, lx, ly, ct, T(ra));
        emit<L, a + 1, T, C, WALLS, SOLID, ZC>(d, rg, R, lx, ly, ct, T(rb));
      } else if constexpr (ua) {
        emit<L, a, T, C, WALLS, SOLID, ZC>(d, rg, R, lx, ly, ct, T(sf_post<L, a, C>(m, om1)));
      } else if constexpr (ub) {
        emit<L, a + 1, T, C, WALLS, SOLID, ZC>(d, rg, R, lx, ly, ct, T(sf_post<L, a + 1, C>(m, om1)));
      }
    }
  });
}

// Halo pushes. A halo node at tile-local (hx, hy) on side (SX, SY) only
// rebuilds the directions that land inside the tile. The four sides (x
// columns including the corners) are split into eight tasks of about equal
// cost -- side = warp / 2, and each of the two warps of a side takes every
// other of the side's directions -- so every warp reaches the barrier with
// the same work.
template <class L, int SX, int SY, int ZC>
__host__ __device__ constexpr bool halo_dir(int a) {
  return !is_reg<L>(a) && (SX == 0 || L::c[a][0] == -SX) && (SY == 0 || L::c[a][1] == -SY) &&
         (ZC == 0 || L::c[a][2] == ZC);
}
template <class L, int SX, int SY, int ZC>
__host__ __device__ constexpr int halo_rank(int a) {
  int r = 0;
  for (int b = 0; b < a; ++b)
    if (halo_dir<L, SX, SY, ZC>(b)) ++r;
  return r;
}

template <class L, typename T, typename C, int SX, int SY, int ZC, int PART>
__device__ __forceinline__ void push_halo(const Ring<L, T>& rg, int hdelta, int hx, int hy,
                                          const NodeMoments<C>& m, C om1) {
  unroll<L::q>([&](auto A) {
    constexpr int a = decltype(A)::value;
    using dd = Dir<L, a>;
    constexpr bool use = halo_dir<L, SX, SY, ZC>(a) && (halo_rank<L, SX, SY, ZC>(a) & 1) == PART;
    if constexpr (use) {
      const int tx = hx + dd::x, ty = hy + dd::y;
      bool in = true;
      if constexpr (SX == 0 && dd::x != 0) in = unsigned(tx) < unsigned(TX);
      if constexpr (SY == 0) in = in && unsigned(ty) < unsigned(TY);  // x columns carry the corners
      Shm<T>::template st_if<slot_off<L, a, dd::x, dd::y, T>()>(ring_addr<L, a, dd::z>(rg) + hdelta, 
                                                                 T(sf_post<L, a, C>(m, om1)), in);
    }
  });
}

template <class L, typename T, typename C, int ZC>
__device__ __forceinline__ void push_ring(const Ring<L, T>& rg, int hdelta, int task, int hx, int hy,
                                          const NodeMoments<C>& m, C om1) {
  switch (task) {
    case 0: push_halo<L, T, C, 0, -1, ZC, 0>(rg, hdelta, hx, hy, m, om1); break;
    case 1: push_halo<L, T, C, 0, -1, ZC, 1>(rg, hdelta, hx, hy, m, om1); break;
    case 2: push_halo<L, T, C, 0, 1, ZC, 0>(rg, hdelta, hx, hy, m, om1); break;
    case 3: push_halo<L, T, C, 0, 1, ZC, 1>(rg, hdelta, hx, hy, m, om1); break;
    case 4: push_halo<L, T, C, -1, 0, ZC, 0>(rg, hdelta, hx, hy, m, om1); break;
    case 5: push_halo<L, T, C, -1, 0, ZC, 1>(rg, hdelta, hx, hy, m, om1); break;
    case 6: push_halo<L, T, C, 1, 0, ZC, 0>(rg, hdelta, hx, hy, m, om1); break;
    default: push_halo<L, T, C, 1, 0, ZC, 1>(rg, hdelta, hx, hy, m, om1); break;
  }
}

// compute_moments of one node from its gathered slots (kernels.hpp:74-107;
// the sums of tslb_msums.cuh: bit-identical to k_moments). DZ: the slots of
// destination plane z + DZ (z = the plane being pushed); register-ring
// directions come from `Rv`.
template <class L, int DZ, typename T>
__device__ __forceinline__ void gather(const Ring<L, T>& rg, const T (&Rv)[L::q], T (&v)[L::q]) {
  unroll<L::q>([&](auto A) {
    constexpr int a = decltype(A)::value;
    if constexpr (is_reg<L>(a)) v[a] = Rv[a];
    else v[a] = Shm<T>::template ld<slot_off<L, a, 0, 0, T>()>(ring_addr<L, a, DZ>(rg));
  });
}

template <class L, typename T, typename C, class Put>
__device__ __forceinline__ void finalize(const Dom& d, const Ring<L, T>& rg, const T (&R)[L::q][3], const Put& put) {
  T rv[L::q], v[L::q];
  unroll<L::q>([&](auto A) {
    constexpr int a = decltype(A)::value;
    if constexpr (is_reg<L>(a)) rv[a] = R[a][0];
  });
  gather<L, -1, T>(rg, rv, v);
  moment_tail<L, T, C>(d, msums<L, T, C>(v), put);
}

// TM: the storage type of the moment arrays (T, or __half: the scaled fp16
// moments of the mixed-precision mode, tslb_store16.cuh); the populations
// are rounded to T in the slots either way
template <class L, typename T, typename C, bool WALLS, bool SOLID, int MINB, typename TM = T, bool PEER = false>
__global__ void __launch_bounds__(NT, MINB)
    k_mstep(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CUtensorMap gmap, Dom d,
            const TM* __restrict__ mi, const TM* __restrict__ gm, TM* __restrict__ mo, C om1, int lz, int zbeg,
            int zend, const uint32_t* __restrict__ sbits, TM* __restrict__ peer_lo, TM* __restrict__ peer_hi) {
  static_assert(L::dim == 3, "the M step is 3-D");
  using SM = Smem<L, T, SOLID, TM>;
  using W = typename MStore<TM>::W;
  constexpr int NM = n_moments<L>();
  extern __shared__ __align__(128) unsigned char smraw[];
  TM* tile = reinterpret_cast<TM*>(smraw);                // [2][NM][TR][TX]
  W* wstg = reinterpret_cast<W*>(smraw + SM::off_wstg);   // [2][NM][2 NH]
  T* sl = reinterpret_cast<T*>(smraw + SM::off_slots);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smraw + SM::off_bar);
  uint32_t* bstg = reinterpret_cast<uint32_t*>(smraw + SM::off_bits);  // [2][NT + 2 NH]
  constexpr int BITS_B = NT + 2 * NH;
  constexpr int TILE_B = int(SM::tile / sizeof(TM)), WSTG_B = int(SM::wstg / sizeof(W));

  const int tid = threadIdx.x, lx = tid & (TX - 1), ly = tid >> 5;
  const int x0 = int(blockIdx.x) * TX, y0 = int(blockIdx.y) * TY;
  const int za = zbeg + int(blockIdx.z) * lz, zb = min(za + lz, zend);
  const int gx = x0 + lx, gy = y0 + ly;
  // partial tiles at the high x / y edge of a grid that does not tile: the
  // tile is tw x th nodes, its right halo column and upper halo row sit
  // right after it; lanes beyond it push and store nothing (the TMA box
  // reads zeros there)
  const int tw = min(TX, d.nx - x0), th = min(TY, d.ny - y0);
  const bool active = lx < tw && ly < th;
  const int64_t col = active ? gx + int64_t(d.nx) * gy : 0;

  // halo task of this warp (see push_ring): side = warp / 2 (row below, row
  // above, column left, column right; the columns run from y0-1 to y0+TY and
  // so include the corners), half = warp % 2. Rows inside the domain come
  // with the TMA tile; the columns and wrapped rows are fetched by the lane
  // itself (cp.async into its half's copy of the ring in wstg).
  constexpr int WH = 2 * NH;  // wstg elements per moment array
  const int side = ly >> 1, half = ly & 1;
  int hnode = -1, hx = 0, hy = 0;
  if (side < 2) {
    if (lx < tw) {
      hnode = side * TX + lx;
      hx = lx;
      hy = side == 0 ? -1 : th;
    }
  } else if (side < 4 && lx < th + 2) {  // (warps beyond the eighth have no halo task)
    hnode = 2 * TX + (side - 2) * (TY + 2) + lx;
    hx = side == 2 ? -1 : tw;
    hy = lx - 1;
  }
  int64_t hcol = 0;
  bool hfetch = false;  // this lane loads its halo node itself
  int hoff = 0;         // where the halo node's moments are staged
  int hsel = 0;         // (2-byte moments: which half of the fetched word)
  if (hnode >= 0) {
    const int hgx = wrap_coord(x0 + hx, d.nx, d.mode[XMin], d.mode[XMax]);
    const int hgy = wrap_coord(y0 + hy, d.ny, d.mode[YMin], d.mode[YMax]);
    if (hgx < 0 || hgy < 0) {
      hnode = -1;
    } else {
      hcol = hgx + int64_t(d.nx) * hgy;
      hfetch = side >= 2 || hgy != y0 + hy;
      if (hfetch) {
        hoff = half * NH + hnode;
        hsel = MStore<TM>::sel(hcol);
      } else {
        hoff = (hy + 1) * TX + hx;
      }
    }
  }
  // halo node's column relative to the thread's own, in bytes
  const int hdelta = ((hy - ly) * TX + (hx - lx)) * int(sizeof(T));
  Contact ct{};
  if constexpr (WALLS) {
    ct.xlo = gx == 0 && d.mode[XMin] == kWall;
    ct.xhi = gx == d.nx - 1 && d.mode[XMax] == kWall;
    ct.ylo = gy == 0 && d.mode[YMin] == kWall;
    ct.yhi = gy == d.ny - 1 && d.mode[YMax] == kWall;
  }
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  constexpr uint32_t kTileBytes = uint32_t(NM * TC * sizeof(TM));
  auto issue = [&](int z, int b) {
    int zz = 0;
    const int src = plane_src(d, z, zz);
    if (src == 0) return;
    if (tid == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(&bar[b], kTileBytes);
      tma_load_4d(tile + b * TILE_B, src == 1 ? &tmap : &gmap, &bar[b], x0, y0 - 1, zz, 0);
    }
    if (hfetch) {
      W* w = wstg + b * WSTG_B + hoff;
      const TM* g = (src == 1 ? mi + int64_t(zz) * d.plane : gm + int64_t(zz) * NM * d.plane) + hcol;
      const int64_t cs = src == 1 ? d.mstride : d.plane;
#pragma unroll
      for (int c = 0; c < NM; ++c) __pipeline_memcpy_async(w + c * WH, MStore<TM>::word(g + c * cs), sizeof(W));
    }
    if constexpr (SOLID) {  // sbits points at plane 0; slab ghost planes at z = -1, nz
      const uint32_t* gb = sbits + int64_t(src == 1 ? zz : z) * d.plane;
      __pipeline_memcpy_async(bstg + b * BITS_B + tid, gb + col, 4);
      if (hnode >= 0) __pipeline_memcpy_async(bstg + b * BITS_B + NT + half * NH + hnode, gb + hcol, 4);
    }
  };

  T R[L::q][3];
#pragma unroll
  for (int a = 0; a < L::q; ++a) R[a][0] = R[a][1] = R[a][2] = T(0);
  Ring<L, T> rg;
  rg.init(smem_u32(sl + ly * TX + lx));
  int buf = 0;
  uint32_t phase = 0;  // bit b: parity of the next completion of bar[b]
  bool solid_prev = false;  // the tile node of the plane being reduced is solid
  const int64_t ms = d.mstride;

  auto plane = [&](auto ZCc, int z) {
    constexpr int ZC = decltype(ZCc)::value;
    if (ZC != -1) issue(z + 1, buf ^ 1);
    __pipeline_commit();
    int zz_unused = 0;
    if (plane_src(d, z, zz_unused) != 0) {
      mbar_wait(&bar[buf], (phase >> buf) & 1u);
      phase ^= 1u << buf;
      __pipeline_wait_prior(1);
      const TM* tb = tile + buf * TILE_B;
      if constexpr (WALLS) {
        ct.zlo = z == 0 && d.mode[ZMin] == kWall;
        ct.zhi = z == d.nz - 1 && d.mode[ZMax] == kWall;
      }
      bool solid = false, hsolid = false;
      if constexpr (SOLID) {
        ct.sb = bstg[buf * BITS_B + tid];
        solid = (ct.sb & kSelfSolid) != 0;
        hsolid = hnode >= 0 && (bstg[buf * BITS_B + NT + half * NH + hnode] & kSelfSolid);
        // solid nodes push nothing (stream_collide skips them); their moment
        // arrays keep their values (compute_moments skips them too), carried
        // into the output buffer of the ping-pong pair here
        if (ZC == 0 && solid && active) {
#pragma unroll
          for (int c = 0; c < NM; ++c)
            mo[c * d.mstride + col + int64_t(z) * d.plane] = tb[c * TC + (ly + 1) * TX + lx];
        }
      }
      if (!solid && active) {
        const NodeMoments<C> m = node_at<L, TM, C>(tb + (ly + 1) * TX + lx, TC);
        // the per-direction wall tests only for nodes on a wall face (whole
        // rows or planes: a warp-uniform branch); every other node pushes
        // without them
        if (WALLS && ZC == 0 && (ct.xlo || ct.xhi || ct.ylo || ct.yhi || ct.zlo || ct.zhi))
          push_tile<L, T, C, WALLS, SOLID, ZC>(d, rg, R, lx, ly, ct, m, om1);
        else
          push_tile<L, T, C, false, SOLID, ZC>(d, rg, R, lx, ly, ct, m, om1);
      }
      if (hnode >= 0 && !hsolid) {
        const NodeMoments<C> hm = hfetch ? staged_at<L, TM, C>(wstg + buf * WSTG_B + hoff, WH, hsel)
                                         : node_at<L, TM, C>(tb + hoff, TC);
        push_ring<L, T, C, ZC>(rg, hdelta, ly, hx, hy, hm, om1);
      }
    }
#ifndef TSLB_MSTEP_NOBAR  // (timing probe only: results are wrong without it)
    __syncthreads();
#endif
    // compute_moments skips solid nodes (their moment arrays keep their values)
    if (active && z - 1 >= za && !(SOLID && solid_prev)) {
      TM* o = mo + col + int64_t(z - 1) * d.plane;
      if constexpr (PEER) {
        // a slab's boundary planes also go straight into the z neighbours'
        // ghost buffers (peer memory: the halo exchange fused into the
        // epilogue of the boundary chunks)
        TM* plo = peer_lo && z - 1 == 0 ? peer_lo + col : nullptr;
        TM* phi = peer_hi && z - 1 == d.nz - 1 ? peer_hi + col : nullptr;
        finalize<L, T, C>(d, rg, R, [&](int c, T v) {
          const TM e = MStore<TM>::enc(c, v);
          o[c * ms] = e;
          if (plo) plo[c * d.plane] = e;
          if (phi) phi[c * d.plane] = e;
        });
      } else {
        finalize<L, T, C>(d, rg, R, [&](int c, T v) { o[c * ms] = MStore<TM>::enc(c, v); });
      }
    }
    if constexpr (SOLID) solid_prev = (ct.sb & kSelfSolid) != 0;  // (ct.sb: plane z)
    if constexpr (L::rd == 0) __syncthreads();
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
  // D3Q19: two planes per loop iteration -- the ping-pong tile buffer index
  // and part of the ring rotation become static (r02: 34.0 vs 33.4 GLUPS;
  // 4: 32.9). D3Q27 keeps one: its twice as large loop body missed the
  // instruction cache (no-instruction stalls 23 %, channel 17.6 vs 20.7)
#ifdef TSLB_MSTEP_UNROLL  // (measurement switch)
  constexpr int kUnroll = TSLB_MSTEP_UNROLL;
#else
  constexpr int kUnroll = L::q <= 19 ? 2 : 1;
#endif
#pragma unroll kUnroll
  for (int z = za; z < zb; ++z) plane(std::integral_constant<int, 0>{}, z);
  plane(std::integral_constant<int, -1>{}, zb);
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encoder() {
  static EncodeFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  }
  return fn;
}

// 4-D map (x, y, z, moment array) with a {TX, TY + 2, 1, NM} box over the
// moment buffer `base` (ghost = false), or over the slab ghost planes
// (ghost = true: layout [2][NM][plane], the "z" coordinate picks the side)
template <typename T>
const CUtensorMap* tensor_map(MstepMaps*& maps, const Dom& d, int nm, const T* base, bool ghost) {
  if (!maps) maps = new MstepMaps();
  const int64_t key[5] = {d.nx, d.ny, ghost ? -1 : d.nz, d.mstride, int64_t(sizeof(T)) * 16 + nm};
  auto same = [&](const MstepMaps::Entry& e) {
    bool eq = e.base == base;
    for (int i = 0; i < 5 && eq; ++i) eq = e.key[i] == key[i];
    return eq;
  };
  if (ghost) {
    if (same(maps->e[2])) return &maps->e[2].map;
  } else {
    for (int i = 0; i < 2; ++i)
      if (same(maps->e[i])) return &maps->e[i].map;
  }
  EncodeFn enc = encoder();
  if (!enc) return nullptr;
  auto& e = ghost ? maps->e[2] : maps->e[maps->next];
  const CUtensorMapDataType dt = sizeof(T) == 4   ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                 : sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64
                                                  : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  const cuuint64_t es = sizeof(T);
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  const cuuint64_t dim[4] = {cuuint64_t(d.nx), cuuint64_t(d.ny), cuuint64_t(ghost ? 2 : d.nz), cuuint64_t(nm)};
  // (ghost planes [2][NM][plane]: the "z" coordinate picks the side)
  const cuuint64_t str[3] = {cuuint64_t(d.nx) * es, (ghost ? cuuint64_t(nm) : 1u) * cuuint64_t(d.plane) * es,
                             ghost ? cuuint64_t(d.plane) * es : cuuint64_t(d.mstride) * es};
  const cuuint32_t box[4] = {cuuint32_t(TX), cuuint32_t(TR), 1, cuuint32_t(nm)};
  if (enc(&e.map, dt, 4, const_cast<T*>(base), dim, str, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return nullptr;
  e.base = base;
  for (int i = 0; i < 5; ++i) e.key[i] = key[i];
  if (!ghost) maps->next ^= 1;
  return &e.map;
}

// Incoming pushes of a slab boundary plane from the neighbour's nodes, built
// from the ghost moments (f materialisation of the M schedule on slabs):
// f_a(x, y, k) = T(post_collision_a(m(x - c_a))) for the directions entering
// through the slab face, exactly the values the F1 exchange would deliver;
// sources beyond an x/y wall do not exist (that slot holds the bounce).
template <class L, typename T, typename C>
__global__ void __launch_bounds__(128) k_ghost_push(Dom d, T* __restrict__ f, const T* __restrict__ gm,
                                                    C om1, int side, const uint8_t* __restrict__ solid) {
  const int i = int(blockIdx.x) * 128 + int(threadIdx.x), j = int(blockIdx.y);
  if (i >= d.nx) return;
  const int k = side ? d.nz - 1 : 0;
  const int cz_in = side ? -1 : 1;
  const T* g = gm + int64_t(side) * n_moments<L>() * d.plane;  // ([2][NM][plane])
  // masked geometries: a solid node keeps its populations, a solid source
  // pushes nothing (that slot holds the node's own bounce)
  if (solid && solid[fidx(d, i, j, k)]) return;
  unroll<L::q>([&](auto A) {
    constexpr int a = decltype(A)::value;
    using dd = Dir<L, a>;
    if constexpr (dd::z != 0) {
      if (dd::z != cz_in) return;
      const int sx = wrap_coord(i - dd::x, d.nx, d.mode[XMin], d.mode[XMax]);
      const int sy = wrap_coord(j - dd::y, d.ny, d.mode[YMin], d.mode[YMax]);
      if (sx < 0 || sy < 0) return;
      if (solid && solid[fidx(d, sx, sy, k - dd::z)]) return;
      const T* p = g + sx + int64_t(d.nx) * sy;
      const int64_t cs = d.plane;
      const NodeMoments<C> m = prepare_node<C>(C(p[0]), C(p[cs]), C(p[2 * cs]), C(p[3 * cs]), C(p[4 * cs]),
                                               C(p[5 * cs]), C(p[6 * cs]), C(p[7 * cs]), C(p[8 * cs]),
                                               C(p[9 * cs]));
      f[a * d.fstride + fidx(d, i, j, k)] = T(sf_post_ref<L, a, C>(m, om1));
    }
  });
}

// Solid bits of every node for the M step on a masked geometry: bit a set
// when the push of direction a crosses no wall face and its (wrapped) target
// is solid -- the bounce case resolve_push adds for solids
// (boundary.hpp:118-144); bit 31 when the node itself is solid. On z slabs
// `bits` has the ghost planes too (index (k + ghost) plane + ...): their
// nodes are halo sources of the M step, only their own bit is used; a push
// across a slab face targets the ghost plane of the mask.
template <class L>
__global__ void __launch_bounds__(128)
    k_solid_bits(Dom d, const uint8_t* __restrict__ solid, uint32_t* __restrict__ bits) {
  const int i = int(blockIdx.x) * 128 + int(threadIdx.x), j = int(blockIdx.y);
  const int k = int(blockIdx.z) - d.ghost;
  if (i >= d.nx) return;
  const int nd[3] = {d.nx, d.ny, d.nz};
  uint32_t b = solid[fidx(d, i, j, k)] ? kSelfSolid : 0u;
  if (k >= 0 && k < d.nz) unroll<L::q>([&](auto A) {
    constexpr int a = decltype(A)::value;
    if constexpr (a > 0) {
      using dd = Dir<L, a>;
      int tc[3] = {i + dd::x, j + dd::y, k + dd::z};
      bool wall = false;
#pragma unroll
      for (int ax = 0; ax < 3; ++ax) {
        if (tc[ax] < 0 || tc[ax] >= nd[ax]) {
          const int m = d.mode[2 * ax + (tc[ax] < 0 ? 0 : 1)];
          if (m == kWrap) tc[ax] += tc[ax] < 0 ? nd[ax] : -nd[ax];
          else if (m == kWall) wall = true;  // (kGhost: the ghost plane)
        }
      }
      if (!wall && solid[fidx(d, tc[0], tc[1], tc[2])]) b |= 1u << a;
    }
  });
  bits[int64_t(d.nx) * (int64_t(j) + int64_t(d.ny) * (k + d.ghost)) + i] = b;
}

}  // namespace mstep

// 3-D: any nx, ny whose rows the TMA tensor map can address (row pitch a
// multiple of 16 bytes); partial tiles at the high x / y edges
bool mstep_supported(int lat, const Dom& d, int esz) {
  if (lat == kD2Q9) return !d.has_solid && d.nz == 1 && d.ghost == 0;  // tslb_mstep2d.cu
  return (lat == kD3Q19 || lat == kD3Q27) && (int64_t(d.nx) * esz) % 16 == 0 && d.nx >= 2 && d.ny >= 2 &&
         mstep::encoder() != nullptr;
}

int launch_solid_bits(int lat, const Dom& d, const uint8_t* solid, uint32_t* bits, cudaStream_t st) {
  using namespace mstep;
  if (d.nz + 2 * d.ghost > 65535 || d.ny > 65535) return 1;
  const dim3 grid(unsigned((d.nx + 127) / 128), unsigned(d.ny), unsigned(d.nz + 2 * d.ghost));
  if (lat == kD3Q19) k_solid_bits<D3Q19><<<grid, 128, 0, st>>>(d, solid, bits);
  else if (lat == kD3Q27) k_solid_bits<D3Q27><<<grid, 128, 0, st>>>(d, solid, bits);
  else return 1;
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

template <typename T>
int launch_ghost_push(int lat, int math, const Dom& d, T* f, const T* gm, double omega, int side,
                      const uint8_t* solid, cudaStream_t st) {
  using namespace mstep;
  const dim3 grid(unsigned((d.nx + 127) / 128), unsigned(d.ny));
  auto go = [&](auto L) {
    using Lat = decltype(L);
    if (math == kMathDouble)
      k_ghost_push<Lat, T, double><<<grid, 128, 0, st>>>(d, f, gm, 1.0 - double(T(omega)), side, solid);
    else
      k_ghost_push<Lat, T, float><<<grid, 128, 0, st>>>(d, f, gm, 1.0f - float(omega), side, solid);
    return 0;
  };
  if (lat == kD3Q19) return go(D3Q19{});
  if (lat == kD3Q27) return go(D3Q27{});
  return 1;
}

template <typename T>
int launch_mstep(int lat, int math, const Dom& d, const T* mi, const T* gm, T* mo, double omega,
                 int lz, int z0, int z1, MstepMaps*& maps, const uint32_t* sbits, cudaStream_t st, T* peer_lo,
                 T* peer_hi) {
  using namespace mstep;
  if (!mstep_supported(lat, d, int(sizeof(T)))) return 1;
  if (d.has_solid && !sbits) return 1;
  if (z1 <= 0) z1 = d.nz;
  if (lat == kD2Q9) return z0 == 0 && z1 == d.nz ? launch_mstep2d<T>(math, d, mi, mo, omega, st) : 1;
  if ((d.mode[ZMin] == kGhost || d.mode[ZMax] == kGhost) && !gm) return 1;
  if (lz <= 0) lz = kDefaultLz;
  if (z0 < 0 || z1 > d.nz || z0 > z1) return 1;
  if (z0 == z1) return 0;
  const int nchunks = (z1 - z0 + lz - 1) / lz;
  bool walls = false;
  for (int fc = 0; fc < 6; ++fc) walls |= d.mode[fc] == kWall;
  const dim3 grid(unsigned((d.nx + TX - 1) / TX), unsigned((d.ny + TY - 1) / TY), unsigned(nchunks));
  if (grid.y > 65535 || grid.z > 65535) return 1;
  const double om1d = 1.0 - double(T(omega));
  const float om1f = 1.0f - float(omega);
  // slot-ring variant: one barrier per plane (deeper rings, two CTAs per SM)
  // for D3Q19 with fp32 storage -- measured faster than two barriers at three
  // CTAs per SM for fp32 node math (43.5 vs 36.7 GLUPS) and equal for fp64
  // (r01 s9); D3Q27 and fp64 storage would lose a CTA, so they keep two
  // barriers. TSLB_MSTEP_RD=0/1 overrides (measurements).
  static const int rd_env = [] {
    const char* e = std::getenv("TSLB_MSTEP_RD");
    return e ? std::atoi(e) : -1;
  }();
  const bool deep = rd_env >= 0 ? rd_env == 1 : (lat == kD3Q19 && sizeof(T) == 4);
  auto by_lat = [&](auto L) {
    using Lat = decltype(L);
    const CUtensorMap* tm = tensor_map<T>(maps, d, n_moments<Lat>(), mi, false);
    if (!tm) return 1;
    const CUtensorMap* gmp = gm ? tensor_map<T>(maps, d, n_moments<Lat>(), gm, true) : tm;
    if (!gmp) return 1;
    // CUDA failures come back as -error (the caller names the kernel)
    int err = 0;
    auto go = [&](auto kern, auto om1, size_t smem) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      if (e == cudaSuccess) {
        kern<<<grid, NT, smem, st>>>(*tm, *gmp, d, mi, gm, mo, om1, lz, z0, z1, sbits, peer_lo, peer_hi);
        e = cudaGetLastError();
      }
      if (e != cudaSuccess) err = -int(e);
    };
    constexpr size_t sm0 = Smem<Lat, T, false>::total, sm1 = Smem<Lat, T, true>::total;
    if ((d.has_solid ? sm1 : sm0) > 227 * 1024) return 1;
    // fp32 storage + fp32 math: three CTAs per SM (~76 KB shared memory, <= 80
    // registers); fp64 math keeps two (capping it at 80 registers costs more
    // ILP than the third CTA buys); fp64 storage holds one CTA per SM
    constexpr int MB = sizeof(T) == 4 && Lat::rd == 0 ? 3 : sizeof(T) == 4 ? 2 : 1;
    constexpr int MBD = sizeof(T) == 4 ? 2 : 1;
    // (peer outputs: slab boundary chunks on the peer-memory transport)
    const bool peer = (peer_lo || peer_hi) && !d.has_solid;
    if (math == kMathDouble) {
      if (d.has_solid && walls) go(k_mstep<Lat, T, double, true, true, MBD>, om1d, sm1);
      else if (d.has_solid) go(k_mstep<Lat, T, double, false, true, MBD>, om1d, sm1);
      else if (peer && walls) go(k_mstep<Lat, T, double, true, false, MBD, T, true>, om1d, sm0);
      else if (peer) go(k_mstep<Lat, T, double, false, false, MBD, T, true>, om1d, sm0);
      else if (walls) go(k_mstep<Lat, T, double, true, false, MBD>, om1d, sm0);
      else go(k_mstep<Lat, T, double, false, false, MBD>, om1d, sm0);
    } else if (peer) {
      if (walls) go(k_mstep<Lat, T, float, true, false, MB, T, true>, om1f, sm0);
      else go(k_mstep<Lat, T, float, false, false, MB, T, true>, om1f, sm0);
    } else {
      if (d.has_solid && walls) go(k_mstep<Lat, T, float, true, true, MB>, om1f, sm1);
      else if (d.has_solid) go(k_mstep<Lat, T, float, false, true, MB>, om1f, sm1);
      else if (walls) go(k_mstep<Lat, T, float, true, false, MB>, om1f, sm0);
      else go(k_mstep<Lat, T, float, false, false, MB>, om1f, sm0);
    }
    return err;
  };
  auto by_rd = [&](auto B) {
    using Base = decltype(B);
    return deep ? by_lat(SL<Base, 1>{}) : by_lat(SL<Base, 0>{});
  };
  return lat == kD3Q19 ? by_rd(D3Q19{}) : by_rd(D3Q27{});
}

// The mixed-precision M step: fp16 moments (MStore<__half>), fp32
// populations and node arithmetic; whole domains without solids.
int launch_mstep16(int lat, const Dom& d, const __half* mi, __half* mo, double omega, int lz, MstepMaps*& maps,
                   cudaStream_t st) {
  using namespace mstep;
  if (!mstep16_supported(lat, d)) return 1;
  if (lz <= 0) lz = kDefaultLz;
  const int nchunks = (d.nz + lz - 1) / lz;
  bool walls = false;
  for (int fc = 0; fc < 6; ++fc) walls |= d.mode[fc] == kWall;
  const dim3 grid(unsigned((d.nx + TX - 1) / TX), unsigned((d.ny + TY - 1) / TY), unsigned(nchunks));
  if (grid.y > 65535 || grid.z > 65535) return 1;
  const float om1 = 1.0f - float(omega);
  int err = 0;
  auto by_lat = [&](auto L) {
    using Lat = decltype(L);
    const CUtensorMap* tm = tensor_map<__half>(maps, d, n_moments<Lat>(), mi, false);
    if (!tm) return 1;
    constexpr size_t smem = Smem<Lat, float, false, __half>::total;
    auto go = [&](auto kern) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      if (e == cudaSuccess) {
        kern<<<grid, NT, smem, st>>>(*tm, *tm, d, mi, nullptr, mo, om1, lz, 0, d.nz, nullptr, nullptr, nullptr);
        e = cudaGetLastError();
      }
      if (e != cudaSuccess) err = -int(e);
    };
    if (walls) go(k_mstep<Lat, float, float, true, false, 2, __half>);
    else go(k_mstep<Lat, float, float, false, false, 2, __half>);
    return err;
  };
  return lat == kD3Q19 ? by_lat(SL<D3Q19, 1>{}) : by_lat(SL<D3Q27, 0>{});
}

bool mstep16_supported(int lat, const Dom& d) {
  return (lat == kD3Q19 || lat == kD3Q27) && d.nx % 8 == 0 && d.nx >= 2 && d.ny >= 2 && !d.has_solid &&
         d.ghost == 0 && mstep::encoder() != nullptr;
}

namespace {
// fp32 moment arrays <-> the fp16 storage codec (MStore<__half>)
__global__ void __launch_bounds__(256) k_moments_to16(const float* __restrict__ src, __half* __restrict__ dst,
                                                      int64_t n, int64_t stride, int nm) {
  const int64_t i = int64_t(blockIdx.x) * 256 + threadIdx.x;
  const int c = int(blockIdx.y);
  if (i < n && c < nm) dst[c * stride + i] = MStore<__half>::enc(c, src[c * stride + i]);
}
__global__ void __launch_bounds__(256) k_moments_from16(const __half* __restrict__ src, float* __restrict__ dst,
                                                        int64_t n, int64_t stride, int nm) {
  const int64_t i = int64_t(blockIdx.x) * 256 + threadIdx.x;
  const int c = int(blockIdx.y);
  if (i < n && c < nm) dst[c * stride + i] = MStore<__half>::dec(c, src[c * stride + i]);
}
}  // namespace

int launch_moments_codec16(const Dom& d, int nm, float* m32, __half* m16, int to16, cudaStream_t st) {
  const dim3 grid(unsigned((d.n + 255) / 256), unsigned(nm));
  if (to16) k_moments_to16<<<grid, 256, 0, st>>>(m32, m16, d.n, d.mstride, nm);
  else k_moments_from16<<<grid, 256, 0, st>>>(m16, m32, d.n, d.mstride, nm);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

template int launch_mstep<float>(int, int, const Dom&, const float*, const float*, float*, double, int, int, int,
                                 MstepMaps*&, const uint32_t*, cudaStream_t, float*, float*);
template int launch_mstep<double>(int, int, const Dom&, const double*, const double*, double*, double, int, int,
                                  int, MstepMaps*&, const uint32_t*, cudaStream_t, double*, double*);
template int launch_ghost_push<float>(int, int, const Dom&, float*, const float*, double, int, const uint8_t*,
                                      cudaStream_t);
template int launch_ghost_push<double>(int, int, const Dom&, double*, const double*, double, int,
                                       const uint8_t*, cudaStream_t);

}  // namespace tslb_cuda
