// Moment-resident single pass for D2Q9 (the M schedule in 2-D): m(t) -> m(t+1)
// in one kernel, bit-identical to compute_moments(stream_collide_fused(m(t)))
// (kernels.hpp:74-107, 154-204), like k_mstep for 3-D (tslb_mstep.cu) but
// with no shared memory and no barriers:
//
//   * a warp owns 30 consecutive columns (lanes 1..30) and marches up a strip
//     of rows; lanes 0 and 31 recompute the columns just left and right of
//     the strip (the halo) from the same instruction stream;
//   * each lane rebuilds the 9 post-collision populations of its node
//     (regularised collision, reference operand order, opposite pairs share
//     Q:Pi^neq) and rounds them to T; pushes along c_x = +-1 move one lane
//     with a warp shuffle, pushes along c_y land in a per-lane register ring
//     of destination rows y-1, y, y+1; wall bounces write the node's own
//     opposite slot (kernels.hpp:178-199), and a slot whose source lies
//     beyond a wall is never taken from the shuffle;
//   * once the march has passed row y, each owned lane reduces its 9 slots in
//     direction order to m(t+1) exactly as compute_moments (same sums, same
//     order) and stores them.
//
// HBM traffic: 2 x 6 scalars per lattice update (48 B fp32) instead of F1's
// 120 B; the row strips overlap by one halo row at each end (the rows just
// outside the strip push only their c_y-inward directions).
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "tslb_collision.cuh"
#include "tslb_domain.cuh"
#include "tslb_kernels.h"
#include "tslb_pair.cuh"

namespace tslb_cuda {
namespace cg = cooperative_groups;
namespace mstep2d {

constexpr int OWN = 30;  // owned columns per warp (lanes 1..30)
constexpr int WPB = 4;   // warps per block
constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ int wrap_coord(int g, int n, int lo, int hi) {
  if (g < 0) return lo == kWrap ? g + n : -1;
  if (g >= n) return hi == kWrap ? g - n : -1;
  return g;
}

template <typename T, typename C>
__device__ __forceinline__ NodeMoments<C> prep(const T (&v)[6]) {
  return prepare_node<C>(C(v[0]), C(v[1]), C(v[2]), C(0), C(v[3]), C(v[4]), C(0), C(v[5]), C(0), C(0));
}

// One warp's strip: columns strip * OWN - 1 .. + 31, rows ya .. ya + rows - 1.
// COH: the moments are read through L2 (ld.global.cg) -- the persistent
// kernel reads buffers that other SMs wrote before the last grid barrier,
// where the non-coherent read-only path could return stale lines.
template <class L, typename T, typename C, bool WALLS, bool COH>
__device__ __forceinline__ void strip_pass(const Dom& d, const T* __restrict__ mi, T* __restrict__ mo, C om1,
                                           int rows, int strip, int ya) {
  using Lat = L;
  const int lane = threadIdx.x & 31;
  const int xg = strip * OWN - 1 + lane;  // this lane's column (may lie outside [0, nx))
  const int xs = xg > d.nx ? -1 : wrap_coord(xg, d.nx, d.mode[XMin], d.mode[XMax]);
  const bool owned = lane >= 1 && lane <= OWN && xg < d.nx;
  const int yb = min(ya + rows, d.ny);
  // is the lane that pushes into this one along c_x = +1 / -1 a real node?
  const bool src = xs >= 0;
  const bool from_left = __shfl_up_sync(FULL, src, 1);
  const bool from_right = __shfl_down_sync(FULL, src, 1);
  const int64_t ms = d.mstride;
  bool cxlo = false, cxhi = false;
  if constexpr (WALLS) {
    cxlo = xg == 0 && d.mode[XMin] == kWall;
    cxhi = xg == d.nx - 1 && d.mode[XMax] == kWall;
  }

  auto load = [&](int y, T (&v)[6]) {
    const int yy = wrap_coord(y, d.ny, d.mode[YMin], d.mode[YMax]);
    if (yy < 0 || !src) {
      v[0] = T(1);
#pragma unroll
      for (int c = 1; c < 6; ++c) v[c] = T(0);
      return;
    }
    const int64_t idx = xs + int64_t(d.nx) * yy;
#pragma unroll
    for (int c = 0; c < 6; ++c) v[c] = COH ? __ldcg(mi + c * ms + idx) : __ldg(mi + c * ms + idx);
  };

  T R[9][3];  // slot of direction a for destination rows y-1, y, y+1
#pragma unroll
  for (int a = 0; a < 9; ++a) R[a][0] = R[a][1] = R[a][2] = T(0);
  T cur[6], nxt[6];
  load(ya - 1, cur);

  auto row = [&](auto ZCc, int y) {
    constexpr int ZC = decltype(ZCc)::value;
    if (ZC != -1) load(y + 1, nxt);
    if (wrap_coord(y, d.ny, d.mode[YMin], d.mode[YMax]) >= 0) {  // uniform: the row exists
      const NodeMoments<C> m = prep<T, C>(cur);
      bool cylo = false, cyhi = false;
      if constexpr (WALLS) {
        cylo = y == 0 && d.mode[YMin] == kWall;
        cyhi = y == d.ny - 1 && d.mode[YMax] == kWall;
      }
      // push of direction A (value o) into the slot of x + c_A, row y + c_y
      auto push = [&](auto A, T o) {
        constexpr int a = decltype(A)::value;
        using dd = Dir<Lat, a>;
        if constexpr (ZC == 0 || dd::y == ZC) {
          T r = o;
          bool ok = src;
          if constexpr (dd::x == 1) {
            r = __shfl_up_sync(FULL, o, 1);
            ok = from_left;
          }
          if constexpr (dd::x == -1) {
            r = __shfl_down_sync(FULL, o, 1);
            ok = from_right;
          }
          if (ok) R[a][1 + dd::y] = r;
          if constexpr (WALLS && ZC == 0) {
            const bool bx = (dd::x == 1 && cxhi) || (dd::x == -1 && cxlo);
            const bool by = (dd::y == 1 && cyhi) || (dd::y == -1 && cylo);
            if (bx || by) R[dd::opp][1] = bounce_value<Lat, a, T, C>(d, o, bx, by, false);
          }
        }
      };
      unroll<9>([&](auto A) {
        constexpr int a = decltype(A)::value;
        if constexpr (a == 0) {
          if constexpr (ZC == 0) push(A, T(sf_post<Lat, 0, C>(m, om1)));
        } else if constexpr (a & 1) {
          constexpr bool ua = ZC == 0 || Dir<Lat, a>::y == ZC;
          constexpr bool ub = ZC == 0 || Dir<Lat, a + 1>::y == ZC;
          if constexpr (ua && ub) {
            C ra, rb;
            sf_pair<Lat, a, C>(m, om1, ra, rb);
            push(A, T(ra));
            push(std::integral_constant<int, a + 1>{}, T(rb));
          } else if constexpr (ua) {
            push(A, T(sf_post<Lat, a, C>(m, om1)));
          } else if constexpr (ub) {
            push(std::integral_constant<int, a + 1>{}, T(sf_post<Lat, a + 1, C>(m, om1)));
          }
        }
      });
    }
    // the march has passed row y - 1: reduce it (compute_moments order)
    if (y - 1 >= ya && owned) {
      C r = 0, jx = 0, jy = 0, jz = 0, pxx = 0, pyy = 0, pxy = 0;
      unroll<9>([&](auto A) {
        constexpr int a = decltype(A)::value;
        using dd = Dir<Lat, a>;
        const C fa = C(R[a][0]);
        r += fa;
        if constexpr (dd::x == 1) jx += fa;
        if constexpr (dd::x == -1) jx -= fa;
        if constexpr (dd::y == 1) jy += fa;
        if constexpr (dd::y == -1) jy -= fa;
        if constexpr (dd::x != 0) pxx += fa;
        if constexpr (dd::y != 0) pyy += fa;
        if constexpr (dd::x * dd::y == 1) pxy += fa;
        if constexpr (dd::x * dd::y == -1) pxy -= fa;
      });
      force_shift<C>(d, jx, jy, jz);
      const C c3 = cs2<C>();
      const int64_t idx = xg + int64_t(d.nx) * (y - 1);
      mo[idx] = T(r);
      mo[ms + idx] = T(jx);
      mo[2 * ms + idx] = T(jy);
      mo[3 * ms + idx] = T(pxx - c3 * r - jx * jx);
      mo[4 * ms + idx] = T(pyy - c3 * r - jy * jy);
      mo[5 * ms + idx] = T(pxy - jx * jy);
    }
#pragma unroll
    for (int a = 0; a < 9; ++a) {
      R[a][0] = R[a][1];
      R[a][1] = R[a][2];
    }
#pragma unroll
    for (int c = 0; c < 6; ++c) cur[c] = nxt[c];
  };

  row(std::integral_constant<int, 1>{}, ya - 1);
#pragma unroll 1
  for (int y = ya; y < yb; ++y) row(std::integral_constant<int, 0>{}, y);
  row(std::integral_constant<int, -1>{}, yb);
}

template <class L, typename T, typename C, bool WALLS>
__global__ void __launch_bounds__(32 * WPB)
    k_mstep2d(Dom d, const T* __restrict__ mi, T* __restrict__ mo, C om1, int rows) {
  strip_pass<L, T, C, WALLS, false>(d, mi, mo, om1, rows, int(blockIdx.x) * WPB + int(threadIdx.x >> 5),
                                    int(blockIdx.y) * rows);
}

// Persistent form for small (launch-bound) domains: one cooperative launch
// runs nsteps M passes, ping-ponging m0 -> m1 -> m0 ..., with a grid barrier
// between passes; each block loops over the (strip block, row block) items
// of the regular grid. Same per-node arithmetic, so the same bits.
template <class L, typename T, typename C, bool WALLS>
__global__ void __launch_bounds__(32 * WPB)
    k_mstep2d_persist(Dom d, T* m0, T* m1, C om1, int rows, int nsteps, int nbx, int nby) {
  cg::grid_group grid = cg::this_grid();
  const int items = nbx * nby;
  for (int s = 0; s < nsteps; ++s) {
    const T* src = (s & 1) ? m1 : m0;
    T* dst = (s & 1) ? m0 : m1;
    for (int it = int(blockIdx.x); it < items; it += int(gridDim.x)) {
      const int bx = it % nbx, by = it / nbx;
      strip_pass<L, T, C, WALLS, true>(d, src, dst, om1, rows, bx * WPB + int(threadIdx.x >> 5), by * rows);
    }
    grid.sync();
  }
}

// ---------------------------------------------------------------------------
// Temporal blocking for small (latency-bound) domains: one cooperative launch
// runs the whole step(n); each block owns 32 x 16 tiles and advances a tile
// K passes at a time in shared memory from its moments plus a K-node halo
// (the region shrinks by one ring per pass), so the grid barrier and the
// trip through L2 come once per K passes instead of once per pass. Per pass:
// (1) every node of the region rebuilds its 9 post-collision populations
// (same forms as strip_pass, rounded to T); (2) every node whose sources are
// still valid gathers f_a(x) = pc_a(x - c_a), or -- when x - c_a lies beyond a
// wall -- the bounce of its own pc_opp(a) (the push x -> x + c_opp crosses that
// wall, kernels.hpp:178-199), and reduces them to m(t+1) in compute_moments'
// order. Regions of small periodic domains may hold a node twice; every copy
// computes the same bits. Same per-node arithmetic as strip_pass: same bits.
#ifndef TSLB_TBX  // (-DTSLB_TBX/TBY/TBT: measurements)
#define TSLB_TBX 32
#define TSLB_TBY 16
#define TSLB_TBT 1024
#endif
constexpr int TBX = TSLB_TBX, TBY = TSLB_TBY, TBT = TSLB_TBT;  // tile, threads per block
template <int K>
struct TbRegion {
  static constexpr int W = TBX + 2 * K, H = TBY + 2 * K, N = W * H;
};
template <typename T, int K>
constexpr size_t tb_smem() {
  return size_t(6 + 2 * 9) * TbRegion<K>::N * sizeof(T);
}

template <class L, typename T, typename C, bool WALLS, int K>
__global__ void __launch_bounds__(TBT, 1)
    k_mstep2d_tb(Dom d, T* m0, T* m1, C om1, int ngroups, int nsteps, int ntx, int nty) {
  using Lat = L;
  using RG = TbRegion<K>;
  constexpr int W = RG::W, H = RG::H, N = RG::N;
  extern __shared__ __align__(16) unsigned char tb_raw[];
  T* mom = reinterpret_cast<T*>(tb_raw);  // [6][N]
  T* pcs = mom + 6 * N;                   // [2][9][N] (double buffered)
  cg::grid_group grid = cg::this_grid();
  const int64_t ms = d.mstride;
  const int tiles = ntx * nty;
  // the node's 9 post-collision populations from its moments (T values, as
  // stored), rounded to T, into population buffer pc
  auto collide = [&](const T (&v)[6], T* pc, int e) {
    const NodeMoments<C> m = prep<T, C>(v);
    unroll<9>([&](auto A) {
      constexpr int a = decltype(A)::value;
      if constexpr (a == 0) {
        pc[e] = T(sf_post<Lat, 0, C>(m, om1));
      } else if constexpr (a & 1) {
        C ra, rb;
        sf_pair<Lat, a, C>(m, om1, ra, rb);
        pc[a * N + e] = T(ra);
        pc[(a + 1) * N + e] = T(rb);
      }
    });
  };
  auto exists = [&](int gx, int gy) {
    return wrap_coord(gx, d.nx, d.mode[XMin], d.mode[XMax]) >= 0 &&
           wrap_coord(gy, d.ny, d.mode[YMin], d.mode[YMax]) >= 0;
  };
  // groups of passes: sizes differ by at most one, their count has the
  // parity of nsteps (the result lands where the per-pass ping-pong would)
  const T* src = m0;
  T* dst = m1;
  int left = nsteps;
  for (int g = 0; g < ngroups; ++g) {
    const int ks = (left + (ngroups - g) - 1) / (ngroups - g);
    left -= ks;
    for (int tile = int(blockIdx.x); tile < tiles; tile += int(gridDim.x)) {
      const int ox = (tile % ntx) * TBX - K, oy = (tile / ntx) * TBY - K;  // region origin (global)
      // load the region's moments and collide every node of it (pass 0)
      for (int e = int(threadIdx.x); e < N; e += TBT) {
        const int gxr = wrap_coord(ox + e % W, d.nx, d.mode[XMin], d.mode[XMax]);
        const int gyr = wrap_coord(oy + e / W, d.ny, d.mode[YMin], d.mode[YMax]);
        if (gxr < 0 || gyr < 0) continue;  // beyond a wall: no node
        const int64_t idx = gxr + int64_t(d.nx) * gyr;
        T v[6];
#pragma unroll
        for (int c = 0; c < 6; ++c) v[c] = __ldcg(src + c * ms + idx);
        collide(v, pcs, e);
      }
      __syncthreads();
      // pass s: every node of the ring [s + 1, W - s - 1) x [s + 1, H - s - 1)
      // gathers f_a(x) = pc_a(x - c_a) (or the bounce of its own opposite
      // push when x - c_a lies beyond a wall), reduces its moments and --
      // still the same thread, the same node -- collides them for pass s + 1
      // into the other population buffer: one barrier per pass
      for (int s = 0; s < ks; ++s) {
        const T* pc = pcs + (s & 1) * 9 * N;
        T* pn = pcs + ((s + 1) & 1) * 9 * N;
        const bool last = s + 1 == ks;
        const int w = W - 2 * (s + 1), cnt = w * (H - 2 * (s + 1));
        for (int q = int(threadIdx.x); q < cnt; q += TBT) {
          const int lx = s + 1 + q % w, ly = s + 1 + q / w, e = lx + W * ly;
          const int gx = ox + lx, gy = oy + ly;
          if (!exists(gx, gy)) continue;
          C r = 0, jx = 0, jy = 0, jz = 0, pxx = 0, pyy = 0, pxy = 0;
          unroll<9>([&](auto A) {
            constexpr int a = decltype(A)::value;
            using dd = Dir<Lat, a>;
            T fa;
            if constexpr (a == 0) {
              fa = pc[e];
            } else {
              bool bx = false, by = false;
              if constexpr (WALLS) {
                const int sx = gx - dd::x, sy = gy - dd::y;
                bx = dd::x != 0 && ((sx < 0 && d.mode[XMin] == kWall) || (sx >= d.nx && d.mode[XMax] == kWall));
                by = dd::y != 0 && ((sy < 0 && d.mode[YMin] == kWall) || (sy >= d.ny && d.mode[YMax] == kWall));
              }
              if (bx || by) fa = bounce_value<Lat, dd::opp, T, C>(d, pc[dd::opp * N + e], bx, by, false);
              else fa = pc[a * N + e - dd::x - W * dd::y];
            }
            const C f = C(fa);
            r += f;
            if constexpr (dd::x == 1) jx += f;
            if constexpr (dd::x == -1) jx -= f;
            if constexpr (dd::y == 1) jy += f;
            if constexpr (dd::y == -1) jy -= f;
            if constexpr (dd::x != 0) pxx += f;
            if constexpr (dd::y != 0) pyy += f;
            if constexpr (dd::x * dd::y == 1) pxy += f;
            if constexpr (dd::x * dd::y == -1) pxy -= f;
          });
          force_shift<C>(d, jx, jy, jz);
          const C c3 = cs2<C>();
          T v[6];
          v[0] = T(r);
          v[1] = T(jx);
          v[2] = T(jy);
          v[3] = T(pxx - c3 * r - jx * jx);
          v[4] = T(pyy - c3 * r - jy * jy);
          v[5] = T(pxy - jx * jy);
          if (last) {
#pragma unroll
            for (int c = 0; c < 6; ++c) mom[c * N + e] = v[c];
          } else {
            collide(v, pn, e);
          }
        }
        __syncthreads();
      }
      // the owned tile (ring K) is exact after ks <= K passes
      for (int q = int(threadIdx.x); q < TBX * TBY; q += TBT) {
        const int lx = K + q % TBX, ly = K + q / TBX;
        const int gx = ox + lx, gy = oy + ly;
        if (gx >= d.nx || gy >= d.ny) continue;
        const int64_t idx = gx + int64_t(d.nx) * gy;
        const int e = lx + W * ly;
#pragma unroll
        for (int c = 0; c < 6; ++c) dst[c * ms + idx] = mom[c * N + e];
      }
      __syncthreads();
    }
    grid.sync();
    const T* t = src;
    src = dst;
    dst = const_cast<T*>(t);
  }
}

}  // namespace mstep2d

namespace mstep2d {
// passes per temporal block (TSLB_TB_K at build time: measurements)
#ifndef TSLB_TB_K
#define TSLB_TB_K 4
#endif
constexpr int kTbPasses = TSLB_TB_K;
// rows per warp: 16 measured best at 4096^2 (72.8 GLUPS vs 67.5 at 64 and
// 71.2 at 8: the two halo rows vs wave quantisation); small domains
// (launch-bound, e.g. the 256^2 cavity) shorten strips for parallelism:
// 256^2 kernel 8.6 us at 2 rows vs 9.5 at 4, 10.1 at 1, 10.6 at 8 (s28)
inline int strip_rows(const Dom& d) {
  const int strips = (d.nx + OWN - 1) / OWN;
  int rows = 16;
  while (rows > 2 && int64_t(strips) * ((d.ny + rows - 1) / rows) < 148 * 32) rows /= 2;
  static const int rows_env = [] {
    const char* e = std::getenv("TSLB_ROWS2D");
    return e ? std::atoi(e) : 0;
  }();
  return rows_env > 0 ? rows_env : rows;
}
}  // namespace mstep2d

template <typename T>
int launch_mstep2d(int math, const Dom& d, const T* mi, T* mo, double omega, cudaStream_t st) {
  using namespace mstep2d;
  if (d.has_solid || d.nz != 1 || d.ghost) return 1;
  const int strips = (d.nx + OWN - 1) / OWN;
  const unsigned bx = unsigned((strips + WPB - 1) / WPB);
  const int rows = strip_rows(d);
  const dim3 grid(bx, unsigned((d.ny + rows - 1) / rows));
  if (grid.y > 65535) return 1;
  bool walls = false;
  for (int fc = 0; fc < 4; ++fc) walls |= d.mode[fc] == kWall;
  if (math == kMathDouble) {
    const double om1 = 1.0 - double(T(omega));
    if (walls) k_mstep2d<D2Q9, T, double, true><<<grid, 32 * WPB, 0, st>>>(d, mi, mo, om1, rows);
    else k_mstep2d<D2Q9, T, double, false><<<grid, 32 * WPB, 0, st>>>(d, mi, mo, om1, rows);
  } else {
    const float om1 = 1.0f - float(omega);
    if (walls) k_mstep2d<D2Q9, T, float, true><<<grid, 32 * WPB, 0, st>>>(d, mi, mo, om1, rows);
    else k_mstep2d<D2Q9, T, float, false><<<grid, 32 * WPB, 0, st>>>(d, mi, mo, om1, rows);
  }
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : -int(e);  // (the caller names the kernel)
}

// nsteps M passes in one cooperative launch (m0 holds m(t); the result is in
// m0 for even nsteps, m1 for odd). Returns 1 (nothing launched) when the
// domain does not qualify or the device refuses a co-resident grid.
template <typename T>
int launch_mstep2d_persist(int math, const Dom& d, T* m0, T* m1, double omega, int nsteps, cudaStream_t st) {
  using namespace mstep2d;
  if (d.has_solid || d.nz != 1 || d.ghost || nsteps < 1) return 1;
  const int strips = (d.nx + OWN - 1) / OWN;
  const int nbx = (strips + WPB - 1) / WPB;
  const int rows = strip_rows(d);
  const int nby = (d.ny + rows - 1) / rows;
  bool walls = false;
  for (int fc = 0; fc < 4; ++fc) walls |= d.mode[fc] == kWall;
  int dev = 0, sms = 0, coop = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 1;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  if (!coop) return 1;
  auto go = [&](auto kern, auto om1) {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * WPB, 0) != cudaSuccess || per_sm < 1)
      return 1;
    const int blocks = std::min(nbx * nby, per_sm * sms);
    Dom dd = d;
    T *a = m0, *b = m1;
    int rr = rows, ns = nsteps, x = nbx, y = nby;
    void* args[] = {&dd, &a, &b, &om1, &rr, &ns, &x, &y};
    // an error still pending from the work enqueued before belongs to the
    // caller: report it (-error) rather than clearing it with the refusal below
    if (const cudaError_t pe = cudaPeekAtLastError(); pe != cudaSuccess) return -int(pe);
    const cudaError_t e =
        cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kern), dim3(blocks), dim3(32 * WPB), args, 0, st);
    if (e == cudaSuccess) return 0;
    cudaGetLastError();  // (a refused launch is not sticky)
    // not co-resident: the caller falls back to per-pass launches; any other
    // failure is reported
    return e == cudaErrorCooperativeLaunchTooLarge ? 1 : -int(e);
  };
  // temporal blocking (TSLB_TB2D=0: the per-pass persistent kernel; read per
  // call, like TSLB_PERSIST)
  const char* tbe = std::getenv("TSLB_TB2D");
  const int tb_env = tbe ? std::atoi(tbe) : 1;
  constexpr int K = kTbPasses;
  const int ntx = (d.nx + TBX - 1) / TBX, nty = (d.ny + TBY - 1) / TBY;
  auto go_tb = [&](auto kern, auto om1) {
    const size_t smem = tb_smem<T, K>();
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess) {
      cudaGetLastError();
      return 1;
    }
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TBT, smem) != cudaSuccess || per_sm < 1) {
      cudaGetLastError();
      return 1;
    }
    const int blocks = std::min(ntx * nty, per_sm * sms);
    // groups of <= K passes whose count has the parity of nsteps
    int groups = (nsteps + K - 1) / K;
    if ((groups - nsteps) % 2 != 0) ++groups;
    Dom dd = d;
    T *a = m0, *b = m1;
    int gg = groups, ns = nsteps, x = ntx, y = nty;
    void* args[] = {&dd, &a, &b, &om1, &gg, &ns, &x, &y};
    if (const cudaError_t pe = cudaPeekAtLastError(); pe != cudaSuccess) return -int(pe);
    const cudaError_t e =
        cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kern), dim3(blocks), dim3(TBT), args, smem, st);
    if (e == cudaSuccess) return 0;
    cudaGetLastError();
    return e == cudaErrorCooperativeLaunchTooLarge ? 1 : -int(e);
  };
  // (regions reach at most K nodes past the padded tiles: one wrap suffices)
  if (tb_env != 0 && nsteps >= 2 && d.nx >= TBX + K && d.ny >= TBY + K) {
    int r;
    if (math == kMathDouble) {
      const double om1 = 1.0 - double(T(omega));
      r = walls ? go_tb(k_mstep2d_tb<D2Q9, T, double, true, K>, om1)
                : go_tb(k_mstep2d_tb<D2Q9, T, double, false, K>, om1);
    } else {
      const float om1 = 1.0f - float(omega);
      r = walls ? go_tb(k_mstep2d_tb<D2Q9, T, float, true, K>, om1)
                : go_tb(k_mstep2d_tb<D2Q9, T, float, false, K>, om1);
    }
    if (r <= 0) return r;
  }
  if (math == kMathDouble) {
    const double om1 = 1.0 - double(T(omega));
    return walls ? go(k_mstep2d_persist<D2Q9, T, double, true>, om1)
                 : go(k_mstep2d_persist<D2Q9, T, double, false>, om1);
  }
  const float om1 = 1.0f - float(omega);
  return walls ? go(k_mstep2d_persist<D2Q9, T, float, true>, om1) : go(k_mstep2d_persist<D2Q9, T, float, false>, om1);
}

template int launch_mstep2d<float>(int, const Dom&, const float*, float*, double, cudaStream_t);
template int launch_mstep2d<double>(int, const Dom&, const double*, double*, double, cudaStream_t);
template int launch_mstep2d_persist<float>(int, const Dom&, float*, float*, double, int, cudaStream_t);
template int launch_mstep2d_persist<double>(int, const Dom&, double*, double*, double, int, cudaStream_t);

}  // namespace tslb_cuda
