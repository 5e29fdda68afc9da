// TMA-staged fused stream-collide (box geometries): the F1 phase-2 kernel
// built around the Tensor Memory Accelerator.
//
// Tile = TX consecutive x nodes of one row (j, k). A CTA walks `kz` planes of
// its (x tile, j) column with a two-stage pipeline:
//   * moments of tile t+2 are fetched by ONE cp.async.bulk.tensor load (all
//     1+D+np arrays in one 4-D box) into shared memory, signalled by an
//     mbarrier, while tile t is collided;
//   * each thread collides its VX nodes (fp64 node math, bit-exact with the
//     reference; or fp32 opt-in) and writes the q outputs to a shared-memory
//     tile;
//   * ONE thread pushes the tile with q cp.async.bulk.tensor stores whose box
//     origin is shifted by c_a: the hardware performs the one-element x shift
//     of c_x = +-1 pushes (element-granular tensor coordinates), y/z shifts
//     and periodic y/z wraps are plain coordinates, and pushes leaving the
//     tensor along x are clipped. The two row-end elements (x wrap or x-wall
//     bounce) and y/z-wall bounces are written directly by the owning thread.
// Every slot still has exactly one writer (reference kernels.hpp:149-153):
// adjacent tiles' shifted boxes abut without overlap, and the clipped slots
// are exactly the ones the row-end writes fill.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "tslb_collision.cuh"
#include "tslb_domain.cuh"
#include "tslb_kernels.h"
#include "tslb_pair.cuh"

namespace tslb_cuda {

struct TmaMaps {
  CUtensorMap fmap;  // populations: (x, y, z incl. ghosts, direction)
  CUtensorMap mmap;  // moments:     (x, y, z, component)
  const void* fbase = nullptr;
  const void* mbase = nullptr;
  int lat = -1, esz = 0, tx = 0;
  int64_t key[6] = {0, 0, 0, 0, 0, 0};
};

void free_tma_maps(TmaMaps* m) { delete m; }

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, const void* src, int c0, int c1, int c2,
                                             int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

constexpr int NT = 128;   // compute threads per CTA
constexpr int NTE = NT + 32;  // + one edge/producer warp

// wall bounce with u_wall summed over crossed wall faces in axis order, in T
// (boundary.hpp:127-137, kernels.hpp:187-192)
template <class L, int A, typename T, typename C>
__device__ __forceinline__ T bounce_of(const Dom& d, T out, bool cx, bool cy, bool cz) {
  using dd = Dir<L, A>;
  T wx = T(0), wy = T(0), wz = T(0);
  auto add = [&](int face) {
    wx += T(d.uw[face][0]);
    wy += T(d.uw[face][1]);
    wz += T(d.uw[face][2]);
  };
  if (cx) add(dd::x > 0 ? XMax : XMin);
  if (cy) add(dd::y > 0 ? YMax : YMin);
  if (cz) add(dd::z > 0 ? ZMax : ZMin);
  return T(C(out) - bounce_correction<L, A, C>(C(wx), C(wy), C(wz)));
}

template <class L, typename T, typename C>
__device__ __forceinline__ NodeMoments<C> node_from(const T* p, int64_t stride) {
  if constexpr (L::dim == 3)
    return prepare_node<C>(C(p[0]), C(p[stride]), C(p[2 * stride]), C(p[3 * stride]), C(p[4 * stride]),
                           C(p[5 * stride]), C(p[6 * stride]), C(p[7 * stride]), C(p[8 * stride]),
                           C(p[9 * stride]));
  else
    return prepare_node<C>(C(p[0]), C(p[stride]), C(p[2 * stride]), C(0), C(p[3 * stride]), C(p[4 * stride]),
                           C(0), C(p[5 * stride]), C(0), C(0));
}

template <class L, typename C>
__device__ __forceinline__ bool needs_exact(const NodeMoments<C>& m) {
  return (m.rho == C(0) && signbit(m.rho)) || m.pxx == C(0) || m.pyy == C(0) ||
         (L::dim == 3 && m.pzz == C(0));
}

}  // namespace

// Tile = TX consecutive x nodes of row (j, k). Slot x of direction a holds
// the push of node x - c_a, so the shared-memory tile of direction a is
// written at element e + c_x and stored by TMA at the ALIGNED origin x0 (TMA
// tensor coordinates must be 16-byte aligned in x): the one element per tile
// and direction that comes from outside the tile (node x0-1 for c_x = +1,
// node x0+TX for c_x = -1) is computed by the edge warp ("halo" pushes; with
// x walls at the row ends the node's own bounce fills it instead). Warps
// 0-3 collide the tile; warp 4 computes the halo and drives the TMA.
template <class L, typename T, typename C, int VX>
__global__ void __launch_bounds__(NTE)
    k_streamcoll_tma(const __grid_constant__ CUtensorMap fmap, const __grid_constant__ CUtensorMap mmap, Dom d,
                     T* __restrict__ f, const T* __restrict__ mo, C om1, int kz) {
  constexpr int TX = NT * VX;
  constexpr int NM = 1 + L::dim + L::dim * (L::dim + 1) / 2;
  constexpr int Q = L::q;
  extern __shared__ __align__(128) unsigned char smem[];
  T* in = reinterpret_cast<T*>(smem);  // [2][NM][TX]
  T* out = in + 2 * NM * TX;           // [2][Q][TX]
  uint64_t* bar = reinterpret_cast<uint64_t*>(out + 2 * Q * TX);

  const int tid = int(threadIdx.x);
  const bool edge_warp = tid >= NT;
  const int lane = tid & 31;
  constexpr int PRODUCER = NT;
  const int x0 = int(blockIdx.x) * TX;
  const int j = int(blockIdx.y);
  const int kb = d.k0 + int(blockIdx.z) * kz;
  const int ke = min(kb + kz, d.k0 + d.nzr);
  const int ntile = ke - kb;
  const bool xwall = d.mode[XMin] == kWall;

  if (tid == PRODUCER) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_async_smem();
  }
  __syncthreads();
  auto issue_load = [&](int t, int s) {
    mbar_expect_tx(&bar[s], uint32_t(NM * TX * sizeof(T)));
    tma_load_4d(in + s * NM * TX, &mmap, &bar[s], x0, j, kb + t, 0);
  };
  if (tid == PRODUCER) {
    issue_load(0, 0);
    if (ntile > 1) issue_load(1, 1);
  }

  // edge warp: lanes [0,16) left halo node x0-1, lanes [16,32) right halo
  // node x0+TX; lane % 16 selects the x-shifted direction pair
  const bool left = lane < 16;
  const int hp = lane & 15;
  int hx = left ? x0 - 1 : x0 + TX;
  bool halo = edge_warp;
  if (hx < 0 || hx >= d.nx) {
    if (xwall) halo = false;  // row end at a wall: the node's own bounce fills the slot
    hx = hx < 0 ? hx + d.nx : hx - d.nx;
  }

#pragma unroll 1
  for (int t = 0; t < ntile; ++t) {
    const int s = t & 1;
    const int k = kb + t;
    const bool jlo = j == 0, jhi = j == d.ny - 1, klo = k == 0, khi = k == d.nz - 1;
    auto bounces = [&](auto A, bool& by, bool& bz) {
      using dd = Dir<L, decltype(A)::value>;
      by = (dd::y == 1 && jhi && d.mode[YMax] == kWall) || (dd::y == -1 && jlo && d.mode[YMin] == kWall);
      bz = (dd::z == 1 && khi && d.mode[ZMax] == kWall) || (dd::z == -1 && klo && d.mode[ZMin] == kWall);
    };
    // halo moments straight from global (issued before the barrier wait)
    NodeMoments<C> hm;
    if (edge_warp)
      hm = node_from<L, T, C>(mo + int64_t(hx) + int64_t(d.nx) * (int64_t(j) + int64_t(d.ny) * k), d.mstride);
    if (tid == PRODUCER && t >= 2) bulk_wait_read<1>();  // tile t-2's stores have read out[s]
    __syncthreads();
    mbar_wait(&bar[s], uint32_t((t >> 1) & 1));

    T* tout = out + s * Q * TX;
    const T* tin = in + s * NM * TX;
    NodeMoments<C> m[VX];
    bool exact = false;
    if (!edge_warp) {
#pragma unroll
      for (int v = 0; v < VX; ++v) {
        m[v] = node_from<L, T, C>(tin + tid * VX + v, TX);
        exact |= needs_exact<L, C>(m[v]);
      }
    } else {
      exact = halo && needs_exact<L, C>(hm);
    }
    const bool ex = __syncthreads_or(exact);

    if (!edge_warp) {
      const int64_t fi = int64_t(d.nx) * (int64_t(j) + int64_t(d.ny) * (int64_t(k) + d.ghost)) + x0 + tid * VX;
      // one direction's VX outputs -> the tile (shifted by c_x), or bounced
      auto emit = [&](auto A, const T (&vals)[VX]) {
        constexpr int a = decltype(A)::value;
        using dd = Dir<L, a>;
        bool by, bz;
        bounces(A, by, bz);
        if (by || bz) {
          T b[VX];
#pragma unroll
          for (int v = 0; v < VX; ++v) {
            const int x = x0 + tid * VX + v;
            const bool cx = xwall && ((dd::x == 1 && x == d.nx - 1) || (dd::x == -1 && x == 0));
            b[v] = bounce_of<L, a, T, C>(d, vals[v], cx, by, bz);
          }
          Vec<T, VX>::st(f + dd::opp * d.fstride + fi, b);
        } else if constexpr (dd::x == 0) {
          Vec<T, VX>::st(tout + a * TX + tid * VX, vals);
        } else {
#pragma unroll
          for (int v = 0; v < VX; ++v) {
            const int e = tid * VX + v + dd::x;
            if (e >= 0 && e < TX) {
              tout[a * TX + e] = vals[v];
            } else if (xwall) {
              const int x = x0 + tid * VX + v;
              if ((dd::x == 1 && x == d.nx - 1) || (dd::x == -1 && x == 0))
                tout[dd::opp * TX + tid * VX + v] = bounce_of<L, a, T, C>(d, vals[v], true, false, false);
            }
          }
        }
      };
      if (ex) {
        unroll<Q>([&](auto A) {
          constexpr int a = decltype(A)::value;
          T vals[VX];
#pragma unroll
          for (int v = 0; v < VX; ++v) vals[v] = T(post_collision<L, a, C>(m[v], om1));
          emit(A, vals);
        });
      } else {
        unroll<Q>([&](auto A) {
          constexpr int a = decltype(A)::value;
          if constexpr (a == 0) {
            T vals[VX];
#pragma unroll
            for (int v = 0; v < VX; ++v) vals[v] = T(post_rest<L, C>(m[v], om1));
            emit(A, vals);
          } else if constexpr (a & 1) {
            T va[VX], vb[VX];
#pragma unroll
            for (int v = 0; v < VX; ++v) {
              C ra, rb;
              post_pair<L, a, C>(m[v], om1, ra, rb);
              va[v] = T(ra);
              vb[v] = T(rb);
            }
            emit(A, va);
            emit(std::integral_constant<int, a + 1>{}, vb);
          }
        });
      }
    } else if (halo) {
      // halo pushes: pair number hp among the x-shifted pairs
      int p = 0;
      unroll<Q>([&](auto A) {
        constexpr int a = decltype(A)::value;
        if constexpr ((a & 1) && Dir<L, a>::x != 0) {
          if (p++ == hp) {
            // member with c_x = +1 feeds the left halo slot, c_x = -1 the right
            constexpr int ap = Dir<L, a>::x == 1 ? a : a + 1;
            constexpr int am = Dir<L, a>::x == 1 ? a + 1 : a;
            bool by, bz;
            C ra, rb;
            if (ex) {
              ra = post_collision<L, a, C>(hm, om1);
              rb = post_collision<L, a + 1, C>(hm, om1);
            } else {
              post_pair<L, a, C>(hm, om1, ra, rb);
            }
            const T vp = T(Dir<L, a>::x == 1 ? ra : rb);
            const T vm = T(Dir<L, a>::x == 1 ? rb : ra);
            if (left) {
              bounces(std::integral_constant<int, ap>{}, by, bz);
              if (!(by || bz)) tout[ap * TX] = vp;
            } else {
              bounces(std::integral_constant<int, am>{}, by, bz);
              if (!(by || bz)) tout[am * TX + TX - 1] = vm;
            }
          }
        }
      });
    }
    fence_async_smem();
    __syncthreads();
    if (tid == PRODUCER) {
      unroll<Q>([&](auto A) {
        constexpr int a = decltype(A)::value;
        using dd = Dir<L, a>;
        bool by, bz;
        bounces(A, by, bz);
        if (by || bz) return;  // bounced directly above
        int yt = j + dd::y, zt = k + dd::z;
        if (yt < 0) yt += d.ny;
        if (yt >= d.ny) yt -= d.ny;
        if ((zt < 0 || zt >= d.nz) && d.mode[zt < 0 ? ZMin : ZMax] == kWrap) zt = zt < 0 ? zt + d.nz : zt - d.nz;
        tma_store_4d(&fmap, tout + a * TX, x0, yt, zt + d.ghost, a);
      });
      bulk_commit();
      if (t + 2 < ntile) issue_load(t + 2, s);
    }
  }
  if (tid == PRODUCER) bulk_wait_all();
}

namespace {

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

}  // namespace

template <typename T, int VX>
int launch_tma_vx(int lat, int math, const Dom& d, T* f, const T* mo, double omega, int kz, TmaMaps*& maps,
                  cudaStream_t st) {
  constexpr int TX = NT * VX;
  if (kz <= 0) kz = 8;
  if (d.nx % TX != 0 || d.ny > 65535) return 1;
  // x walls must be resting (the clipped row ends bounce with zero velocity)
  if (d.mode[XMin] == kWall)
    for (int c = 0; c < 3; ++c)
      if (d.uw[XMin][c] != 0 || d.uw[XMax][c] != 0) return 1;
  const int nzc = (d.nzr + kz - 1) / kz;
  if (nzc > 65535) return 1;
  EncodeFn enc = encoder();
  if (!enc) return 1;
  int q = 0, dim = 0;
  if (lat == kD2Q9) q = D2Q9::q, dim = 2;
  else if (lat == kD3Q19) q = D3Q19::q, dim = 3;
  else if (lat == kD3Q27) q = D3Q27::q, dim = 3;
  else return 1;
  const int nm = 1 + dim + dim * (dim + 1) / 2;
  const int64_t key[6] = {d.nx, d.ny, d.nz, d.ghost, d.fstride, d.mstride};
  if (!maps || maps->fbase != f || maps->mbase != mo || maps->lat != lat || maps->esz != int(sizeof(T)) ||
      maps->tx != TX ||
      std::memcmp(maps->key, key, sizeof key) != 0) {
    if (!maps) maps = new TmaMaps();
    const CUtensorMapDataType dt = sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
    const cuuint64_t es = sizeof(T);
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    cuuint64_t fdim[4] = {cuuint64_t(d.nx), cuuint64_t(d.ny), cuuint64_t(d.nz + 2 * d.ghost), cuuint64_t(q)};
    cuuint64_t fstr[3] = {cuuint64_t(d.nx) * es, cuuint64_t(d.plane) * es, cuuint64_t(d.fstride) * es};
    cuuint32_t fbox[4] = {cuuint32_t(TX), 1, 1, 1};
    if (enc(&maps->fmap, dt, 4, f, fdim, fstr, fbox, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return 1;
    cuuint64_t mdim[4] = {cuuint64_t(d.nx), cuuint64_t(d.ny), cuuint64_t(d.nz), cuuint64_t(nm)};
    cuuint64_t mstr[3] = {cuuint64_t(d.nx) * es, cuuint64_t(d.plane) * es, cuuint64_t(d.mstride) * es};
    cuuint32_t mbox[4] = {cuuint32_t(TX), 1, 1, cuuint32_t(nm)};
    if (enc(&maps->mmap, dt, 4, const_cast<T*>(mo), mdim, mstr, mbox, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return 1;
    maps->fbase = f;
    maps->mbase = mo;
    maps->lat = lat;
    maps->esz = int(sizeof(T));
    maps->tx = TX;
    std::memcpy(maps->key, key, sizeof key);
  }
  const dim3 grid(unsigned(d.nx / TX), unsigned(d.ny), unsigned(nzc));
  const double om1d = 1.0 - double(T(omega));
  const float om1f = 1.0f - float(omega);
  auto go = [&](auto L) {
    using Lat = decltype(L);
    const size_t sm = size_t(2) * (1 + Lat::dim + Lat::dim * (Lat::dim + 1) / 2) * TX * sizeof(T) +
                      size_t(2) * Lat::q * TX * sizeof(T) + 2 * sizeof(uint64_t);
    auto launch = [&](auto kern, auto om) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
      kern<<<grid, NTE, sm, st>>>(maps->fmap, maps->mmap, d, f, mo, om, kz);
    };
    if (math == kMathDouble) launch(k_streamcoll_tma<Lat, T, double, VX>, om1d);
    else launch(k_streamcoll_tma<Lat, T, float, VX>, om1f);
  };
  switch (lat) {
    case kD2Q9: go(D2Q9{}); break;
    case kD3Q19: go(D3Q19{}); break;
    case kD3Q27: go(D3Q27{}); break;
  }
  return 0;
}


template <typename T>
int launch_streamcoll_tma(int lat, int math, const Dom& d, T* f, const T* mo, double omega, int kz, int vx,
                          TmaMaps*& maps, cudaStream_t st) {
  if (vx <= 0) vx = 1;
  if (vx > 2 || vx * int(sizeof(T)) > 8) return 1;
  return vx == 1 ? launch_tma_vx<T, 1>(lat, math, d, f, mo, omega, kz, maps, st)
                 : launch_tma_vx<T, 2>(lat, math, d, f, mo, omega, kz, maps, st);
}

template int launch_streamcoll_tma<float>(int, int, const Dom&, float*, const float*, double, int, int, TmaMaps*&,
                                          cudaStream_t);
template int launch_streamcoll_tma<double>(int, int, const Dom&, double*, const double*, double, int, int, TmaMaps*&,
                                           cudaStream_t);

}  // namespace tslb_cuda
