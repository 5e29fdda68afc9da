// Device-side diagnostics: deterministic fp64 tree reductions (totals,
// colour masses, stability scan) and the chunked FNV-1a state digest.
//
// Reference counterparts are serial host scans (solver.hpp:39-65, 104-113,
// 172-181; bench.hpp:83-109). Reductions here use a FIXED launch shape and a
// fixed combine order, so they are bit-reproducible run to run; they are not
// bit-identical to the reference's serial T-precision sums (tests hold a
// stated tolerance).
#include <cstdint>

#include "tslb_domain.cuh"
#include "tslb_kernels.h"

namespace tslb_cuda {

constexpr int RB = 256;        // threads per reduction block
constexpr int RBLOCKS = 592;   // 4 x 148 SMs; fixed => deterministic order
constexpr int RSLOTS = 7;      // doubles per partial

size_t reduce_partial_count() { return size_t(RBLOCKS) * RSLOTS; }

template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* sh) {
  // fixed-shape tree: warp shuffles then one warp over the warp results
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < NV; ++c) {
    double x = v[c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if (lane == 0) sh[c * (RB / 32) + w] = x;
  }
  __syncthreads();
  if (w == 0) {
#pragma unroll
    for (int c = 0; c < NV; ++c) {
      double x = lane < RB / 32 ? sh[c * (RB / 32) + lane] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
      v[c] = x;
    }
  }
}

// Owned-node linear index -> (mi, fi)
__device__ __forceinline__ void owned(const Dom& d, int64_t t, int64_t& mi,
                                      int64_t& fi) {
  mi = t;
  fi = t + int64_t(d.ghost) * d.plane;
}

template <typename T, int DIM>
__global__ void __launch_bounds__(RB)
    k_totals(Dom d, const T* __restrict__ rho, const T* __restrict__ mom,
             const uint8_t* __restrict__ solid, double* partial) {
  __shared__ double sh[4 * (RB / 32)];
  double v[4] = {0, 0, 0, 0};
  // contiguous chunk per block, strided per thread: fixed assignment. The
  // loads are unconditional (solid nodes are skipped in the sums only), so
  // with the unrolled loop four iterations' loads are in flight together
  const int64_t per = (d.n + RBLOCKS - 1) / RBLOCKS;
  const int64_t b0 = int64_t(blockIdx.x) * per;
  const int64_t b1 = min(d.n, b0 + per);
#pragma unroll 4
  for (int64_t t = b0 + threadIdx.x; t < b1; t += RB) {
    int64_t mi, fi;
    owned(d, t, mi, fi);
    const bool sol = solid[fi] != 0;
    const double r = double(rho[mi]);
    double m[DIM];
#pragma unroll
    for (int c = 0; c < DIM; ++c) m[c] = double(mom[c * d.mstride + mi]);
    if (sol) continue;
    v[0] += r;
#pragma unroll
    for (int c = 0; c < DIM; ++c) v[1 + c] += m[c];
  }
  block_sum<4>(v, sh);
  if (threadIdx.x == 0)
    for (int c = 0; c < 4; ++c) partial[blockIdx.x * RSLOTS + c] = v[c];
}

__global__ void k_fold_sum(const double* partial, int nslots, double* out) {
  // one thread, fixed order
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  for (int c = 0; c < nslots; ++c) {
    double s = 0;
    for (int b = 0; b < RBLOCKS; ++b) s += partial[b * RSLOTS + c];
    out[c] = s;
  }
}

// scan_stability (solver.hpp:39-65). min/max are order-independent except
// for NaN: the reference's std::min/std::max keep a NaN only when it is the
// FIRST fluid node's rho (every later comparison with it is false), and
// drop later NaNs -- so the scan also carries the first fluid node (lowest
// index) and its rho; with no fluid node at all min = max = 0.
template <typename T>
__global__ void __launch_bounds__(RB)
    k_stability(Dom d, int dim, const T* __restrict__ rho,
                const T* __restrict__ mom, const uint8_t* __restrict__ solid,
                double* partial) {
  __shared__ double sh[7 * (RB / 32)];
  double bad = 0, mx = 0, lo = 1e300, hi = -1e300, first = 1e300, ffirst = 1e300, frho = 0;
  const int64_t per = (d.n + RBLOCKS - 1) / RBLOCKS;
  const int64_t b0 = int64_t(blockIdx.x) * per;
  const int64_t b1 = min(d.n, b0 + per);
  // (unrolled: the loads of four iterations are in flight together; the
  // accumulation order is unchanged)
#pragma unroll 4
  for (int64_t t = b0 + threadIdx.x; t < b1; t += RB) {
    int64_t mi, fi;
    owned(d, t, mi, fi);
    if (solid[fi]) continue;
    T u2 = T(0);
    for (int c = 0; c < dim; ++c) {
      const T m = mom[c * d.mstride + mi];
      u2 += m * m;
    }
    const T r = rho[mi];
    if (ffirst > 1e299) {  // (t ascends per thread)
      ffirst = double(t);
      frho = double(r);
    }
    if (!isfinite(double(r)) || !isfinite(double(u2))) {
      bad = 1;
      first = fmin(first, double(t));
    }
    const double sp = double(sqrt(u2));
    mx = fmax(mx, sp);
    lo = fmin(lo, double(r));
    hi = fmax(hi, double(r));
  }
  // min/max are order-independent: reduce with shuffles; the first fluid
  // node travels with its rho
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) {
    bad = fmax(bad, __shfl_down_sync(0xffffffffu, bad, o));
    mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, o));
    lo = fmin(lo, __shfl_down_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_down_sync(0xffffffffu, hi, o));
    first = fmin(first, __shfl_down_sync(0xffffffffu, first, o));
    const double of = __shfl_down_sync(0xffffffffu, ffirst, o);
    const double orh = __shfl_down_sync(0xffffffffu, frho, o);
    if (of < ffirst) {
      ffirst = of;
      frho = orh;
    }
  }
  if (lane == 0) {
    sh[w] = bad;
    sh[8 + w] = mx;
    sh[16 + w] = lo;
    sh[24 + w] = hi;
    sh[32 + w] = first;
    sh[40 + w] = ffirst;
    sh[48 + w] = frho;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < RB / 32; ++k) {
      bad = fmax(bad, sh[k]);
      mx = fmax(mx, sh[8 + k]);
      lo = fmin(lo, sh[16 + k]);
      hi = fmax(hi, sh[24 + k]);
      first = fmin(first, sh[32 + k]);
      if (sh[40 + k] < ffirst) {
        ffirst = sh[40 + k];
        frho = sh[48 + k];
      }
    }
    double* p = partial + blockIdx.x * RSLOTS;
    p[0] = bad;
    p[1] = mx;
    p[2] = lo;
    p[3] = hi;
    p[4] = first;
    p[5] = ffirst;
    p[6] = frho;
  }
}

__global__ void k_fold_stability(const double* partial, double* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double bad = 0, mx = 0, lo = 1e300, hi = -1e300, first = 1e300, ffirst = 1e300, frho = 0;
  for (int b = 0; b < RBLOCKS; ++b) {
    const double* p = partial + b * RSLOTS;
    bad = fmax(bad, p[0]);
    mx = fmax(mx, p[1]);
    lo = fmin(lo, p[2]);
    hi = fmax(hi, p[3]);
    first = fmin(first, p[4]);
    if (p[5] < ffirst) {
      ffirst = p[5];
      frho = p[6];
    }
  }
  if (ffirst > 1e299) {
    lo = hi = 0.0;  // no fluid node: the report's zero-initialised fields
  } else if (isnan(frho)) {
    lo = hi = frho;  // the reference's min/max stay at a NaN first value
  }
  out[0] = bad > 0 ? 0.0 : 1.0;  // finite flag
  out[1] = mx;
  out[2] = lo;
  out[3] = hi;
  out[4] = first < 1e299 ? first : -1.0;
}

template <typename T>
int launch_totals(const Dom& d, int dim, const T* rho, const T* mom,
                  const uint8_t* solid, double* partial, double* out,
                  cudaStream_t st) {
  if (dim == 3) k_totals<T, 3><<<RBLOCKS, RB, 0, st>>>(d, rho, mom, solid, partial);
  else k_totals<T, 2><<<RBLOCKS, RB, 0, st>>>(d, rho, mom, solid, partial);
  k_fold_sum<<<1, 32, 0, st>>>(partial, 4, out);
  return 0;
}

template <typename T>
int launch_stability(const Dom& d, int dim, const T* rho, const T* mom,
                     const uint8_t* solid, double* partial, double* out,
                     cudaStream_t st) {
  k_stability<T><<<RBLOCKS, RB, 0, st>>>(d, dim, rho, mom, solid, partial);
  k_fold_stability<<<1, 32, 0, st>>>(partial, out);
  return 0;
}

// ---------------------------------------------------------------------------
// chunked FNV-1a digest: chunk = 16 KiB of a plane; plane hash = FNV-1a over
// its chunk hashes (little-endian u64 bytes); the host folds plane hashes in
// (array, z) order, so the value is independent of slab decomposition.
constexpr int64_t kChunk = 16384;
constexpr uint64_t kFnvBasis = 0xcbf29ce484222325ull;
constexpr uint64_t kFnvPrime = 0x100000001b3ull;

__device__ __forceinline__ uint64_t fnv_bytes(uint64_t h, uint32_t w, int nb) {
  for (int b = 0; b < nb; ++b) {
    h ^= (w >> (8 * b)) & 0xffu;
    h *= kFnvPrime;
  }
  return h;
}

__global__ void k_chunk_hash(const uint8_t* __restrict__ base, int narrays,
                             int64_t stride_bytes, int64_t first_bytes,
                             int nz, int64_t plane_bytes, int64_t cpp,
                             uint64_t* __restrict__ out) {
  const int64_t id = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t total = int64_t(narrays) * nz * cpp;
  if (id >= total) return;
  const int64_t c = id % cpp;
  const int64_t pk = id / cpp;  // plane linear (a * nz + k)
  const int64_t a = pk / nz, k = pk % nz;
  const uint8_t* p = base + a * stride_bytes + first_bytes + k * plane_bytes +
                     c * kChunk;
  const int64_t len = min(kChunk, plane_bytes - c * kChunk);
  uint64_t h = kFnvBasis;
  int64_t o = 0;
  if ((reinterpret_cast<uintptr_t>(p) & 3) == 0) {
    for (; o + 4 <= len; o += 4)
      h = fnv_bytes(h, *reinterpret_cast<const uint32_t*>(p + o), 4);
  }
  for (; o < len; ++o) {
    h ^= p[o];
    h *= kFnvPrime;
  }
  out[id] = h;
}

__global__ void k_plane_fold(const uint64_t* __restrict__ chunks, int64_t nplanes,
                             int64_t cpp, uint64_t* __restrict__ out) {
  const int64_t pk = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (pk >= nplanes) return;
  uint64_t h = kFnvBasis;
  for (int64_t c = 0; c < cpp; ++c) {
    const uint64_t v = chunks[pk * cpp + c];
    h = fnv_bytes(h, uint32_t(v), 4);
    h = fnv_bytes(h, uint32_t(v >> 32), 4);
  }
  out[pk] = h;
}

int launch_plane_digest(const Dom& d, const void* arr, int narrays,
                        int64_t stride, int64_t base, int elem_bytes,
                        uint64_t* chunk_scratch, uint64_t* out,
                        cudaStream_t st) {
  const int64_t plane_bytes = d.plane * elem_bytes;
  const int64_t cpp = (plane_bytes + kChunk - 1) / kChunk;
  const int64_t total = int64_t(narrays) * d.nz * cpp;
  k_chunk_hash<<<unsigned((total + 127) / 128), 128, 0, st>>>(
      static_cast<const uint8_t*>(arr), narrays, stride * elem_bytes,
      base * elem_bytes, d.nz, plane_bytes, cpp, chunk_scratch);
  const int64_t np = int64_t(narrays) * d.nz;
  k_plane_fold<<<unsigned((np + 127) / 128), 128, 0, st>>>(chunk_scratch, np,
                                                           cpp, out);
  return 0;
}

template int launch_totals<float>(const Dom&, int, const float*, const float*,
                                  const uint8_t*, double*, double*, cudaStream_t);
template int launch_totals<double>(const Dom&, int, const double*, const double*,
                                   const uint8_t*, double*, double*, cudaStream_t);
template int launch_stability<float>(const Dom&, int, const float*, const float*,
                                     const uint8_t*, double*, double*, cudaStream_t);
template int launch_stability<double>(const Dom&, int, const double*,
                                      const double*, const uint8_t*, double*,
                                      double*, cudaStream_t);

}  // namespace tslb_cuda
