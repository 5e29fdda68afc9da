// Storage codecs of the moment arrays the M kernel reads and writes.
//
// MStore<T>: the identity -- moments stored in the storage type T (fp32 or
// fp64), every reference-parity path.
//
// MStore<__half>: the mixed-precision mode (the paper's
// outlook, PAPER.md:479, 485 -- half-precision storage, single-precision
// arithmetic). Each moment array is stored as IEEE fp16 of a shifted and
// scaled value, (m_c - off_c) * sc_c, with power-of-two scales chosen so the
// lattice-Boltzmann magnitudes sit in fp16's normal range:
//   rho   : (rho - 1) * 2^10     (density fluctuations ~1e-6 .. 1e-1)
//   j     : j * 2^4               (|u| up to 4000, Mach-scale values ~0.01 .. 0.3)
//   Pi^neq: Pi * 2^12             (|Pi| up to 16, typical 1e-7 .. 1e-2)
// The scale is exact (power of two), so the decode m = h / sc + off rounds
// once, in fp32. 20 B per node for the ten D3Q19 moments, 40 B per lattice
// update for the M step (80 B at fp32). A tolerance mode (tests state it):
// the node arithmetic runs in fp32.
#pragma once

#include <cuda_fp16.h>

#include <cstdint>

namespace tslb_cuda {

template <typename TM>
struct MStore {
  using W = TM;  // staging word of a lane-fetched halo element
  __host__ __device__ static TM dec(int, TM v) { return v; }
  template <typename V>
  __host__ __device__ static TM enc(int, V v) {
    return TM(v);
  }
  __device__ static TM pick(W w, int) { return w; }
  __device__ static int sel(int64_t) { return 0; }
  __device__ static const W* word(const TM* p) { return p; }
};

template <>
struct MStore<__half> {
  // cp.async moves 4, 8 or 16 bytes: a halo element is fetched as the
  // aligned 4-byte word that contains it (all array bases, strides and plane
  // sizes are even, so the half is picked by the node index's parity)
  using W = uint32_t;
  __host__ __device__ static constexpr float off(int c) { return c == 0 ? 1.0f : 0.0f; }
  __host__ __device__ static constexpr float sc(int c) { return c == 0 ? 1024.0f : c < 4 ? 16.0f : 4096.0f; }
  __device__ static float dec(int c, __half h) { return fmaf(__half2float(h), 1.0f / sc(c), off(c)); }
  __device__ static __half enc(int c, float v) { return __float2half_rn((v - off(c)) * sc(c)); }
  __device__ static __half pick(uint32_t w, int sel) {
    return __ushort_as_half(static_cast<unsigned short>(sel ? (w >> 16) : (w & 0xffffu)));
  }
  __device__ static int sel(int64_t node) { return int(node & 1); }
  __device__ static const uint32_t* word(const __half* p) {
    return reinterpret_cast<const uint32_t*>(reinterpret_cast<uintptr_t>(p) & ~uintptr_t(3));
  }
};

}  // namespace tslb_cuda
