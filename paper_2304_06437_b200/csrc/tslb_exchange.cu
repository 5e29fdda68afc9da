// Slab-interface unpack for masked geometries.
//
// With solids present, a ghost-plane slot is written by the neighbour only if
// its source node (in the neighbour's boundary plane) is fluid and the push
// did not cross a wall face; every other slot of the received plane is stale.
// Received planes are therefore staged and copied into the owned boundary
// plane only where the sender really wrote -- preserving the one-writer-per-
// slot rule (kernels.hpp:149-153) across GPUs. Unmasked boxes receive in
// place and never launch this kernel.
#include <cstdint>

#include "tslb_domain.cuh"
#include "tslb_kernels.h"

namespace tslb_cuda {

struct UnpackDirs {
  int n;
  int a[9], cx[9], cy[9];
};

template <typename T>
__global__ void k_unpack(Dom d, T* __restrict__ f, const T* __restrict__ recv,
                         const uint8_t* __restrict__ solid, UnpackDirs dirs,
                         int kdst, int ksrc_ghost) {
  const int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= d.plane) return;
  const int i = int(p % d.nx), j = int(p / d.nx);
  for (int e = 0; e < dirs.n; ++e) {
    // source node of slot (i, j) along direction a, in the ghost plane
    int si = i - dirs.cx[e], sj = j - dirs.cy[e];
    bool ok = true;
    if (si < 0 || si >= d.nx) {
      const int face = si < 0 ? XMin : XMax;
      if (d.mode[face] == kWrap) si = si < 0 ? si + d.nx : si - d.nx;
      else ok = false;  // the sender bounced instead of pushing
    }
    if (sj < 0 || sj >= d.ny) {
      const int face = sj < 0 ? YMin : YMax;
      if (d.mode[face] == kWrap) sj = sj < 0 ? sj + d.ny : sj - d.ny;
      else ok = false;
    }
    if (ok && solid[fidx(d, si, sj, ksrc_ghost)]) ok = false;
    if (ok && !solid[fidx(d, i, j, kdst)])
      f[dirs.a[e] * d.fstride + fidx(d, i, j, kdst)] = recv[e * d.plane + p];
  }
}

template <typename T>
int launch_unpack(const Dom& d, T* f, const T* recv, const uint8_t* solid,
                  int ndirs, const int* a, const int* cx, const int* cy,
                  int kdst, int ksrc_ghost, cudaStream_t st) {
  UnpackDirs u{};
  u.n = ndirs;
  for (int e = 0; e < ndirs; ++e) {
    u.a[e] = a[e];
    u.cx[e] = cx[e];
    u.cy[e] = cy[e];
  }
  k_unpack<T><<<unsigned((d.plane + 255) / 256), 256, 0, st>>>(
      d, f, recv, solid, u, kdst, ksrc_ghost);
  return 0;
}

template int launch_unpack<float>(const Dom&, float*, const float*,
                                  const uint8_t*, int, const int*, const int*,
                                  const int*, int, int, cudaStream_t);
template int launch_unpack<double>(const Dom&, double*, const double*,
                                   const uint8_t*, int, const int*, const int*,
                                   const int*, int, int, cudaStream_t);

// ---------------------------------------------------------------------------
// Peer-memory halo transport (CUDA IPC, one process per GPU): after a rank
// has copied its new boundary planes into a neighbour's ghost buffer, one
// thread publishes the exchange number into the neighbour's flag word (a
// system-scope release store behind a system fence); before the ghost planes
// are read, one thread of the consumer's stream waits for the number with
// acquire loads. A neighbour that never arrives traps after 60 s (a sticky
// launch failure the host reports) instead of hanging the device.
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void k_ipc_signal(uint64_t* a, uint64_t* b, uint64_t v) {
  __threadfence_system();
  if (a) st_release_sys(a, v);
  if (b) st_release_sys(b, v);
}

__global__ void k_ipc_wait(const uint64_t* a, const uint64_t* b, uint64_t v) {
  const uint64_t t0 = global_ns();
  for (;;) {
    const bool ok = (!a || ld_acquire_sys(a) >= v) && (!b || ld_acquire_sys(b) >= v);
    if (ok) return;
    if (global_ns() - t0 > 60ull * 1000000000ull) __trap();
    __nanosleep(500);
  }
}

int launch_ipc_signal(uint64_t* a, uint64_t* b, uint64_t v, cudaStream_t st) {
  k_ipc_signal<<<1, 1, 0, st>>>(a, b, v);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int launch_ipc_wait(const uint64_t* a, const uint64_t* b, uint64_t v, cudaStream_t st) {
  k_ipc_wait<<<1, 1, 0, st>>>(a, b, v);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace tslb_cuda
