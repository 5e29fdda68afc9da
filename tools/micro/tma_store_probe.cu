// Probe: which innermost coordinates may a TMA tensor STORE / LOAD use?
// usage: tma_store_probe <coord> <load|store> ; exit 0 = ok, prints result
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__global__ void k(const __grid_constant__ CUtensorMap map, int c, int load) {
  __shared__ __align__(128) float buf[256];
  __shared__ __align__(8) unsigned long long bar;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) buf[i] = float(i + 1);
  uint32_t sb = static_cast<uint32_t>(__cvta_generic_to_shared(buf));
  uint32_t bb = static_cast<uint32_t>(__cvta_generic_to_shared(&bar));
  __syncthreads();
  if (threadIdx.x == 0) {
    if (load) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bb));
      asm volatile("fence.proxy.async.shared::cta;");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bb), "r"(1024));
      asm volatile("cp.async.bulk.tensor.1d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3}], [%2];"
                   ::"r"(sb), "l"(reinterpret_cast<uint64_t>(&map)), "r"(bb), "r"(c) : "memory");
      uint32_t done = 0;
      do {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p; }"
                     : "=r"(done) : "r"(bb) : "memory");
      } while (!done);
    } else {
      asm volatile("fence.proxy.async.shared::cta;");
      asm volatile("cp.async.bulk.tensor.1d.global.shared::cta.bulk_group [%0, {%2}], [%1];"
                   ::"l"(reinterpret_cast<uint64_t>(&map)), "r"(sb), "r"(c) : "memory");
      asm volatile("cp.async.bulk.commit_group;");
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
  }
}

int main(int argc, char** argv) {
  int c = atoi(argv[1]);
  int load = argc > 2 && argv[2][0] == 'l';
  float* g;
  cudaMalloc(&g, 4096 * 4);
  cudaMemset(g, 0, 4096 * 4);
  void* p;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  CUtensorMap map;
  cuuint64_t dim[1] = {1024};
  cuuint64_t str[1] = {4096};
  cuuint32_t box[1] = {256}, es[1] = {1};
  CUresult r = reinterpret_cast<EncodeFn>(p)(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 1, g, dim, str, box, es,
                                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  k<<<1, 128>>>(map, c, load);
  cudaError_t e = cudaDeviceSynchronize();
  float h[1024];
  cudaMemcpy(h, g, sizeof h, cudaMemcpyDeviceToHost);
  int first = -1, last = -1;
  for (int i = 0; i < 1024; ++i)
    if (h[i] != 0) { if (first < 0) first = i; last = i; }
  printf("%s coord %d: encode=%d kernel=%s written=[%d,%d] h[first]=%g\n", load ? "load" : "store", c, int(r),
         cudaGetErrorString(e), first, last, first >= 0 ? h[first] : 0.f);
  return e != cudaSuccess;
}
