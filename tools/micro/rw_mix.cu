// HBM bandwidth of streaming kernels with a given read:write array mix
// (measurement only): R arrays read, W arrays written, n floats each,
// scalar 4-byte accesses per thread (the access shape of the population
// kernels) or 8- / 16-byte vectors. Prints GB/s of (R + W) * n * 4 bytes per
// launch, best of 10, CUDA events.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o rw_mix rw_mix.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

constexpr int kMax = 40;
struct Ptrs {
  const float* r[kMax];
  float* w[kMax];
};

template <int R, int W>
__global__ void __launch_bounds__(256) k_mix4(Ptrs p, long n4) {
  for (long i = blockIdx.x * 256L + threadIdx.x; i < n4; i += long(gridDim.x) * 256) {
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int a = 0; a < R; ++a) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(p.r[a]) + i);
      s.x += v.x, s.y += v.y, s.z += v.z, s.w += v.w;
    }
#pragma unroll
    for (int b = 0; b < W; ++b) reinterpret_cast<float4*>(p.w[b])[i] = make_float4(s.x + b, s.y, s.z, s.w);
  }
}

template <int R, int W>
__global__ void __launch_bounds__(256) k_mix2(Ptrs p, long n2) {
  for (long i = blockIdx.x * 256L + threadIdx.x; i < n2; i += long(gridDim.x) * 256) {
    float2 s = make_float2(0.f, 0.f);
#pragma unroll
    for (int a = 0; a < R; ++a) {
      const float2 v = __ldg(reinterpret_cast<const float2*>(p.r[a]) + i);
      s.x += v.x, s.y += v.y;
    }
#pragma unroll
    for (int b = 0; b < W; ++b) reinterpret_cast<float2*>(p.w[b])[i] = make_float2(s.x + b, s.y);
  }
}

// scalar accesses, two elements per thread (a warp covers 64 consecutive
// elements with two 128-byte accesses per array)
template <int R, int W>
__global__ void __launch_bounds__(256) k_mixu2(Ptrs p, long n) {
  const int lane = threadIdx.x & 31;
  for (long w = (blockIdx.x * 256L + threadIdx.x) >> 5; w * 64 < n; w += long(gridDim.x) * 8) {
    const long i = w * 64 + lane;
    float s0 = 0.f, s1 = 0.f;
#pragma unroll
    for (int a = 0; a < R; ++a) {
      s0 += __ldg(p.r[a] + i);
      s1 += __ldg(p.r[a] + i + 32);
    }
#pragma unroll
    for (int b = 0; b < W; ++b) {
      p.w[b][i] = s0 + float(b);
      p.w[b][i + 32] = s1;
    }
  }
}

template <int R, int W>
__global__ void __launch_bounds__(256) k_mix(Ptrs p, long n) {
  for (long i = blockIdx.x * 256L + threadIdx.x; i < n; i += long(gridDim.x) * 256) {
    float s = 0.f;
#pragma unroll
    for (int a = 0; a < R; ++a) s += __ldg(p.r[a] + i);
#pragma unroll
    for (int b = 0; b < W; ++b) p.w[b][i] = s + float(b);
    if (W == 0 && s == -1.f) p.w[0][i] = s;  // (never: keeps the reads of the read-only case)
  }
}

template <int R, int W, int V = 1>
void run(long n, float** bufs, int sms) {
  Ptrs p{};
  for (int a = 0; a < R; ++a) p.r[a] = bufs[a];
  for (int b = 0; b < W || b < 1; ++b) p.w[b] = bufs[R + b];
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int grid = sms * 8;
  float best = 1e30f;
  for (int it = 0; it < 12; ++it) {
    cudaEventRecord(e0);
    if (V == 4) k_mix4<R, W><<<grid, 256>>>(p, n / 4);
    else if (V == 2) k_mix2<R, W><<<grid, 256>>>(p, n / 2);
    else if (V == -2) k_mixu2<R, W><<<grid, 256>>>(p, n);
    else k_mix<R, W><<<grid, 256>>>(p, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (it >= 2 && ms < best) best = ms;
  }
  const double bytes = double(R + W) * n * 4;
  printf("{\"reads\": %d, \"writes\": %d, \"vector\": %d, \"bytes\": %.0f, \"ms\": %.4f, \"gbs\": %.1f}\n", R, W, V, bytes, best,
         bytes / best / 1e6);
}

int main(int argc, char** argv) {
  const long n = argc > 1 ? atol(argv[1]) : (64L << 20);  // floats per array (256 MB)
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  float* bufs[kMax * 2];
  for (int i = 0; i < 52; ++i) {
    if (cudaMalloc(&bufs[i], n * 4) != cudaSuccess) {
      printf("alloc failed\n");
      return 1;
    }
    cudaMemset(bufs[i], 0, n * 4);
  }
  run<1, 1>(n, bufs, sms);    // copy
  run<2, 2>(n, bufs, sms);
  run<1, 3>(n, bufs, sms);    // write-heavy
  run<13, 38>(n, bufs, sms);  // the recolouring kernel's mix (52 B in, 152 B out per node)
  run<38, 13>(n, bufs, sms);  // the colour-moments kernel's mix
  run<0, 1>(n, bufs, sms);    // write only
  run<1, 0>(n, bufs, sms);    // read only
  run<13, 38, -2>(n, bufs, sms);  // scalar, two elements per thread
  run<1, 3, 2>(n, bufs, sms);  // 8-byte accesses
  run<13, 38, 2>(n, bufs, sms);
  run<1, 1, 4>(n, bufs, sms);  // 16-byte accesses
  run<1, 3, 4>(n, bufs, sms);
  run<13, 38, 4>(n, bufs, sms);
  run<38, 13, 4>(n, bufs, sms);
  return 0;
}
