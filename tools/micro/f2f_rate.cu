// Issue rates of the fp64 instructions the bit-exact M kernel lives on
// (measurement only): F2F.F64.F32 (cvt.f64.f32), F2F.F32.F64
// (cvt.rn.f32.f64), DADD, and mixes, as thread-instructions per clock per
// SM. 8 independent chains per thread, full occupancy, CUDA events.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o f2f_rate f2f_rate.cu
#include <cuda_runtime.h>

#include <cstdio>

constexpr int kIters = 4096;

template <int MODE>
__global__ void __launch_bounds__(256) k_rate(float* out, double* outd) {
  float f[8];
  double d[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    f[c] = 1.0f + 1e-3f * float(threadIdx.x + c);
    d[c] = 1.0 + 1e-6 * double(threadIdx.x + c);
  }
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (MODE == 0) {  // widen + narrow: 2 F2F
        double t;
        asm volatile("cvt.f64.f32 %0, %1;" : "=d"(t) : "f"(f[c]));
        asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(f[c]) : "d"(t));
      } else if (MODE == 1) {  // 2 DADD
        asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(d[c]) : "d"(d[(c + 1) & 7]));
        asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(d[c]) : "d"(d[(c + 3) & 7]));
      } else if (MODE == 2) {  // 1 F2F.F64.F32 + 1 DADD
        double t;
        asm volatile("cvt.f64.f32 %0, %1;" : "=d"(t) : "f"(f[c]));
        asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(d[c]) : "d"(t));
      } else if (MODE == 3) {  // 2 widen only
        double t, u;
        asm volatile("cvt.f64.f32 %0, %1;" : "=d"(t) : "f"(f[c]));
        asm volatile("cvt.f64.f32 %0, %1;" : "=d"(u) : "f"(f[(c + 1) & 7]));
        d[c] += 0.0 * (t + u);  // (kept; not counted)
      } else if (MODE == 4) {  // 2 narrow, inputs perturbed by an integer op (ALU)
        float g, h;
        asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(g) : "d"(d[c]));
        asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(h) : "d"(d[(c + 1) & 7]));
        d[c] = __longlong_as_double(__double_as_longlong(d[c]) ^ (long long)(__float_as_int(g) & 1));
        f[c] = __int_as_float(__float_as_int(f[c]) ^ (__float_as_int(h) & 1));
      } else {  // 2 widen, inputs perturbed by an integer op
        double t, u;
        asm volatile("cvt.f64.f32 %0, %1;" : "=d"(t) : "f"(f[c]));
        asm volatile("cvt.f64.f32 %0, %1;" : "=d"(u) : "f"(f[(c + 1) & 7]));
        f[c] = __int_as_float(__float_as_int(f[c]) ^ int(__double_as_longlong(t) & 1) ^ int(__double_as_longlong(u) & 2));
      }
    }
  }
  float s = 0.f;
  double sd = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += f[c], sd += d[c];
  out[blockIdx.x * 256 + threadIdx.x] = s;
  outd[blockIdx.x * 256 + threadIdx.x] = sd;
}

template <int MODE>
void run(const char* name, int sms, int clk_khz, float* o, double* od) {
  const int grid = sms * 8;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k_rate<MODE><<<grid, 256>>>(o, od);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double ops = double(grid) * 256 * kIters * 8 * 2;  // two counted instructions per chain step
  const double clk = double(clk_khz) * 1e3 * best * 1e-3;  // (at the max clock; the run may be slower)
  printf("{\"mode\": \"%s\", \"ms\": %.4f, \"thread_ops_per_clk_per_sm\": %.2f}\n", name, best, ops / clk / sms);
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* o;
  double* od;
  cudaMalloc(&o, sms * 8 * 256 * 4);
  cudaMalloc(&od, sms * 8 * 256 * 8);
  run<0>("F2F.F64.F32 + F2F.F32.F64", sms, clk, o, od);
  run<1>("DADD x2", sms, clk, o, od);
  run<2>("F2F.F64.F32 + DADD", sms, clk, o, od);
  run<3>("F2F.F64.F32 x2 (results barely used)", sms, clk, o, od);
  run<4>("F2F.F32.F64 x2 (+2 LOP3)", sms, clk, o, od);
  run<5>("F2F.F64.F32 x2 (+LOP3)", sms, clk, o, od);
  printf("{\"sms\": %d, \"clock_khz\": %d}\n", sms, clk);
  return 0;
}
