// MUFU.EX2 stream of one warp per SMSP with the softmax's companion
// instructions (sm_100a): cycles per MUFU for 128 exps per thread.
//   mode 0: ex2 only (inputs in registers)
//   mode 1: FFMA2 (x = s*scale - m) feeding the ex2 pairs
//   mode 2: mode 1 + F2FP pack of each pair
//   mode 3: mode 2 + FADD2 row-sum accumulation (4 chains)
//   mode 4: mode 2 with the FFMA2s of the whole row issued first
//   mode 5: FFMA2 -> F2FP (x to bf16x2) -> packed ex2.approx.ftz.bf16x2
//   mode 6: FFMA2 -> F2FP (x to f16x2) -> packed ex2.approx.f16x2
//   (cycles are per element exp in every mode)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2603_01960_b200/csrc \
//        -o /tmp/mbm scripts/microbench_mufu_mix.cu && /tmp/mbm
#include <cstdio>
#include "ptx_sm100.cuh"
using namespace ta;
constexpr int kReps = 64;
// volatile versions: nothing may be hoisted out of the repetition loop
__device__ __forceinline__ float vex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint64_t vffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint32_t vpack(float lo, float hi) {
  uint32_t r;
  asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ uint32_t vex2_bf16x2(uint32_t x) {
  uint32_t y;
  asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ uint32_t vex2_f16x2(uint32_t x) {
  uint32_t y;
  asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ uint32_t vpack_f16(float lo, float hi) {
  uint32_t r;
  asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ uint64_t vfadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) bench(const float* in, long long* cycles, uint32_t* sink) {
  float s[128];
  for (int i = 0; i < 128; ++i) s[i] = in[(threadIdx.x * 131 + i) & 1023];
  const float sl2 = in[1], m = in[2];
  const uint64_t sl2x2 = f2(sl2, sl2);
  uint32_t acc_pk = 0;
  uint64_t acc[4] = {0, 0, 0, 0};
  __syncwarp();
  long long t0 = clock64();
  for (int rep = 0; rep < kReps; ++rep) {
    const float mr = m + float(rep) * 1e-6f;  // per-repetition input: nothing is loop-invariant
    const uint64_t negm2 = f2(-mr, -mr);
    if constexpr (MODE == 4) {
      uint64_t x[64];
#pragma unroll
      for (int u = 0; u < 64; ++u) x[u] = vffma2(f2(s[2 * u], s[2 * u + 1]), sl2x2, negm2);
#pragma unroll
      for (int u = 0; u < 64; ++u) {
        float a, b;
        f2_split(x[u], a, b);
        const float p0 = vex2(a), p1 = vex2(b);
        acc_pk ^= vpack(p0, p1);
      }
    } else if constexpr (MODE == 5 || MODE == 6) {
#pragma unroll
      for (int u = 0; u < 64; ++u) {
        float a, b;
        f2_split(vffma2(f2(s[2 * u], s[2 * u + 1]), sl2x2, negm2), a, b);
        acc_pk ^= MODE == 5 ? vex2_bf16x2(vpack(a, b)) : vex2_f16x2(vpack_f16(a, b));
      }
    } else {
#pragma unroll
      for (int u = 0; u < 64; ++u) {
        float a, b;
        if constexpr (MODE == 0) {
          a = s[2 * u] - mr;
          b = s[2 * u + 1] - mr;
        } else {
          f2_split(vffma2(f2(s[2 * u], s[2 * u + 1]), sl2x2, negm2), a, b);
        }
        const float p0 = vex2(a), p1 = vex2(b);
        if constexpr (MODE >= 2) acc_pk ^= vpack(p0, p1);
        else acc_pk ^= __float_as_uint(p0) ^ __float_as_uint(p1);
        if constexpr (MODE == 3) acc[u & 3] = vfadd2(acc[u & 3], f2(p0, p1));
      }
    }
    // feed the outputs back so iterations depend on each other minimally
  }
  long long t1 = clock64();
  if (threadIdx.x % 32 == 0) cycles[blockIdx.x * 16 + threadIdx.x / 32] = t1 - t0;
  sink[blockIdx.x * 512 + threadIdx.x] = acc_pk ^ uint32_t(acc[0] ^ acc[1] ^ acc[2] ^ acc[3]);
}

template <int MODE>
void run(const char* name, int warps_per_smsp, const float* in, long long* cyc, uint32_t* sink) {
  const int threads = 128 * warps_per_smsp;
  bench<MODE><<<148, threads>>>(in, cyc, sink);
  cudaDeviceSynchronize();
  bench<MODE><<<148, threads>>>(in, cyc, sink);
  cudaError_t e = cudaDeviceSynchronize();
  long long c[148 * 16];
  cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int b = 0; b < 148; ++b)
    for (int w = 0; w < 4 * warps_per_smsp; ++w) avg += c[b * 16 + w];
  avg /= 148 * 4 * warps_per_smsp;
  printf("%-40s warps/SMSP %d: %6.2f cyc per MUFU per warp (%.2f per SMSP) %s\n", name,
         warps_per_smsp, avg / (kReps * 128.0), avg / (kReps * 128.0) / warps_per_smsp,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  float* in;
  long long* cyc;
  uint32_t* sink;
  cudaMalloc(&in, 1024 * 4);
  float h[1024];
  for (int i = 0; i < 1024; ++i) h[i] = -float(i % 17) * 0.25f;
  h[1] = 0.1275f;
  h[2] = 0.5f;
  cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaMalloc(&cyc, 148 * 16 * sizeof(long long));
  cudaMalloc(&sink, 148 * 512 * 4);
  for (int w = 1; w <= 4; w *= 2) {
    run<0>("ex2 only", w, in, cyc, sink);
    run<1>("FFMA2 -> ex2 pair", w, in, cyc, sink);
    run<2>("FFMA2 -> ex2 pair -> F2FP", w, in, cyc, sink);
    run<3>("... + FADD2 row sum", w, in, cyc, sink);
    run<4>("all FFMA2 first, then ex2 + F2FP", w, in, cyc, sink);
    run<5>("FFMA2 -> F2FP -> ex2.bf16x2 (per elem)", w, in, cyc, sink);
    run<6>("FFMA2 -> F2FP -> ex2.f16x2 (per elem)", w, in, cyc, sink);
  }
  return 0;
}
