// Pipe-throughput microbenchmark for the softmax inner loop on sm_100a.
// Measures element-ops per clock per SM for MUFU ex2 (f32, f16x2, bf16x2),
// FFMA, packed FFMA2/FADD2 (f32x2), FMNMX3.  Build + run on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb scripts/microbench_pipes.cu && /tmp/mb
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

constexpr int kIters = 4096;
constexpr int kUnroll = 16;

template <int OP>
__global__ void bench(float* out, long long* cycles, int warps) {
  float a[kUnroll];
  uint32_t h[kUnroll];
  uint64_t w[kUnroll];
  for (int i = 0; i < kUnroll; ++i) {
    a[i] = -float(threadIdx.x + i) * 1e-3f;
    h[i] = 0x3c003c00u ^ (threadIdx.x + i);
    w[i] = 0x3F0000003F000000ull ^ (threadIdx.x + i);
  }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kUnroll; ++i) {
      if constexpr (OP == 0) {
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      } else if constexpr (OP == 1) {
        asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h[i]));
      } else if constexpr (OP == 2) {
        asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h[i]));
      } else if constexpr (OP == 3) {
        asm volatile("fma.rn.f32 %0, %0, 0f3F000001, 0f3E000000;" : "+f"(a[i]));
      } else if constexpr (OP == 4) {
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(w[i]) : "l"(w[(i + 3) % kUnroll]), "l"(w[(i + 5) % kUnroll]));
      } else if constexpr (OP == 5) {
        asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(w[i]) : "l"(w[(i + 3) % kUnroll]));
      } else if constexpr (OP == 6) {
        asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(a[(i + 1) % kUnroll]), "f"(a[(i + 2) % kUnroll]));
      } else if constexpr (OP == 7) {
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(h[i]) : "f"(a[i]), "f"(__uint_as_float(h[i])));
      } else if constexpr (OP == 8) {
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(a[(i + 3) % kUnroll]), "f"(a[(i + 5) % kUnroll]));
      }
    }
  }
  long long t1 = clock64();
  float s = 0.f;
  for (int i = 0; i < kUnroll; ++i) s += a[i] + __uint_as_float(h[i]) + __uint_as_float(uint32_t(w[i]));
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int elems_per_op, int warps) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * sizeof(float));
  cudaMalloc(&cyc, 148 * sizeof(long long));
  bench<OP><<<148, warps * 32>>>(out, cyc, warps);
  cudaDeviceSynchronize();
  bench<OP><<<148, warps * 32>>>(out, cyc, warps);
  cudaDeviceSynchronize();
  long long c[148];
  cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += c[i];
  avg /= 148;
  double ops = double(kIters) * kUnroll * warps * 32 * elems_per_op;
  printf("%-28s warps=%2d  %8.2f elem-ops/clk/SM  (%.2f warp-instr/clk/SM)\n", name, warps,
         ops / avg, ops / elems_per_op / 32 / avg);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {4, 8, 16}) {
    run<0>("ex2.approx.ftz.f32", 1, w);
    run<1>("ex2.approx.f16x2", 2, w);
    run<2>("ex2.approx.ftz.bf16x2", 2, w);
    run<3>("fma.rn.f32 (imm)", 1, w);
    run<8>("fma.rn.f32 (3 reg)", 1, w);
    run<4>("fma.rn.f32x2", 2, w);
    run<5>("add.rn.f32x2", 2, w);
    run<6>("max.f32 (3-input)", 2, w);
    run<7>("cvt.rn.bf16x2.f32", 2, w);
  }
  return 0;
}
