// Does a warp issuing tcgen05.mma slow the other warps of its SMSP?
// Warps 0-3 (one per SMSP) run an FFMA2 / MUFU mix for a fixed number of
// iterations; warp 7 (SMSP 3) concurrently issues MODE: 0 nothing, 1 MMAs
// (128x128x16, groups of 4 + commit), 2 mbarrier polling, 3 ALU spin.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2603_01960_b200/csrc \
//        -o build/mb_mmaint scripts/microbench_mma_interference.cu && build/mb_mmaint
#include <cstdio>
#include "ptx_sm100.cuh"
using namespace ta;

template <int MODE>
__global__ void __launch_bounds__(256, 1) bench(long long* out, float* sink, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 65536);
  uint32_t* holder = reinterpret_cast<uint32_t*>(smem + 65536 + 64);
  volatile int* stop = reinterpret_cast<volatile int*>(smem + 65536 + 128);
  const uint32_t warp = warp_id(), lane = lane_id();
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar[0]), 1); *stop = 0; fence_barrier_init(); }
  if (warp == 0) tmem_alloc<512>(smem_u32(holder));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *holder;
  if (warp < 4) {
    float a[16];
    for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 16; i += 2) {
        uint64_t x = ffma2(f2(a[i], a[i + 1]), f2(0.999f, 0.999f), f2(1e-3f, 1e-3f));
        float p, q;
        f2_split(x, p, q);
        a[i] = ex2(p * -1e-3f) + p;
        a[i + 1] = q;
      }
    }
    long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 16; ++i) s += a[i];
    sink[blockIdx.x * 128 + threadIdx.x] = s;
    if (lane == 0) { out[blockIdx.x * 4 + warp] = t1 - t0; atomicAdd((int*)stop, 1); }
  } else if (warp == 7) {
    const uint32_t idesc = make_idesc_f16(true, 128, 128, false, false);
    const uint64_t d = sdesc_sw128(smem_u32(smem), 16, 1024);
    int n = 0;
    uint32_t ph = 0;
    while (*stop < 4) {
      if (MODE == 1) {
        for (int k = 0; k < 4; ++k) umma_ss_warp(tmem + 256, d, d, idesc, 1);
        umma_commit_warp(smem_u32(&bar[0]));
        mbar_wait(smem_u32(&bar[0]), ph);
        ph ^= 1;
      } else if (MODE == 2) {
        uint32_t ok;
        asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.u32 %0, 1, 0, P;\n\t}"
                     : "=r"(ok) : "r"(smem_u32(&bar[0])), "r"(0u) : "memory");
        n += ok;
      } else if (MODE == 3) {
        for (int k = 0; k < 64; ++k) n = n * 3 + k;
      }
      ++n;
    }
    if (lane == 0) sink[148 * 128 + blockIdx.x] = n;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int MODE>
void run(const char* name) {
  long long* out; float* sink;
  cudaMalloc(&out, 148 * 4 * 8); cudaMalloc(&sink, 149 * 128 * 4 + 4096);
  const int smem = 65536 + 2048;
  cudaFuncSetAttribute(bench<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  bench<MODE><<<148, 256, smem>>>(out, sink, 2000);
  bench<MODE><<<148, 256, smem>>>(out, sink, 2000);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148 * 4];
  cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
  double w[4] = {0, 0, 0, 0};
  for (int b = 0; b < 148; ++b) for (int i = 0; i < 4; ++i) w[i] += h[b * 4 + i] / 148.0;
  printf("%-22s warp0..3 cycles: %8.0f %8.0f %8.0f %8.0f  (warp3/warp0 %.3f) %s\n", name, w[0], w[1], w[2], w[3],
         w[3] / w[0], e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  run<0>("idle");
  run<1>("MMA issue (4+commit)");
  run<2>("mbarrier poll");
  run<3>("ALU spin");
  return 0;
}
