// UMMA issue-side bubbles: groups of G MMAs, each followed by a commit and W
// mbarrier waits on an already-completed barrier (what the attention MMA warp
// does between groups).  cycles per MMA vs the 64-cycle floor.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2603_01960_b200/csrc \
//        -o /tmp/mbu3 scripts/microbench_umma3.cu && /tmp/mbu3
#include <cstdio>
#include "ptx_sm100.cuh"
using namespace ta;
constexpr int kGroups = 512;

template <int G, int W, int C, int KIND = 0>
__global__ void __launch_bounds__(128, 1) bench(long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 65536);
  uint32_t* holder = reinterpret_cast<uint32_t*>(smem + 65536 + 128);
  const uint32_t sa = smem_u32(smem), sb = sa + 32768;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(smem_u32(&bar[i]), 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc<512>(smem_u32(holder));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *holder;
  if (threadIdx.x == 0) {
    mbar_arrive(smem_u32(&bar[1]));  // phase 0 of bar[1] completes: "already ready" barrier
    const uint32_t idesc = make_idesc_f16(true, 128, 128, false, false);
    long long t0 = clock64();
    for (int g = 0; g < kGroups; ++g) {
      for (int w = 0; w < W; ++w) {
        if (KIND == 0) { mbar_wait(smem_u32(&bar[1]), 0); tc_fence_after(); }
        if (KIND == 1) { mbar_wait(smem_u32(&bar[1]), 0); }
        if (KIND == 2) { tc_fence_after(); }
        if (KIND == 3) {  // single try_wait probe, no loop
          uint32_t ok;
          asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.u32 %0, 1, 0, P;\n\t}"
                       : "=r"(ok) : "r"(smem_u32(&bar[1])), "r"(0u) : "memory");
          if (!ok) mbar_wait(smem_u32(&bar[1]), 0);
        }
        if (KIND == 4) {  // test_wait probe
          uint32_t ok;
          asm volatile("{\n\t.reg .pred P;\n\tmbarrier.test_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.u32 %0, 1, 0, P;\n\t}"
                       : "=r"(ok) : "r"(smem_u32(&bar[1])), "r"(0u) : "memory");
          if (!ok) mbar_wait(smem_u32(&bar[1]), 0);
        }
      }
#pragma unroll
      for (int i = 0; i < G; ++i) {
        const uint32_t ks = i & 7;
        const uint32_t off = (ks >> 2) * 16384 + (ks & 3) * 32;
        umma_ss(tmem + (g & 1) * 128, sdesc_sw128(sa + off, 16, 1024), sdesc_sw128(sb + off, 16, 1024), idesc, i > 0);
      }
      for (int c = 0; c < C; ++c) umma_commit(smem_u32(&bar[2 + (c & 1)]));
    }
    umma_commit(smem_u32(&bar[0]));
    mbar_wait(smem_u32(&bar[0]), 0);
    long long t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}

template <int G, int W, int C, int KIND = 0>
void run() {
  long long* cyc;
  cudaMalloc(&cyc, 148 * sizeof(long long));
  const int smem = 65536 + 2048;
  cudaFuncSetAttribute(bench<G, W, C, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  bench<G, W, C, KIND><<<148, 128, smem>>>(cyc);
  cudaDeviceSynchronize();
  bench<G, W, C, KIND><<<148, 128, smem>>>(cyc);
  cudaError_t e = cudaDeviceSynchronize();
  long long c[148];
  cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += c[i];
  avg /= 148;
  printf("kind=%d group=%d waits/group=%d commits/group=%d : %7.2f cyc/MMA %s\n", KIND, G, W, C, avg / (kGroups * G),
         e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(cyc);
}

int main() {
  run<8, 0, 0>();
  run<8, 0, 1>();
  run<8, 0, 2>();
  run<8, 1, 1>();
  run<8, 2, 2>();
  run<4, 1, 1>();
  run<4, 2, 1>();
  run<16, 2, 2>();
  run<8, 2, 1, 1>();
  run<8, 2, 1, 2>();
  run<8, 2, 1, 3>();
  run<8, 2, 1, 4>();
  run<4, 2, 1, 1>();
  run<4, 2, 1, 2>();
  return 0;
}
