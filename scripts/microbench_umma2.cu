// UMMA throughput under contention (sm_100a), one CTA per SM, 256 threads:
//   warp 0 lane 0 issues kN MMAs (M=128, N=128, K=16, bf16) back to back;
//   warps 4..7 optionally stream tcgen05.ld / tcgen05.st on other TMEM columns;
//   warp 1 lane 0 optionally streams bulk global->smem copies (TMA engine).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2603_01960_b200/csrc \
//        -o /tmp/mbu2 scripts/microbench_umma2.cu && /tmp/mbu2
#include <cstdio>
#include "ptx_sm100.cuh"
using namespace ta;
constexpr int kN = 4096;

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}

// MMA: 0 = SS, 1 = TS ; LDST: 0 none, 1 tcgen05.ld, 2 tcgen05.st, 3 ld+st ; TMA: 0/1
template <int MMA, int LDST, int TMA>
__global__ void __launch_bounds__(256, 1) bench(const uint8_t* gsrc, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 196608);
  uint32_t* holder = reinterpret_cast<uint32_t*>(smem + 196608 + 64);
  volatile int* done = reinterpret_cast<volatile int*>(smem + 196608 + 128);
  const uint32_t sa = smem_u32(smem), sb = sa + 32768, stma = sa + 65536;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar[0]), 1);
    mbar_init(smem_u32(&bar[1]), 1);
    *done = 0;
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(smem_u32(holder));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *holder;
  if (warp == 0) {
    if (lane == 0) {
      const uint32_t idesc = make_idesc_f16(true, 128, 128, false, false);
      long long t0 = clock64();
      for (int i = 0; i < kN; ++i) {
        const uint32_t ks = i & 7;
        const uint32_t off = (ks >> 2) * 16384 + (ks & 3) * 32;
        if (MMA == 0)
          umma_ss(tmem, sdesc_sw128(sa + off, 16, 1024), sdesc_sw128(sb + off, 16, 1024), idesc, 1);
        else
          umma_ts(tmem, tmem + 384 + ks * 8, sdesc_sw128(sb + off, 16, 1024), idesc, 1);
      }
      umma_commit(smem_u32(&bar[0]));
      mbar_wait(smem_u32(&bar[0]), 0);
      long long t1 = clock64();
      cycles[blockIdx.x] = t1 - t0;
      *done = 1;
    }
  } else if (warp == 1) {
    if (TMA && lane == 0) {
      uint32_t phase = 0;
      while (!*done) {
        mbar_arrive_expect_tx(smem_u32(&bar[1]), 65536);
        for (int c = 0; c < 4; ++c)
          bulk_g2s(stma + c * 16384, gsrc + (size_t(blockIdx.x) * 4 + c) * 16384, 16384, smem_u32(&bar[1]));
        mbar_wait(smem_u32(&bar[1]), phase);
        phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    const uint32_t base = tmem + (((warp & 3) * 32u) << 16) + 128;
    uint32_t r[32];
    for (int i = 0; i < 32; ++i) r[i] = i;
    while (!*done) {
      for (int c = 0; c < 8; ++c) {
        if (LDST & 1) { tmem_ld32(base + (c & 3) * 32, r); tmem_wait_ld(); reg_fence(r); }
        if (LDST & 2) { tmem_st32(base + 128 + (c & 1) * 32, r); tmem_wait_st(); }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

template <int MMA, int LDST, int TMA>
void run(const char* name, const uint8_t* gsrc) {
  long long* cyc;
  cudaMalloc(&cyc, 148 * sizeof(long long));
  const int smem = 196608 + 2048;
  cudaFuncSetAttribute(bench<MMA, LDST, TMA>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  bench<MMA, LDST, TMA><<<148, 256, smem>>>(gsrc, cyc);
  cudaDeviceSynchronize();
  bench<MMA, LDST, TMA><<<148, 256, smem>>>(gsrc, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  long long c[148];
  cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += c[i];
  avg /= 148;
  printf("%-44s %7.2f cyc/MMA %s\n", name, avg / kN, e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(cyc);
}

int main() {
  uint8_t* g;
  cudaMalloc(&g, 148 * 4 * 16384);
  run<0, 0, 0>("SS alone", g);
  run<0, 1, 0>("SS + tcgen05.ld stream (4 warps)", g);
  run<0, 2, 0>("SS + tcgen05.st stream", g);
  run<0, 3, 0>("SS + ld+st stream", g);
  run<0, 0, 1>("SS + TMA bulk g2s stream", g);
  run<0, 3, 1>("SS + ld+st + TMA", g);
  run<1, 0, 0>("TS alone", g);
  run<1, 1, 0>("TS + tcgen05.ld stream", g);
  run<1, 2, 0>("TS + tcgen05.st stream", g);
  run<1, 3, 0>("TS + ld+st", g);
  run<1, 0, 1>("TS + TMA", g);
  run<1, 3, 1>("TS + ld+st + TMA", g);
  return 0;
}
