// UMMA (tcgen05.mma kind::f16) issue-rate microbenchmark on sm_100a.
// One CTA per SM, one thread issues kN MMAs back to back; cycles per MMA are
// reported for SS (A,B from smem) / TS (A from TMEM) at several N.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2603_01960_b200/csrc \
//        -o /tmp/mbu scripts/microbench_umma.cu && /tmp/mbu
#include <cstdio>
#include "ptx_sm100.cuh"

using namespace ta;

constexpr int kN = 2048;

template <int MODE, int N>
__global__ void __launch_bounds__(128, 1) bench(long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 131072);
  uint32_t* holder = reinterpret_cast<uint32_t*>(smem + 131072 + 64);
  const uint32_t sa = smem_u32(smem), sb = sa + 65536;
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(bar), 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc<512>(smem_u32(holder));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *holder;
  if (threadIdx.x == 0) {
    const uint32_t idesc = make_idesc_f16(true, 128, N, false, MODE == 2);
    long long t0 = clock64();
    for (int i = 0; i < kN; ++i) {
      const uint32_t ks = i & 7;
      const uint32_t off = (ks >> 2) * 16384 + (ks & 3) * 32;
      if (MODE == 0) {
        umma_ss(tmem, sdesc_sw128(sa + off, 16, 1024), sdesc_sw128(sb + off, 16, 1024), idesc, 1);
      } else if (MODE == 1) {
        umma_ts(tmem, tmem + 256 + ks * 8, sdesc_sw128(sb + off, 16, 1024), idesc, 1);
      } else {
        umma_ts(tmem, tmem + 256 + ks * 8, sdesc_sw128(sb + ks * 2048, 16384, 1024), idesc, 1);
      }
    }
    umma_commit(smem_u32(bar));
    mbar_wait(smem_u32(bar), 0);
    long long t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}

template <int MODE, int N>
void run(const char* name) {
  long long* cyc;
  cudaMalloc(&cyc, 148 * sizeof(long long));
  const int smem = 131072 + 2048;
  cudaFuncSetAttribute(bench<MODE, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  bench<MODE, N><<<148, 128, smem>>>(cyc);
  cudaDeviceSynchronize();
  bench<MODE, N><<<148, 128, smem>>>(cyc);
  cudaError_t e = cudaDeviceSynchronize();
  long long c[148];
  cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += c[i];
  avg /= 148;
  const double flop_per = 2.0 * 128 * N * 16;
  printf("%-34s N=%3d  %7.2f cyc/MMA  %7.1f flop/clk/SM (ideal 8192) %s\n", name, N, avg / kN,
         flop_per * kN / avg, e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(cyc);
}

int main() {
  run<0, 64>("SS  K-major A,B");
  run<0, 128>("SS  K-major A,B");
  run<0, 256>("SS  K-major A,B");
  run<1, 64>("TS  A tmem, B K-major");
  run<1, 128>("TS  A tmem, B K-major");
  run<1, 256>("TS  A tmem, B K-major");
  run<2, 128>("TS  A tmem, B MN-major");
  return 0;
}
