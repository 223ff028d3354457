// Softmax exp phase with the P hand-off: exps of one 128-key row tile per
// thread (4096 scores per warp), P packed to 16 bit and written to TMEM with
// tcgen05.st, then tcgen05.wait::st before the (simulated) mbarrier arrive.
// MODE 0: no stores; 1: st + wait::st per half (current kernel); 2: per
// quarter; 3: st per quarter, wait::st deferred by one quarter; 4: st, one
// wait at the end.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2603_01960_b200/csrc \
//        -o build/mb_sm3 scripts/microbench_softmax3.cu && build/mb_sm3
#include <cstdio>
#include "ptx_sm100.cuh"
using namespace ta;
constexpr int kIters = 128;

template <int MODE>
__global__ void __launch_bounds__(256, 1) bench(const float* in, float sl2, uint32_t* out,
                                                long long* cycles) {
  __shared__ uint32_t holder;
  __shared__ uint64_t bar;
  const uint32_t warp = warp_id();
  if (warp == 0) tmem_alloc<512>(smem_u32(&holder));
  if (threadIdx.x == 0) mbar_init(smem_u32(&bar), 1u << 16);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = holder + (((warp & 3) * 32u) << 16) + (warp >> 2) * 128;
  float s[128];
#pragma unroll
  for (int i = 0; i < 128; ++i) s[i] = in[(threadIdx.x * 7 + i) & 1023];
  uint32_t sink = 0;
  float l = 0.f, m = 0.5f;
  long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
    const uint64_t sl2x2 = f2(sl2, sl2), negm2 = f2(-m, -m);
    uint64_t acc[2] = {0, 0};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t pk[16];
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const int c0 = q * 32 + g * 8;
        uint64_t x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) x[u] = ffma2(f2(s[c0 + 2 * u], s[c0 + 2 * u + 1]), sl2x2, negm2);
        float p[8];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (u == 3) {
            ex2_poly2(x[u], p[2 * u], p[2 * u + 1]);
          } else {
            float a, b;
            f2_split(x[u], a, b);
            p[2 * u] = ex2(a);
            p[2 * u + 1] = ex2(b);
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          acc[u & 1] = fadd2(acc[u & 1], f2(p[2 * u], p[2 * u + 1]));
          pk[g * 4 + u] = pack2<true>(p[2 * u], p[2 * u + 1]);
        }
      }
      if (MODE == 0) {
#pragma unroll
        for (int i = 0; i < 16; ++i) sink ^= pk[i];
      } else {
        if (MODE == 3 && q > 0) {
          tmem_wait_st();
          tc_fence_before();
          __syncwarp();
          if ((threadIdx.x & 31) == 0) mbar_arrive(smem_u32(&bar));
        }
        tmem_st16(tm + q * 16, pk);
        if (MODE == 2 || (MODE == 1 && (q & 1))) {
          tmem_wait_st();
          tc_fence_before();
          __syncwarp();
          if ((threadIdx.x & 31) == 0) mbar_arrive(smem_u32(&bar));
        }
      }
    }
    if (MODE == 3 || MODE == 4) {
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(smem_u32(&bar));
    }
    float lo, hi;
    f2_split(fadd2(acc[0], acc[1]), lo, hi);
    l += lo + hi;
    m += 1e-7f;
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = sink ^ __float_as_uint(l);
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(holder);
}

template <int MODE>
void run(int warps) {
  float* in; uint32_t* out; long long* cyc;
  cudaMalloc(&in, 1024 * 4); cudaMemset(in, 0, 1024 * 4);
  cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  bench<MODE><<<148, warps * 32>>>(in, 0.1275f, out, cyc); cudaDeviceSynchronize();
  bench<MODE><<<148, warps * 32>>>(in, 0.1275f, out, cyc); cudaError_t e = cudaDeviceSynchronize();
  long long c[148]; cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < 148; ++i) avg += c[i]; avg /= 148;
  printf("mode %d warps/SM=%2d: %7.1f cyc per warp-tile (%.1f per SMSP-tile) %s\n", MODE, warps,
         avg / kIters, avg / kIters * 4 / warps, e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(in); cudaFree(out); cudaFree(cyc);
}

int main() {
  for (int w : {4, 8}) {
    run<0>(w); run<1>(w); run<2>(w); run<3>(w); run<4>(w);
  }
  return 0;
}
