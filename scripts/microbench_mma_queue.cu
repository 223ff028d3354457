// Does a warp that keeps the tensor-core queue full stall the other warps of
// its SMSP?  Warps 0-3 (one per SMSP) run a throughput-bound FFMA2 -> MUFU ->
// F2FP stream (128 independent exps per repetition, as the softmax does);
// warp 7 (SMSP 3) concurrently issues MODE:
//   0: nothing
//   1: groups of 4 MMAs + commit, wait for the group (queue nearly empty)
//   2: groups of G MMAs + commit, wait for the group before the previous one
//      (up to 2G MMAs queued), G = 16
//   3: same with G = 32 (the attention step issues 32 MMAs per K/V tile)
// Reported: cycles of warps 0..3 for the same work; warp 3 / warp 0 > 1 means
// the MMA issue stalls the SMSP it runs on.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2603_01960_b200/csrc \
//        -o /tmp/mbq scripts/microbench_mma_queue.cu && /tmp/mbq
#include <cstdio>
#include "ptx_sm100.cuh"
using namespace ta;
constexpr int kReps = 48;

__device__ __forceinline__ float vex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int MODE>
__global__ void __launch_bounds__(256, 1) bench(const float* in, long long* out, uint32_t* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 65536);
  uint32_t* holder = reinterpret_cast<uint32_t*>(smem + 65536 + 64);
  volatile int* stop = reinterpret_cast<volatile int*>(smem + 65536 + 128);
  const uint32_t warp = warp_id(), lane = lane_id();
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar[0]), 1);
    mbar_init(smem_u32(&bar[1]), 1);
    *stop = 0;
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(smem_u32(holder));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *holder;
  if (warp < 4) {
    float s[128];
    for (int i = 0; i < 128; ++i) s[i] = in[(threadIdx.x * 131 + i) & 1023];
    const uint64_t sl2x2 = f2(in[1], in[1]);
    uint32_t acc = 0;
    long long t0 = clock64();
    for (int rep = 0; rep < kReps; ++rep) {
      const float mr = in[2] + float(rep) * 1e-6f;
      const uint64_t negm2 = f2(-mr, -mr);
#pragma unroll
      for (int u = 0; u < 64; ++u) {
        float a, b;
        f2_split(ffma2(f2(s[2 * u], s[2 * u + 1]), sl2x2, negm2), a, b);
        acc ^= pack2<true>(vex2(a), vex2(b));
      }
    }
    long long t1 = clock64();
    sink[blockIdx.x * 256 + threadIdx.x] = acc;
    if (lane == 0) {
      out[blockIdx.x * 4 + warp] = t1 - t0;
      atomicAdd((int*)stop, 1);
    }
  } else if (warp == 7) {
    const uint32_t idesc = make_idesc_f16(true, 128, 128, false, false);
    const uint64_t d = sdesc_sw128(smem_u32(smem), 16, 1024);
    constexpr int G = MODE == 1 ? 4 : MODE == 2 ? 16 : 32;
    uint32_t ph[2] = {0, 0};
    int g = 0;
    while (*stop < 4) {
      if (MODE == 0) {
        __nanosleep(200);
        continue;
      }
      for (int k = 0; k < G; ++k) umma_ss_warp(tmem + 256, d, d, idesc, 1);
      umma_commit_warp(smem_u32(&bar[g & 1]));
      if (MODE == 1) {
        mbar_wait(smem_u32(&bar[g & 1]), ph[g & 1]);
        ph[g & 1] ^= 1;
      } else if (g > 0) {  // wait for the previous group: <= 2G MMAs in flight
        mbar_wait(smem_u32(&bar[(g - 1) & 1]), ph[(g - 1) & 1]);
        ph[(g - 1) & 1] ^= 1;
      }
      ++g;
    }
    if (MODE >= 2 && g > 0) {  // drain
      mbar_wait(smem_u32(&bar[(g - 1) & 1]), ph[(g - 1) & 1]);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int MODE>
void run(const char* name, const float* in) {
  long long* out;
  uint32_t* sink;
  cudaMalloc(&out, 148 * 4 * 8);
  cudaMalloc(&sink, 148 * 256 * 4);
  const int smem = 65536 + 2048;
  cudaFuncSetAttribute(bench<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  bench<MODE><<<148, 256, smem>>>(in, out, sink);
  bench<MODE><<<148, 256, smem>>>(in, out, sink);
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaGetLastError();
  long long h[148 * 4];
  cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
  double w[4] = {0, 0, 0, 0};
  for (int b = 0; b < 148; ++b)
    for (int i = 0; i < 4; ++i) w[i] += h[b * 4 + i] / 148.0;
  printf("%-34s cyc/MUFU warp0..3: %6.2f %6.2f %6.2f %6.2f (warp3/warp0 %.3f) %s\n", name,
         w[0] / (kReps * 128.0), w[1] / (kReps * 128.0), w[2] / (kReps * 128.0),
         w[3] / (kReps * 128.0), w[3] / w[0], e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(out);
  cudaFree(sink);
}

int main() {
  float* in;
  cudaMalloc(&in, 1024 * 4);
  float h[1024];
  for (int i = 0; i < 1024; ++i) h[i] = -float(i % 17) * 0.25f;
  h[1] = 0.1275f;
  h[2] = 0.5f;
  cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  run<0>("idle", in);
  run<1>("MMA groups of 4, wait each", in);
  run<2>("MMA groups of 16, 2 in flight", in);
  run<3>("MMA groups of 32, 2 in flight", in);
  return 0;
}
