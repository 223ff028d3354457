// Marginal cost of each softmax component (isolated, 1 or 2 warps per SMSP).
// FLAGS bits: 1 = scalar FFMA scale (else FFMA2), 2 = no row sum, 4 = no F2FP pack,
//             8 = no row max, 16 = scalar emulation (else packed)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2603_01960_b200/csrc \
//        -o /tmp/mbs2 scripts/microbench_softmax2.cu && /tmp/mbs2
#include <cstdio>
#include "ptx_sm100.cuh"
using namespace ta;
constexpr int kIters = 256;

__device__ __forceinline__ float ex2_poly_s(float x) { return ex2_poly(x); }

template <int EMU, int FLAGS>
__global__ void bench(const float* in, float sl2, uint32_t* out, long long* cycles) {
  float s[128];
#pragma unroll
  for (int i = 0; i < 128; ++i) s[i] = in[(threadIdx.x * 7 + i) & 1023];
  uint32_t sink = 0;
  float l = 0.f, m = 0.5f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
    if (!(FLAGS & 8)) {
      float mx4[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) mx4[i] = s[i];
#pragma unroll
      for (int i = 4; i < 128; ++i) mx4[i & 3] = fmaxf(mx4[i & 3], s[i]);
      m = fmaxf(m, fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3])) * sl2) - 1e-3f;
    } else {
      m += 1e-7f;
    }
    const uint64_t sl2x2 = f2(sl2, sl2), negm2 = f2(-m, -m);
    uint64_t acc[4] = {0, 0, 0, 0};
    float accs[4] = {0, 0, 0, 0};
#pragma unroll
    for (int g = 0; g < 16; ++g) {
      const int c0 = g * 8;
      float xs[8];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (FLAGS & 1) {
          xs[2 * u] = fmaf(s[c0 + 2 * u], sl2, -m);
          xs[2 * u + 1] = fmaf(s[c0 + 2 * u + 1], sl2, -m);
        } else {
          f2_split(ffma2(f2(s[c0 + 2 * u], s[c0 + 2 * u + 1]), sl2x2, negm2), xs[2 * u], xs[2 * u + 1]);
        }
      }
      float p[8];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (2 * u >= 8 - EMU) {
          if (FLAGS & 16) {
            p[2 * u] = ex2_poly_s(xs[2 * u]);
            p[2 * u + 1] = ex2_poly_s(xs[2 * u + 1]);
          } else {
            ex2_poly2(f2(xs[2 * u], xs[2 * u + 1]), p[2 * u], p[2 * u + 1]);
          }
        } else {
          p[2 * u] = ex2(xs[2 * u]);
          p[2 * u + 1] = ex2(xs[2 * u + 1]);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (!(FLAGS & 2)) acc[u] = fadd2(acc[u], f2(p[2 * u], p[2 * u + 1]));
        if (!(FLAGS & 4)) sink ^= pack2<true>(p[2 * u], p[2 * u + 1]);
        else sink ^= __float_as_uint(p[2 * u]) ^ __float_as_uint(p[2 * u + 1]);
      }
    }
    float lo, hi;
    f2_split(fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3])), lo, hi);
    l += lo + hi + accs[0];
    m += 1e-7f;
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = sink ^ __float_as_uint(l);
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int EMU, int FLAGS>
void run(int warps, const char* name) {
  float* in; uint32_t* out; long long* cyc;
  cudaMalloc(&in, 1024 * 4); cudaMemset(in, 0, 1024 * 4);
  cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  bench<EMU, FLAGS><<<148, warps * 32>>>(in, 0.1275f, out, cyc); cudaDeviceSynchronize();
  bench<EMU, FLAGS><<<148, warps * 32>>>(in, 0.1275f, out, cyc); cudaError_t e = cudaDeviceSynchronize();
  long long c[148]; cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < 148; ++i) avg += c[i]; avg /= 148;
  printf("%-34s emu=%d/8 warps/SM=%2d: %7.1f cyc per 4096-elem warp-tile (%.1f per SMSP-tile)\n", name, EMU, warps,
         avg / kIters, avg / kIters * 4 / warps);
  cudaFree(in); cudaFree(out); cudaFree(cyc);
}

int main() {
  for (int w : {4, 8}) {
    run<2, 0>(w, "baseline (packed)");
    run<2, 1>(w, "scalar FFMA scale");
    run<2, 2>(w, "no row sum");
    run<2, 4>(w, "no F2FP");
    run<2, 8>(w, "no row max");
    run<2, 16>(w, "scalar emulation");
    run<2, 1 | 16>(w, "scalar scale + scalar emu");
    run<0, 1>(w, "scalar scale, no emu");
    run<4, 1 | 16>(w, "scalar scale+emu, emu 4/8");
    run<0, 2 | 4 | 8>(w, "MUFU only (+scale)");
  }
  return 0;
}
