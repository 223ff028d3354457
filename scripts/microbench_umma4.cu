// UMMA sequence throughput (sm_100a): the per-tile MMA mixes of the D=128
// attention loop, one CTA per SM on all SMs, one thread issuing.
//   seq 0: QK^T N=128 (8 x SS M128 N128 K16) + PV (8 x TS M128 N128 K16)   [128-key tile]
//   seq 1: QK^T N=64  (8 x SS M128 N64  K16) + PV (4 x TS M128 N128 K16)   [64-key tile] x2
//   seq 2: QK^T N=128 only (8 x SS)                                         x2
//   seq 3: QK^T N=64 only (8 x SS N64)                                      x4
//   seq 4: PV only (8 x TS N128)                                            x2
//   seq 5: QK^T N=64 as TS (A = Q from TMEM) + PV                           [64-key tile] x2
//   seq 6: QK^T N=256 (8 x SS M128 N256 K16) + PV (16 x TS N128)           [256-key tile] / 2
// Reported: cycles per 128 keys of one 128-row Q tile at D=128 (ideal 1024).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2603_01960_b200/csrc \
//        -o /tmp/mbu4 scripts/microbench_umma4.cu && /tmp/mbu4
#include <cstdio>
#include "ptx_sm100.cuh"
using namespace ta;
constexpr int kReps = 1024;

template <int SEQ>
__global__ void __launch_bounds__(128, 1) bench(long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 3 * 65536);
  uint32_t* holder = reinterpret_cast<uint32_t*>(smem + 3 * 65536 + 128);
  const uint32_t sq = smem_u32(smem), sk = sq + 65536, sv = sk + 65536;
  const uint32_t warp = warp_id(), lane = lane_id();
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(smem_u32(&bar[i]), 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(smem_u32(holder));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *holder;
  if (warp == 0 && lane == 0) {
    const uint32_t id_qk128 = make_idesc_f16(true, 128, 128, false, false);
    const uint32_t id_qk64 = make_idesc_f16(true, 128, 64, false, false);
    const uint32_t id_qk256 = make_idesc_f16(true, 128, 256, false, false);
    const uint32_t id_pv = make_idesc_f16(true, 128, 128, false, true);
    const uint32_t tS = tmem, tO = tmem + 256, tP = tmem + 128, tQ = tmem + 192;
    auto qk = [&](uint32_t idesc, bool ts) {
      for (int ks = 0; ks < 8; ++ks) {
        const uint32_t off = (ks >> 2) * 16384 + (ks & 3) * 32;
        if (ts)
          umma_ts(tS, tQ + ks * 8, sdesc_sw128(sk + off, 16, 1024), idesc, ks > 0);
        else
          umma_ss(tS, sdesc_sw128(sq + off, 16, 1024), sdesc_sw128(sk + off, 16, 1024), idesc, ks > 0);
      }
    };
    auto pv = [&](int n) {
      for (int ks = 0; ks < n; ++ks)
        umma_ts(tO, tP + (ks & 7) * 8, sdesc_sw128(sv + (ks & 7) * 2048, 16384, 1024), id_pv, 1);
    };
    long long t0 = clock64();
    for (int i = 0; i < kReps; ++i) {
      if (SEQ == 0) { qk(id_qk128, false); pv(8); }
      if (SEQ == 1) { qk(id_qk64, false); pv(4); qk(id_qk64, false); pv(4); }
      if (SEQ == 2) { qk(id_qk128, false); qk(id_qk128, false); }
      if (SEQ == 3) { for (int r = 0; r < 4; ++r) qk(id_qk64, false); }
      if (SEQ == 4) { pv(8); pv(8); }
      if (SEQ == 5) { qk(id_qk64, true); pv(4); qk(id_qk64, true); pv(4); }
      if (SEQ == 6) { qk(id_qk256, false); pv(16); }
      if ((i & 15) == 15) {  // bounded queue: drain every 16 reps
        umma_commit(smem_u32(&bar[0]));
        mbar_wait(smem_u32(&bar[0]), (i >> 4) & 1);
      }
    }
    umma_commit(smem_u32(&bar[1]));
    mbar_wait(smem_u32(&bar[1]), 0);
    cycles[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

template <int SEQ>
void run(const char* name, double units_per_rep) {
  long long* cyc;
  cudaMalloc(&cyc, 148 * sizeof(long long));
  const int smem = 3 * 65536 + 2048;
  cudaFuncSetAttribute(bench<SEQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  bench<SEQ><<<148, 128, smem>>>(cyc);
  cudaDeviceSynchronize();
  bench<SEQ><<<148, 128, smem>>>(cyc);
  cudaError_t e = cudaDeviceSynchronize();
  long long c[148];
  cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += c[i];
  avg /= 148;
  printf("%-52s %7.1f cyc per 128-key unit (ideal 1024 for QK+PV) %s\n", name,
         avg / kReps / units_per_rep, e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(cyc);
}

int main() {
  run<0>("seq0 QK N128 SS + PV (128-key tile)", 1.0);
  run<1>("seq1 QK N64 SS + PV (2 x 64-key tiles)", 1.0);
  run<2>("seq2 QK N128 SS only (x2 = 2 units of QK)", 2.0);
  run<3>("seq3 QK N64 SS only (x4 = 2 units of QK)", 2.0);
  run<4>("seq4 PV only (x2 = 2 units of PV)", 2.0);
  run<5>("seq5 QK N64 TS (Q in TMEM) + PV (2 x 64-key)", 1.0);
  run<6>("seq6 QK N256 SS + PV (256-key tile = 2 units)", 2.0);
  return 0;
}
