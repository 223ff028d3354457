// Internal interface between the C-ABI host layer (c_api.cpp) and the
// sm_100a kernels (sdpa_fwd_sm100.cu).  Not part of the public ABI.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace ta {

// MaskKind (reference types.hpp:41-76)
enum FwdMask { kMaskNone = 0, kMaskCausal = 1, kMaskPadding = 2 };
// key-side padding lengths travel in the kernel parameters (no device copy)
// padding lengths of up to kInlinePadding batches travel in the kernel
// parameters; more come through a device array (a 4 KB parameter block
// measured +3.5 us per launch)
constexpr int kInlinePadding = 32;

struct FwdArgs {
  void* o;           // [BH, S, D] 16-bit, same dtype as inputs
  float* lse;        // [BH, S] fp32 natural-log LSE, or nullptr
  int seq_len;       // S
  int head_dim;      // D of the tensors in memory (<= the kernel's D; the
                     // kernel's extra columns are TMA zero-fill)
  float scale_log2;  // softmax scale * log2(e)
  int mask;          // FwdMask
  int heads;         // H: batch index of flattened head bh is (bh_offset + bh) / H
  int bh_offset;     // first flattened head of this launch (chunked host path)
  int bh_count;      // flattened heads of this launch (persistent kernels' item count)
  // diagnostics: when non-null, CTA (0,0) records clock64 timestamps
  // trace[event * kTraceIters + j] for the first kTraceIters K/V iterations
  long long* trace;
  int valid_len[kInlinePadding];  // Padding: keys j < valid_len[b] admitted (B <= 32)
  const int* valid_len_dev;       // ... or this device array [B] (nullptr: inline)
};

constexpr int kTraceIters = 64;
// trace events
enum TraceEvent {
  kEvMmaWaitP0 = 0,  // MMA warp: P0(j-1) ready observed
  kEvMmaIssuedPV0,   // PV0(j-1) + S0(j) issued
  kEvMmaWaitP1,      // P1(j-1) ready observed
  kEvMmaIssuedPV1,   // PV1(j-1) + S1(j) issued
  kEvSm0SReady,      // softmax WG0: S0(j) observed ready
  kEvSm0Loaded,      // S0 in registers
  kEvSm0Max,         // row max done
  kEvSm0Exp,         // exps + pack done
  kEvSm0PArrive,     // P0(j) written + arrived
  kEvSm1SReady,
  kEvSm1Loaded,
  kEvSm1Max,
  kEvSm1Exp,
  kEvSm1PArrive,
  kEvTcPV0Done,  // tracer warp: o_full[0] phase j completed (PV0(j) done)
  kEvTcS0Done,   // s_full[0] phase j+1 completed (S0(j+1) done)
  kEvTcPV1Done,
  kEvTcS1Done,
  kEvSm0ArriveW1,  // Q tile 0, warps 1..3: last P part arrived (warp skew)
  kEvSm0ArriveW2,
  kEvSm0ArriveW3,
  kEvKernelStart,  // [0]: CTA entry; [1]: after the TMEM alloc / barrier-init sync
  kEvEpilogueDone,  // [t]: Q tile t's row-0 warp has stored O and LSE
  kNumTraceEvents
};

struct FwdLaunch {
  const CUtensorMap* tmap_q;
  const CUtensorMap* tmap_k;
  const CUtensorMap* tmap_v;
  const CUtensorMap* tmap_o;  // O, boxes of 64 cols x 128 rows (epilogue TMA store)
  FwdArgs args;
  int64_t bh;
  int head_dim;  // kernel instantiation: 64, 128, 192 or 256
  int block_n;   // keys per K/V tile: 128, or 64 (head_dim 128 only)
  bool pair;     // CTA-pair (cta_group::2) kernel: K map boxes of block_n / 2 rows
  bool bf16;
  void* stream;
};

struct FwdGeometry {
  int block_m;
  int block_n;
  int q_tiles_per_cta;
  int threads;
  int64_t ctas;
};

// keys per K/V tile executed for a head dim and the schedule's t_n
int fwd_block_n(int64_t D, int t_n);
// whether a launch runs the CTA-pair kernel (mask: kMaskNone / Causal / Padding)
bool fwd_use_pair(int64_t D, int block_n, int mask);
FwdGeometry fwd_geometry(int64_t S, int64_t BH, int64_t D, int block_n = 128);
int fwd_ring_slots(int D, int block_n = 128);
// kernel instantiation for a head dim: 64, 128, 192 or 256 (memory D <= it;
// the TMA boxes zero-fill the extra columns)
int fwd_kernel_head_dim(int64_t D);
cudaError_t launch_sdpa_fwd(const FwdLaunch& launch);
cudaError_t launch_exp2_unit(const float* x, float* y, int64_t n, int mode, void* stream);
cudaError_t launch_umma_selftest(const CUtensorMap* a_map, const CUtensorMap* b_map,
                                 const void* a_glob, float* d_out, int mode, bool bf16,
                                 void* stream);

}  // namespace ta
