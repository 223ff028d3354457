// SDPA forward for B200 (sm_100a): TMA -> 128B-swizzled smem ring -> tcgen05.mma
// (QK^T and PV, fp32 accumulators in TMEM) with warp-specialised roles and an
// online softmax in registers (one thread == one query row).
//
// Replaces the reference CPU hot path tileattn::sdpa_tiled / run_tiled
// (reference proj/src/tiled.cpp:119-272, proj/include/tileattn/tiled.hpp:
// 147-238).  Algorithm per (bh, query block) is the reference's item_body
// (tiled.cpp:144-221): load Q tile once, stream K/V tiles, score_tile ->
// mask -> online_update, finalize O = o / l.  Differences are B200-native:
//   * two 128-row Q tiles per CTA ping-pong on the tensor core (the MMA of
//     one tile overlaps the softmax of the other);
//   * scores never leave TMEM except into the softmax registers; P (16-bit)
//     is written back into the S columns of TMEM and consumed by a TS-MMA;
//   * exp2 with the softmax scale folded into one FFMA; the running max is
//     updated lazily (only when it grows by > 2^8), so the O correction in
//     TMEM is rare (tiled.hpp:212 skips the rescale only when alpha == 1);
//   * LSE = m + ln(l) is emitted as a second output (the reference computes
//     m and l but never returns them, tiled.hpp:223-238).
// Instantiations (launch_sdpa_fwd): D=128 two-tile ping-pong with 128-key
// tiles (the product path) or 64-key tiles (TileSchedule t_n <= 64, split
// softmax: two warps per row); D=64 and D > 128 one Q tile per CTA with the
// S/P rotation.  Build options kept for A/B:
// TA_D128_SPLIT (split softmax at 128 keys), TA_PAIR (cta_group::2 pair),
// TA_D64_PERSIST (persistent D=64, sdpa_d64_sm100.cuh), TA_OBSERVE_PHASES
// (synccheck build); TA_DEBUG_* are ablations with wrong results.
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <type_traits>

#include "ptx_sm100.cuh"
#include "sdpa_fwd_sm100.h"

// Roles<kQT> constants are used through local aliases; the front end reports
// the static members as unreferenced (#177) for some instantiations.
#pragma nv_diag_suppress 177

namespace ta {
namespace {

constexpr int kBM = 128;        // rows per Q tile (UMMA M)
constexpr int kBN128 = 128;     // default keys per K/V tile (UMMA N of QK^T, K of PV);
                                // the kernels take kBN (128, or 64 for t_n <= 64 at D=128)
constexpr int kQTiles = 2;      // max Q tiles per CTA (ping-pong)

// Warp roles and register split of a CTA with kQT Q tiles (kQT = 2: the
// D=128 ping-pong, one CTA per SM; kQT = 1: D=64, two CTAs per SM, each
// with one Q tile, so one CTA's prologue / epilogue overlaps the other's
// loop).  Softmax warps 4t..4t+3 own Q tile t (warp w <-> TMEM lane quadrant
// w % 4); the control warps take the top ids (the SM's warp arbiter favours
// high ids, so the single-thread roles are never starved).
// kWide (D > 128): one Q tile, one CTA per SM (the O accumulator needs up
// to 256 TMEM columns), no register rebalancing (255 registers per thread).
template <int kQT, bool kWide = false, bool kSplit = false>
struct Roles {
  // kSplit: two softmax warps per TMEM lane quadrant and Q tile, each owning
  // 64 of the tile's 128 key columns
  static constexpr int kSoftmaxWarps = 4 * kQT * (kSplit ? 2 : 1);
  static constexpr int kThreads = 32 * (kSoftmaxWarps + 4);
  static constexpr int kMinBlocks = kQT == 1 && !kWide ? 2 : 1;
  static constexpr bool kSetMaxNReg = !kWide;
  static constexpr int kWarpAlloc = kSoftmaxWarps + 0;  // TMEM allocator (otherwise idle)
  static constexpr int kWarpTma = kSoftmaxWarps + 1;
  static constexpr int kWarpTrace = kSoftmaxWarps + 2;  // diagnostics only
  static constexpr int kWarpMma = kSoftmaxWarps + 3;
  static constexpr uint32_t kTmemCols = kQT == 1 && !kWide ? 256 : 512;
  // setmaxnreg.inc only draws on registers released by setmaxnreg.dec in
  // the same CTA, so the split must balance around the launch allocation
  // (kQT=2: 65536/384 -> 168, 256*(208-168) == 128*(168-88); kQT=1, two
  // CTAs: 32768/256 -> 128, 128*(200-128) == 128*(128-56)).
  static constexpr int kLaunchRegs = kWide ? 248 : (65536 / (kThreads * kMinBlocks)) & ~7;
  // (kSplit: 640 threads -> 96; 512 * (104 - 96) <= 128 * (96 - 56))
#ifndef TA_QT1_REGS_SOFTMAX  // register split at QT=1 (two CTAs per SM), A/B knob
#define TA_QT1_REGS_SOFTMAX 200
#endif
  static constexpr int kRegsSoftmax = kWide ? 248 : kSplit ? 104 : kQT == 1 ? TA_QT1_REGS_SOFTMAX : 208;
  static constexpr int kRegsControl =
      kWide ? 248 : kSplit ? 56 : kQT == 1 ? 256 - TA_QT1_REGS_SOFTMAX : 88;
  static_assert(kSoftmaxWarps * 32 * (kRegsSoftmax - kLaunchRegs) <=
                    (kThreads - kSoftmaxWarps * 32) * (kLaunchRegs - kRegsControl),
                "setmaxnreg.inc would wait forever: register pool does not balance");
};
// Q tiles per CTA by head dim (TA_D64_TILES: 1 or 2 for A/B builds)
#ifndef TA_D64_TILES
#define TA_D64_TILES 1
#endif
#ifndef TA_D128_TILES
#define TA_D128_TILES 2
#endif
template <int D>
constexpr int kQTilesFor = D == 64 ? TA_D64_TILES : D == 128 ? TA_D128_TILES : 1;
// D=128 softmax split over two warps per lane quadrant and tile (TA_D128_SPLIT)
// (the 64-key kernel always splits: 32 keys per warp)
#ifndef TA_D128_SPLIT
#define TA_D128_SPLIT 0
#endif
template <int D, int kQT, int kBN = 128>
constexpr bool kSplitFor = (D == 128 || D == 64) && kQT == 2 && (TA_D128_SPLIT || kBN == 64);
template <int D, int kQT, int kBN = 128>
using RolesFor = Roles<kQT, (D > 128), kSplitFor<D, kQT, kBN>>;
constexpr float kLn2 = 0.69314718055994530942f;
// lazy rescale threshold in log2 units: exps may reach 2^8 before O is
// rescaled (fp32 accumulators, 16-bit P: both fine).
constexpr float kRescaleThreshold = 8.0f;
// exp2 work split: of every 16 score columns, kEmu16 (even: emulated in
// packed pairs) use the FMA-pipe polynomial (ex2_poly2) and the rest the MUFU
// (measured 16 exp2/clk/SM).  D=128 is tensor-bound with the softmax on the
// chain: MUFU only.  D=64 is softmax-throughput bound: 4 of 16 on the FMA
// pipe (same-box A/B in profiles/r01/microbench.md).
#ifndef TA_EMU16_D128
#define TA_EMU16_D128 0
#endif
// split softmax (D=128): a quarter of the exps on the FMA pipe keeps the
// four softmax warps per SMSP below the MUFU pipe's 8 cycles per warp-exp
#ifndef TA_EMU16_SPLIT
#define TA_EMU16_SPLIT 4
#endif
#ifndef TA_EMU16_D64
#define TA_EMU16_D64 4
#endif
// P hand-off granularity to the PV MMAs (2 = halves, 4 = quarters of 32 keys)
#ifndef TA_P_PARTS
#define TA_P_PARTS 2
#endif
constexpr int kPParts = TA_P_PARTS;
// Stale max: after the first K/V tile, exponentiate against the running max
// without a per-tile row max; a P part whose row sum exceeds 2^8 (some p may
// exceed the lazy-rescale bound) takes the slow path.
#ifndef TA_STALE_MAX
#define TA_STALE_MAX 1
#endif
constexpr bool kStaleMax = TA_STALE_MAX != 0;
constexpr float kSumGuard = 256.0f;

// every completed mbarrier phase is waited on by some thread (the slow-path
// barriers o_full / o_half included), so compute-sanitizer synccheck sees no
// unobserved phase
// (off in the product build: the observation costs 4-6% -- a same-box A/B;
// scripts/sanitize.sh checks both builds)
#ifndef TA_OBSERVE_PHASES
#define TA_OBSERVE_PHASES 0
#endif
constexpr bool kObservePhases = TA_OBSERVE_PHASES != 0;

#ifndef TA_SLOTS_D128
#define TA_SLOTS_D128 4
#endif
#ifndef TA_TRACE_ROW  // row whose softmax phases the diagnostic trace records
#define TA_TRACE_ROW 0
#endif
#ifndef TA_TMA_STORE_O  // epilogue: TMA store of O from shared memory (1) or 16-B global stores (0)
#define TA_TMA_STORE_O 1
#endif
constexpr bool kTmaStoreO = TA_TMA_STORE_O != 0;
#ifndef TA_SLOTS_D64
#define TA_SLOTS_D64 4
#endif
// D=64, one Q tile per CTA: S rotates through three 64-column TMEM units so
// that S(j+1) is computed while the softmax works on tile j (below)
#ifndef TA_D64_ROT
#define TA_D64_ROT 1
#endif

template <int D, int kQT = kQTilesFor<D>, int kBN = kBN128, bool kPair = false>
struct Cfg {
  static constexpr int kRegions = D / 64;                   // 128-B swizzle atoms along D
  static constexpr int kTileBytes = kBM * D * 2;            // one Q / K / V tile
  static constexpr int kRegionBytes = kBM * 128;            // 128 rows x 128 B
  // kPair (CTA pair, cta_group::2): each CTA holds half of every K / V tile
  // -- K: its kBN / 2 keys x D; V: all kBN keys x its D / 2 columns
  static constexpr int kKVBytes = kBN * D * 2 / (kPair ? 2 : 1);  // one K / V tile (slot)
  static constexpr int kKVRegionBytes = kBN * 128;          // kBN rows x 128 B (V regions)
  static constexpr int kKRegionBytes = (kPair ? kBN / 2 : kBN) * 128;  // K regions
  static_assert(!kPair || (D == 128 && kQT == 2 && kBN == 128), "pair: the D=128 kernel");
  static_assert(kBN == 128 || (kBN == 64 && D == 128 && kQT == 2),
                "64-key tiles: the D=128 split-softmax kernel only");
  // K/V ring depth (two CTAs per SM at kQT = 1: 16 KB Q + 4 x 16 KB ring each)
  // (D > 128: Q + 3 x 48 KB or 2 x 64 KB = 192 KB, one CTA per SM)
  static constexpr int kSlots = D > 128 ? (D == 192 ? 3 : 2)
                                : D == 128 ? (kQT == 1 ? 2 : TA_SLOTS_D128 * (128 / kBN) * (kPair ? 2 : 1))
                                : kQT == 1 ? TA_SLOTS_D64 : 8;
  static constexpr bool kSplit = kSplitFor<D, kQT, kBN>;
  static constexpr int kSmemData = kQT * kTileBytes + kSlots * kKVBytes;
  // (kSplit: + 4 KB of per-row exchange between the two warps of a row:
  // [max | l][Q tile][lane quadrant][column half][lane] floats)
  static constexpr int kSmemXch = kSplit ? 2 * kQT * 4 * 2 * 32 * 4 : 0;
  static constexpr int kSmemBytes = kSmemData + 1024 /*barriers*/ + kSmemXch + 1024 /*align pad*/;
  // S/P rotation (D=64, kQT=1): TMEM units U0 = [0,64), U1 = [64,128),
  // U2 = [128,192), O at [192,256).  S(j) occupies U0U1 (j even) or U1U2 (j
  // odd) and P(j) its unit U0 (even) or U2 (odd), so S(j+1) never touches
  // P(j) and can be issued as soon as the softmax has read S(j).
  static constexpr bool kRot = TA_D64_ROT && kQT == 1 && (D == 64 || D > 128);
  // ring filled in the rotation's consumption order (K_{j+1} before V_j):
  // with the 2-3 slot rings of D > 128 the next K no longer waits behind a V
  // slot that frees only when PV completes (+32-36% at D=160/256; D=64 with
  // 4 slots gains nothing and keeps the plain order)
#ifndef TA_D64_CONSUME
#define TA_D64_CONSUME 0
#endif
  static constexpr bool kConsumeOrder = kRot && (D > 128 || TA_D64_CONSUME);
  static constexpr uint32_t kTmemS = 0;                  // S_t at col 128 t (fp32)
  static constexpr uint32_t kTmemO = kRot ? 192 : 128 * kQT;  // O_t at kTmemO + D t (fp32)
  __device__ static constexpr uint32_t s_col(int j) { return kRot ? 64u * uint32_t(j & 1) : 0u; }
  __device__ static constexpr uint32_t p_col(int j) { return kRot ? 128u * uint32_t(j & 1) : 0u; }
  // P hand-off barriers: with the rotation a warp may write P(j+1) before a
  // slower warp of its warpgroup has written P(j) (S(j+1) only waits for every
  // warp to have READ S(j)), so even and odd tiles arrive on separate
  // barriers (p_full[j & 1], phase j / 2); no warp gets two tiles ahead
  // (S(j+2) waits for PV(j), i.e. for all of P(j)).
  __device__ static constexpr int p_bar(int t, int j) { return kRot ? (j & 1) : t; }
  __device__ static constexpr uint32_t p_parity(int j) { return uint32_t(kRot ? (j >> 1) & 1 : j & 1); }
};

struct Barriers {
  uint64_t q_full;
  uint64_t s_full[kQTiles];
  uint64_t p_full[kQTiles][4];  // P key columns [32q, 32q+32) written (q < kPParts)
  uint64_t o_full[kQTiles];
  uint64_t o_half[kQTiles];  // PV(j) over P part 0 complete (stale-max slow path)
  uint64_t s_read;           // the softmax warps hold S(j) in registers (kRot)
  uint64_t o_last;           // the last PV complete (kRot: o_full may run ahead)
  uint64_t slot_full[8];
  uint64_t slot_empty[8];
  uint32_t tmem_base;
};

template <int D, bool kBF16, bool kTrace, int kQT = kQTilesFor<D>, int kBN = kBN128,
          bool kPair = false>
__global__ void __launch_bounds__(RolesFor<D, kQT, kBN>::kThreads, RolesFor<D, kQT, kBN>::kMinBlocks)
    sdpa_fwd_kernel(const __grid_constant__ CUtensorMap tmap_q,
                    const __grid_constant__ CUtensorMap tmap_k,
                    const __grid_constant__ CUtensorMap tmap_v,
                    const __grid_constant__ CUtensorMap tmap_o, FwdArgs args) {
  using C = Cfg<D, kQT, kBN, kPair>;
  using R = RolesFor<D, kQT, kBN>;
  constexpr int kWarpAlloc = R::kWarpAlloc, kWarpTma = R::kWarpTma, kWarpTrace = R::kWarpTrace,
                kWarpMma = R::kWarpMma;
  // stale max at both head dims: it takes the row max (and its latency)
  // off the softmax of every K/V tile after the first (D=128 +2.3%, D=64
  // with the S/P rotation +4.5%, same-box A/B)
  constexpr bool kStale = kStaleMax;
  constexpr int kEmu16 = D == 64 ? TA_EMU16_D64 : C::kSplit ? TA_EMU16_SPLIT : TA_EMU16_D128;
  static_assert(kEmu16 % 2 == 0 && kEmu16 >= 0 && kEmu16 <= 16, "emulated pairs per 16 columns");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const uint32_t sq = smem_u32(smem);                          // Q tiles
  const uint32_t sring = sq + kQT * C::kTileBytes;             // K/V ring
  Barriers* bars = reinterpret_cast<Barriers*>(smem + C::kSmemData);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const int S = args.seq_len;
  // 1-D grid over (head, query block), query block fastest (concurrent CTAs
  // share a head's K/V in L2); no 65535 limit on B*H
  const int n_qblk = (args.seq_len + kBM * kQT - 1) / (kBM * kQT);
  // CTA pair: clusters of two CTAs on adjacent query blocks of one head (an
  // odd last block gets an idle partner whose rows are all >= S)
  uint32_t rank = 0;
  int bh, qblk_in;
  if constexpr (kPair) {
    rank = cluster_ctarank();
    const int n_pairs = (n_qblk + 1) >> 1;
    const int pair = int(blockIdx.x) >> 1;
    bh = pair / n_pairs;
    qblk_in = (pair - bh * n_pairs) * 2 + int(rank);
  } else {
    bh = int(blockIdx.x) / n_qblk;
    qblk_in = int(blockIdx.x) - bh * n_qblk;
  }
  // causal: heaviest query blocks first (longest-processing-time order)
  const int qblk = args.mask == kMaskCausal ? n_qblk - 1 - qblk_in : qblk_in;
  const int q0 = qblk * (kBM * kQT);
  // keys admitted by the mask (reference MaskSpec::admits, types.hpp:48-67):
  // None -> j < S; Padding -> j < valid_len[b]; Causal -> j <= i, which also
  // bounds the K/V tiles a query tile visits (kv_end = last_row / t_n + 1,
  // tiled.cpp:159).  n_kv_t[t] is the trip count of Q tile t.
  const int kv_len =
      args.mask != kMaskPadding ? S
      : args.valid_len_dev != nullptr ? args.valid_len_dev[(args.bh_offset + bh) / args.heads]
                                      : args.valid_len[(args.bh_offset + bh) / args.heads];
  const int n_kv_seq = (kv_len + kBN - 1) / kBN;
  const int diag0 = q0 / kBN;  // K/V tile on Q tile 0's diagonal (kBN = 128)
  int n_kv_t[kQTiles] = {0, 0};
#pragma unroll
  for (int t = 0; t < kQT; ++t)  // causal: up to the tile holding Q tile t's last row
    n_kv_t[t] = args.mask == kMaskCausal ? min((q0 + (t + 1) * kBM - 1) / kBN + 1, n_kv_seq)
                                         : n_kv_seq;
  const int n_kv = n_kv_t[kQT - 1];  // K/V tiles streamed (max over the Q tiles)
  long long* const trace = (kTrace && blockIdx.x == 0) ? args.trace : nullptr;
  auto rec = [&](int ev, int j) {
    if (trace != nullptr && j < kTraceIters) trace[ev * kTraceIters + j] = clock64();
  };

  if (threadIdx.x == 0) rec(kEvKernelStart, 0);
  // ring position p -> K (kv = 0) or V (kv = 1) of tile j: K_j, V_j
  // alternating, or (kConsumeOrder) the rotation's consumption order K_0,
  // K_1, V_0, K_2, V_1, ..., K_{n-1}, V_{n-2}, V_{n-1}
  auto ring_tile = [&](int p, int& kv, int& j) {
    if constexpr (!C::kConsumeOrder) {
      kv = p & 1;
      j = p >> 1;
    } else {
      kv = p == 0 ? 0 : p == 2 * n_kv - 1 ? 1 : (p & 1) ? 0 : 1;
      j = p == 0 ? 0 : p == 2 * n_kv - 1 ? n_kv - 1 : (p & 1) ? (p + 1) >> 1 : (p - 2) >> 1;
    }
  };
  auto load_ring = [&](int p) {
    int kv, j;
    ring_tile(p, kv, j);
    const int slot = p % C::kSlots;
    const uint32_t fbar = smem_u32(&bars->slot_full[slot]);
#ifdef TA_DEBUG_HALF_KV  // power ablation only (wrong results): half the K/V bytes
    constexpr int kLoadRegions = C::kRegions > 1 ? C::kRegions / 2 : 1;
#else
    constexpr int kLoadRegions = C::kRegions;
#endif
    if constexpr (kPair) {
      // each CTA loads its half into its own slot; the bytes of both halves
      // are counted on the leader's barrier (the MMA issuer waits there)
      const uint32_t fbar0 = mapa_shared(fbar, 0);
      if (rank == 0) mbar_arrive_expect_tx(fbar, 2 * C::kKVBytes);
      if (kv == 0) {  // K: keys [j kBN + 64 rank, + 64), all D columns
        for (int r = 0; r < C::kRegions; ++r)
          tma_load_3d_pair(sring + slot * C::kKVBytes + r * C::kKRegionBytes, &tmap_k, fbar0,
                           r * 64, j * kBN + (kBN / 2) * int(rank), bh);
      } else {  // V: all kBN keys, columns [64 rank, + 64)
        tma_load_3d_pair(sring + slot * C::kKVBytes, &tmap_v, fbar0, 64 * int(rank), j * kBN, bh);
      }
      return;
    }
    mbar_arrive_expect_tx(fbar, kLoadRegions * C::kKVRegionBytes);
    for (int r = 0; r < kLoadRegions; ++r)
      tma_load_3d(sring + slot * C::kKVBytes + r * C::kKVRegionBytes, kv == 0 ? &tmap_k : &tmap_v,
                  fbar, r * 64, j * kBN, bh);
  };
  // The TMA thread initialises the barriers and issues Q and the first ring
  // fill before the CTA barrier (fresh slots need no empty-wait), so the
  // loads overlap the TMEM allocation and the barrier round trip.
  const int ring_prefill = min(C::kSlots, 2 * n_kv);
  if (threadIdx.x == R::kWarpTma * 32) {
    mbar_init(smem_u32(&bars->q_full), 1);
    for (int t = 0; t < kQTiles; ++t)
      for (int q = 0; q < kPParts; ++q)  // one arrive per warp (of both CTAs of a pair)
        mbar_init(smem_u32(&bars->p_full[t][q]), (kBM / 32) * (kPair ? 2 : 1));
    for (int t = 0; t < kQT; ++t) {
      mbar_init(smem_u32(&bars->s_full[t]), 1);
      mbar_init(smem_u32(&bars->o_full[t]), 1);
      mbar_init(smem_u32(&bars->o_half[t]), 1);
    }
    mbar_init(smem_u32(&bars->s_read), kBM / 32);
    mbar_init(smem_u32(&bars->o_last), 1);
    for (int s = 0; s < C::kSlots; ++s) {
      mbar_init(smem_u32(&bars->slot_full[s]), 1);
      mbar_init(smem_u32(&bars->slot_empty[s]), 1);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tmap_q);
    tma_prefetch_desc(&tmap_k);
    tma_prefetch_desc(&tmap_v);
  }
  auto first_loads = [&]() {
    const uint32_t qbar = smem_u32(&bars->q_full);
    if constexpr (kPair) {  // both CTAs' Q tiles counted on the leader's q_full
      if (rank == 0 && n_kv > 0) mbar_arrive_expect_tx(qbar, 2 * kQT * C::kTileBytes);
      const uint32_t qbar0 = mapa_shared(qbar, 0);
      for (int t = 0; t < kQT && n_kv > 0; ++t)
        for (int r = 0; r < C::kRegions; ++r)
          tma_load_3d_pair(sq + t * C::kTileBytes + r * C::kRegionBytes, &tmap_q, qbar0, r * 64,
                           q0 + t * kBM, bh);
    } else {
      if (n_kv > 0) mbar_arrive_expect_tx(qbar, kQT * C::kTileBytes);
      for (int t = 0; t < kQT && n_kv > 0; ++t)  // (no key admitted: Q unused)
        for (int r = 0; r < C::kRegions; ++r)
          tma_load_3d(sq + t * C::kTileBytes + r * C::kRegionBytes, &tmap_q, qbar, r * 64,
                      q0 + t * kBM, bh);
    }
    for (int p = 0; p < ring_prefill; ++p) load_ring(p);
  };
  if (!kPair && threadIdx.x == R::kWarpTma * 32) first_loads();
  if constexpr (kPair) {
    // both CTAs allocate (same warp, same smem offset) and every barrier of
    // the pair is initialised before any cross-CTA load or arrive
    if (warp == kWarpAlloc) tmem_alloc_pair<R::kTmemCols>(smem_u32(&bars->tmem_base));
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    if (threadIdx.x == R::kWarpTma * 32) first_loads();
  } else {
    if (warp == kWarpAlloc) tmem_alloc<R::kTmemCols>(smem_u32(&bars->tmem_base));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  const uint32_t tmem = bars->tmem_base;
  if (threadIdx.x == 0) rec(kEvKernelStart, 1);

  if (warp >= uint32_t(R::kSoftmaxWarps)) {
    if constexpr (R::kSetMaxNReg)
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(R::kRegsControl));
  if (warp == kWarpTma) {
    // ------------------------------------------------------------------ TMA
    if (lane == 0) {
      for (int p = ring_prefill; p < 2 * n_kv; ++p) {
        mbar_wait_ctrl(smem_u32(&bars->slot_empty[p % C::kSlots]),
                       uint32_t((p / C::kSlots) & 1) ^ 1u);
        load_ring(p);
      }
      if constexpr (kPair) {
        // the leader's last slot releases land in this CTA too: wait for them
        // before the teardown so no arrive targets an exited CTA
        for (int p = max(0, 2 * n_kv - C::kSlots); p < 2 * n_kv; ++p)
          mbar_wait_ctrl(smem_u32(&bars->slot_empty[p % C::kSlots]), uint32_t((p / C::kSlots) & 1));
      }
    }
  } else if (warp == kWarpTrace) {
    // optional tracer: timestamps of tensor-core completions (diagnostics only)
    if (kTrace && C::kRot && lane == 0 && trace != nullptr) {  // S(j+1), then PV(j)
      for (int j = 0; j < n_kv && j < kTraceIters; ++j) {
        if (j + 1 < n_kv) {
          mbar_wait(smem_u32(&bars->s_full[0]), uint32_t((j + 1) & 1));
          rec(kEvTcS0Done, j);
        }
        mbar_wait(smem_u32(&bars->o_full[0]), uint32_t(j & 1));
        rec(kEvTcPV0Done, j);
      }
    }
    if (kTrace && kQT == 2 && lane == 0 && trace != nullptr) {
      for (int j = 0; j < n_kv && j < kTraceIters; ++j) {
        mbar_wait(smem_u32(&bars->o_full[0]), uint32_t(j & 1));
        rec(kEvTcPV0Done, j);
        if (j + 1 < n_kv) {
          mbar_wait(smem_u32(&bars->s_full[0]), uint32_t((j + 1) & 1));
          rec(kEvTcS0Done, j);
        }
        mbar_wait(smem_u32(&bars->o_full[1]), uint32_t(j & 1));
        rec(kEvTcPV1Done, j);
        if (j + 1 < n_kv) {
          mbar_wait(smem_u32(&bars->s_full[1]), uint32_t((j + 1) & 1));
          rec(kEvTcS1Done, j);
        }
      }
    }
  } else if (warp == kWarpMma && rank == 0) {  // (pair: the leader issues for both CTAs)
    // ------------------------------------------------------------------ MMA
    // The whole warp runs this loop (uniform control flow, descriptors in
    // uniform registers); one elected lane issues each tcgen05 instruction.
    {
      // (pair: M = 256, 128 rows in each CTA's TMEM)
      constexpr uint32_t kM = kBM * (kPair ? 2 : 1);
      constexpr uint32_t idesc_qk = make_idesc_f16(kBF16, kM, kBN, false, false);
      constexpr uint32_t idesc_pv = make_idesc_f16(kBF16, kM, D, false, true);
      // commits arrive on the barrier in both CTAs of a pair
      auto commit = [&](uint32_t bar) {
        if constexpr (kPair) umma_commit_pair(bar); else umma_commit_warp(bar);
      };
      // wide kernels with a smaller head dim (D=160 on the 192-column kernel,
      // TMA zero-fill past D): QK^T skips the all-zero K-steps and PV computes
      // only the O columns that are stored (+4% at D=160; at D <= 128 the
      // loop is softmax-bound and the trimming measured -1%, so it is off)
      const int n_kstep = D > 128 ? (args.head_dim + 15) >> 4 : D / 16;
      const uint32_t idesc_pv_n =
          D > 128 ? (idesc_pv & ~(0x3Fu << 17)) | (uint32_t(n_kstep * 16 >> 3) << 17) : idesc_pv;
      // ring position r (K_j at 2j, V_j at 2j+1) -> slot / phase
      auto slot_of = [](int r) { return r % C::kSlots; };
      auto phase_of = [](int r) { return uint32_t((r / C::kSlots) & 1); };
      auto wait_full = [&](int r) {
        mbar_wait_ctrl(smem_u32(&bars->slot_full[slot_of(r)]), phase_of(r));
        tc_fence_after();
      };
      auto release = [&](int r) { commit(smem_u32(&bars->slot_empty[slot_of(r)])); };
      // descriptors: base built once, K-step offsets added to the start-address
      // field (addr >> 4; smem addresses < 256 KB never carry out of 14 bits)
      const uint64_t qdesc = sdesc_sw128(sq, 16, 1024);
      const uint64_t kvdesc_k = sdesc_sw128(sring, 16, 1024);
      const uint64_t kvdesc_v = sdesc_sw128(sring, C::kKVRegionBytes, 1024);
      auto issue_qk = [&](int t, int r, uint32_t scol = 0) {
        uint64_t qd = qdesc + uint64_t((t * C::kTileBytes) >> 4);
        uint64_t kd = kvdesc_k + uint64_t((slot_of(r) * C::kKVBytes) >> 4);
        const uint32_t dS = tmem + C::kTmemS + t * kBN + scol;
#pragma unroll
        for (int r = 0; r < C::kRegions; ++r) {  // 4 K-steps of 16 per 128-B swizzle region
          const uint32_t off = (r * C::kRegionBytes) >> 4;      // Q region r
          const uint32_t koff = (r * C::kKRegionBytes) >> 4;  // K region r
#ifdef TA_DEBUG_NO_MMA  // energy ablation only (wrong results): no tensor-core work
          if (true) {
          } else
#endif
          if constexpr (kPair) {
            umma_ss_x4_pair<2, 2>(dS, qd + off, kd + koff, idesc_qk, r > 0);
          } else if (D <= 128 || n_kstep >= 4 * r + 4) {
            umma_ss_x4<2, 2>(dS, qd + off, kd + koff, idesc_qk, r > 0);
          } else {  // head dim below the kernel's: skip the all-zero K-steps
            for (int ks = 0; ks < n_kstep - 4 * r; ++ks)
              umma_ss_warp(dS, qd + off + 2 * ks, kd + koff + 2 * ks, idesc_qk, (r > 0 || ks > 0));
          }
        }
        commit(smem_u32(&bars->s_full[t]));
      };
      // PV in two halves of 64 keys, each issued as soon as the softmax
      // warpgroup has written that half of P (P aliases S in TMEM).
      // Padding: keys >= valid_len inside the last K/V tile are real memory
      // (not TMA zero-fill) and get weight 0; the reference skips zero
      // weights (online_update, tiled.hpp:215-216), so a NaN / inf there
      // must not reach O: the MMA warp zeroes those V rows (whole 128-B
      // swizzle rows) before the tile's first PV reads the slot.
      auto zero_v_tail = [&](int r, int j) {
        if (args.mask != kMaskPadding || j != n_kv_seq - 1) return;
        const int r0 = kv_len - j * kBN;  // first masked key row of the tile
        if (r0 >= kBN) return;
        const uint32_t vbase = sring + slot_of(r) * C::kKVBytes;
        if constexpr (kPair) {
          // each CTA of the pair holds 64 of the V columns (one region): the
          // leader's MMA warp zeroes the rows in both through shared::cluster
          for (uint32_t cta = 0; cta < 2; ++cta) {
            const uint32_t vb = mapa_shared(vbase, cta);
            for (int i = r0 * 8 + int(lane); i < kBN * 8; i += 32)  // 16-B pieces
              st_cluster_zero_v4(vb + (i >> 3) * 128 + (i & 7) * 16);
          }
          fence_proxy_async_cluster();
        } else {
          for (int i = r0 * 8 + int(lane); i < kBN * 8; i += 32) {  // 16-B pieces
            for (int g = 0; g < C::kRegions; ++g)
              st_shared_v4(vbase + g * C::kKVRegionBytes + (i >> 3) * 128 + (i & 7) * 16, 0u, 0u,
                           0u, 0u);
          }
          fence_proxy_async_smem();  // generic-proxy writes before the tensor core reads
        }
        __syncwarp();
      };
      auto issue_pv = [&](int t, int r, bool accumulate, int j) {
        const uint32_t tP = tmem + C::kTmemS + t * kBN + C::p_col(j);
        uint64_t vd = kvdesc_v + uint64_t((slot_of(r) * C::kKVBytes) >> 4);
#pragma unroll
        for (int h = 0; h < kPParts; ++h) {
          mbar_wait_ctrl(smem_u32(&bars->p_full[C::p_bar(t, j)][h]), C::p_parity(j));
          tc_fence_after();
          if (h == kPParts - 1 && lane == 0) rec(t == 0 ? kEvMmaWaitP0 : kEvMmaWaitP1, j);
          static_assert((kBN / 16 / kPParts) % 2 == 0, "P part = 2k K-steps of 16 keys");
          constexpr int kSteps = kBN / 16 / kPParts;
          constexpr int kVStep = (16 * 128) >> 4;  // 16 V rows per K-step
          // P columns: 8 per K-step of 16 keys; split softmax: part h (one
          // warp's kBN / 2 keys) over the first kBN / 4 S columns of its half
          const uint32_t tPh = tP + (C::kSplit ? h * (kBN / 2 - kSteps * 8) : 0);
#ifdef TA_DEBUG_NO_MMA
          if (false)
#endif
          if constexpr (kSteps % 4 == 0) {
#pragma unroll
            for (int g = 0; g < kSteps / 4; ++g) {
              const int ks0 = h * kSteps + g * 4;
              if constexpr (kPair)
                umma_ts_x4_pair<kVStep>(tmem + C::kTmemO + t * D, tPh + ks0 * 8,
                                        vd + uint64_t((ks0 * 16 * 128) >> 4), idesc_pv_n,
                                        (accumulate || ks0 > 0) ? 1u : 0u);
              else
                umma_ts_x4<kVStep>(tmem + C::kTmemO + t * D, tPh + ks0 * 8,
                                   vd + uint64_t((ks0 * 16 * 128) >> 4), idesc_pv_n,
                                   (accumulate || ks0 > 0) ? 1u : 0u);
            }
          } else {
#pragma unroll
            for (int g = 0; g < kSteps / 2; ++g) {
              const int ks0 = h * kSteps + g * 2;
              umma_ts_x2<kVStep>(tmem + C::kTmemO + t * D, tPh + ks0 * 8,
                                 vd + uint64_t((ks0 * 16 * 128) >> 4), idesc_pv_n,
                                 (accumulate || ks0 > 0) ? 1u : 0u);
            }
          }
          if (kStale && h == 0 && !C::kSplit) commit(smem_u32(&bars->o_half[t]));
        }
        commit(smem_u32(&bars->o_full[t]));
        if (lane == 0) rec(t == 0 ? kEvMmaIssuedPV0 : kEvMmaIssuedPV1, j);
      };

      if constexpr (C::kRot) {
        // S(j+1) as soon as the softmax holds S(j) in registers (its columns
        // are disjoint from P(j)'s), then PV(j) once P(j) lands
        const int n = n_kv_t[0];
        if (n > 0) {
          mbar_wait(smem_u32(&bars->q_full), 0);
          tc_fence_after();
          wait_full(0);
          issue_qk(0, 0, C::s_col(0));
          release(0);
          for (int j = 0; j + 1 < n; ++j) {
            // K_{j+1}'s ring position (written out: a constexpr helper
            // call here changes nvcc's unrolling of this loop at D=64 and
            // costs 100 spill instructions)
            int rk = 2 * (j + 1);
            if constexpr (C::kConsumeOrder) rk = 2 * j + 1;
            mbar_wait_ctrl(smem_u32(&bars->s_read), uint32_t(j & 1));
            tc_fence_after();
            if (lane == 0) rec(kEvMmaWaitP1, j);  // (rotation traces: s_read(j) seen)
            wait_full(rk);
            if (lane == 0) rec(kEvMmaIssuedPV1, j);  // (... K_{j+1} landed)
            issue_qk(0, rk, C::s_col(j + 1));
            if (lane == 0) rec(kEvSm1PArrive, j);  // (... QK(j+1) issued)
            release(rk);
            int rv = 2 * j + 1;  // V_j
            if constexpr (C::kConsumeOrder) rv = 2 * j + 2;
            wait_full(rv);
            issue_pv(0, rv, j > 0, j);
            release(rv);
          }
          // the last V tile (peeled: the padding tail is zeroed outside the
          // steady-state loop, whose code nvcc otherwise schedules worse)
          const int rv = 2 * n - 1;
          wait_full(rv);
          zero_v_tail(rv, n - 1);
          issue_pv(0, rv, n > 1, n - 1);
          release(rv);
          umma_commit_warp(smem_u32(&bars->o_last));
        }
      } else if constexpr (kQT == 1) {
        // one Q tile: PV(j-1) once P(j-1) lands, then S(j); the tensor core
        // idles through this CTA's softmax, which the other CTA on the SM fills
        const int n = n_kv_t[0];
        if (n > 0) {
          mbar_wait(smem_u32(&bars->q_full), 0);
          tc_fence_after();
          wait_full(0);
          issue_qk(0, 0);
          release(0);
          for (int j = 1; j < n; ++j) {
            // S(j) overwrites the S / P columns PV(j-1) reads: in-order
            // after it on the tensor pipe
            // (V_{j-1} is never the padding tail: that is tile n - 1)
            const int rk = 2 * j, rv = 2 * j - 1;
            wait_full(rv);
            issue_pv(0, rv, j > 1, j - 1);
            release(rv);
            wait_full(rk);
            issue_qk(0, rk);
            release(rk);
          }
          const int rv = 2 * n - 1;
          wait_full(rv);
          zero_v_tail(rv, n - 1);
          issue_pv(0, rv, n > 1, n - 1);
          release(rv);
        }
      }
      // Q tile 0 visits n0 <= n1 K/V tiles (fewer under the causal mask)
      const int n0 = n_kv_t[0], n1 = n_kv_t[1];
      if (kQT == 2 && n1 > 0) {
        mbar_wait(smem_u32(&bars->q_full), 0);
        tc_fence_after();
        wait_full(0);
        if (n0 > 0) issue_qk(0, 0);
        issue_qk(1, 0);
        release(0);
        for (int j = 1; j < n1; ++j) {
          // (V_{j-1} is never the padding tail: padding has n1 = n_kv_seq)
          const int rk = 2 * j, rv = 2 * j - 1;
          wait_full(rv);
          if (j - 1 < n0) issue_pv(0, rv, j > 1, j - 1);
          wait_full(rk);
          if (j < n0) issue_qk(0, rk);
          issue_pv(1, rv, j > 1, j - 1);
          release(rv);
          issue_qk(1, rk);
          release(rk);
        }
        const int rv = 2 * n1 - 1;
        wait_full(rv);
        zero_v_tail(rv, n1 - 1);
        if (n1 - 1 < n0) issue_pv(0, rv, n1 > 1, n1 - 1);
        issue_pv(1, rv, n1 > 1, n1 - 1);
        release(rv);
      }
    }
  }
  } else if constexpr (C::kSplit) {
    // --------------------------------------------------- softmax, split rows
    // Two warps per TMEM lane quadrant and Q tile: warp w owns tile t = w / 8,
    // quadrant w % 4 (rows 32 (w % 4) + lane) and key columns [64 c, 64 c + 64)
    // of each 128-key tile, c = (w / 4) % 2.  Per SMSP that is four softmax
    // warps (both tiles, both halves): a tile's 128 exps per row are issued by
    // two warps at once, which halves the per-warp MUFU issue chain that bounds
    // the one-warp-per-row softmax (profiles/r02/microbench.md).  The two warps
    // of a row share the running max: exact on the first tile (exchanged
    // through shared memory), stale afterwards with the half-row sums voted
    // (bar.red.or) so both halves take the slow path together.  Each keeps its
    // own partial l; P of its 64 keys goes over its own first 32 S columns
    // (16-bit pairs); the epilogue normalises its half of the O columns.
    if constexpr (R::kSetMaxNReg)
      asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(R::kRegsSoftmax));
    const int t = int(warp) / 8;
    const int c = int(warp / 4) & 1;
    const uint32_t wq = warp & 3;
    const int row = int(wq * 32 + lane);
    const uint32_t lane_off = (wq * 32u) << 16;
    constexpr int kHalf = kBN / 2;  // key columns per warp
    const uint32_t tS = tmem + lane_off + C::kTmemS + t * kBN + kHalf * c;  // its S columns
    const uint32_t tO = tmem + lane_off + C::kTmemO + t * D + (D / 2) * c;  // its O columns
    const float sl2 = args.scale_log2;
    const uint32_t sbar = smem_u32(&bars->s_full[t]);
    const uint32_t obar = smem_u32(&bars->o_full[t]);
    const uint32_t pbar = smem_u32(&bars->p_full[t][c]);
    const uint32_t pair_bar = 1 + t * 4 + wq;  // named barrier of the row's two warps
    // exchange slots [max|l][t][wq][c][lane]
    float* xch = reinterpret_cast<float*>(smem + C::kSmemData + 1024);
    float* xm_mine = xch + ((t * 4 + int(wq)) * 2 + c) * 32 + lane;
    float* xm_other = xch + ((t * 4 + int(wq)) * 2 + (c ^ 1)) * 32 + lane;
    constexpr int kXL = 2 * 4 * 2 * 32;  // offset of the l slots
    auto pair_max = [&](float v) {
      *xm_mine = v;
      named_bar_sync(pair_bar, 64);
      return fmaxf(v, *xm_other);
    };
    auto pair_max_nan = [&](float v) {  // (slow path: a NaN half poisons the row)
      *xm_mine = v;
      named_bar_sync(pair_bar, 64);
      return fmax_nan(v, *xm_other);
    };
    constexpr int kEmu = kEmu16;
    float m_run = -INFINITY;  // shared by the row's two warps (scaled, log2 units)
    float l_run = 0.f;        // this warp's partial normaliser over its columns
    const int my_n_kv = n_kv_t[t];
    const uint64_t sl2x2 = f2(sl2, sl2);

    auto load_s = [&](float (&sv)[kHalf], int j) {
      uint32_t sr[kHalf / 32][32];
#pragma unroll
      for (int h = 0; h < kHalf / 32; ++h) tmem_ld32(tS + 32 * h, sr[h]);
      tmem_wait_ld();
#pragma unroll
      for (int h = 0; h < kHalf / 32; ++h) reg_fence(sr[h]);
#pragma unroll
      for (int h = 0; h < kHalf / 32; ++h)
#pragma unroll
        for (int i = 0; i < 32; ++i) sv[h * 32 + i] = __uint_as_float(sr[h][i]);
      // last admitted key of this row in the tile (ragged tail / padding /
      // causal: key j kBN + i admitted iff <= query q0 + 128 t + row); column
      // i here is key kHalf c + i of the tile
      int lim = kBN - 1;
      if (j == n_kv_seq - 1) lim = min(lim, kv_len - j * kBN - 1);
      if (args.mask == kMaskCausal) lim = min(lim, q0 + t * kBM + row - j * kBN);
      lim -= kHalf * c;
      if (lim < kHalf - 1) {
#pragma unroll
        for (int i = 0; i < kHalf; ++i)
          if (i > lim) sv[i] = -INFINITY;
      }
    };
    // exps of the warp's 64 columns against m_use: P packed into pk, sum
    auto exps = [&](const float (&sv)[kHalf], float m_use, uint32_t (&pk)[kHalf / 2]) {
      const uint64_t negm2 = f2(-m_use, -m_use);
      uint64_t acc[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
      for (int g = 0; g < kHalf / 8; ++g) {  // groups of 8 columns
        const int c0 = g * 8;
        const int emu_pairs = (g & 1) ? kEmu / 4 : kEmu / 2 - kEmu / 4;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint64_t x = ffma2(f2(sv[c0 + 2 * u], sv[c0 + 2 * u + 1]), sl2x2, negm2);
          float p0, p1;
          if (u >= 4 - emu_pairs) {
            ex2_poly2(x, p0, p1);
          } else {
            float a, b;
            f2_split(x, a, b);
            p0 = ex2(a);
            p1 = ex2(b);
          }
          acc[u] = fadd2(acc[u], f2(p0, p1));
          pk[g * 4 + u] = pack2<kBF16>(p0, p1);
        }
      }
      float lo, hi;
      f2_split(fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3])), lo, hi);
      return lo + hi;
    };

    for (int j = 0; j < my_n_kv; ++j) {
      mbar_wait(sbar, uint32_t(j & 1));
      tc_fence_after();
      const bool tr = kTrace && row == TA_TRACE_ROW && c == 0;
      if (tr) rec(kEvSm0SReady + 5 * t, j);
      float sv[kHalf];
      load_s(sv, j);
      if (tr) rec(kEvSm0Loaded + 5 * t, j);
      if (j == 0) {
        // first tile: the exact row max over both halves (no O yet)
        float mx4[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) mx4[i] = sv[i];
#pragma unroll
        for (int i = 4; i < kHalf; ++i) mx4[i & 3] = fmaxf(mx4[i & 3], sv[i]);
        const float mx = pair_max(fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3])));
        m_run = mx * sl2;
        if (tr) rec(kEvSm0Max + 5 * t, j);
      }
      float m_use = m_run == -INFINITY ? 0.f : m_run;
      uint32_t pk[kHalf / 2];
      float psum = exps(sv, m_use, pk);
      if (tr) rec(kEvSm0Exp + 5 * t, j);
      // stale max: if some p of either half may exceed 2^8 (sum > 2^8, inf or
      // NaN), both warps move m to the row's true max, rescale l and their O
      // columns (after PV(j-1) has landed; PV(j) waits for this P) and redo
      if (j > 0 && named_bar_or(pair_bar, 64, !(psum <= kSumGuard))) {
        load_s(sv, j);  // S(j) is intact: P(j) is not written yet
        float mx4[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) mx4[i] = sv[i];
#pragma unroll
        for (int i = 4; i < kHalf; ++i) mx4[i & 3] = fmax_nan(mx4[i & 3], sv[i]);
        const float m_new =
            pair_max_nan(fmax_nan(fmax_nan(mx4[0], mx4[1]), fmax_nan(mx4[2], mx4[3]))) * sl2;
        const bool need = m_new > m_run;
        const float alpha = need ? ex2(m_run - m_new) : 1.f;
        if (need) {
          l_run *= alpha;
          m_run = m_new;
          m_use = m_run;
        }
        // the row's whole O is rescaled by its c = 0 warp: PV(j) over the first
        // key half -- issued once the four c = 0 warps have handed off P --
        // accumulates into every O column, so a c = 1 warp still rescaling
        // its half would race with it
        if (c == 0) {
          mbar_wait(obar, uint32_t((j - 1) & 1));
          tc_fence_after();
          const uint32_t tOrow = tO - (D / 2) * c;  // (c == 0: the tile's O columns)
#pragma unroll 1
          for (int cc = 0; cc < D; cc += 16) {
            uint32_t orow[16];
            tmem_ld16(tOrow + cc, orow);
            tmem_wait_ld();
            reg_fence(orow);
#pragma unroll
            for (int i = 0; i < 16; ++i)
              orow[i] = __float_as_uint(__uint_as_float(orow[i]) * alpha);
            tmem_st16(tOrow + cc, orow);
          }
        }
        psum = exps(sv, m_use, pk);
        // a NaN score (NaN in q or k) reaches this path on every row it hits
        // (MUFU gives NaN, the FMA-pipe emulation saturates at 2^127); the
        // NaN-propagating max above carries it into m_new: make the row's l
        // NaN so its O and LSE are NaN, as the reference's are
        if (kEmu > 0 && m_new != m_new) psum = __int_as_float(0x7fffffff);
      }
      l_run += psum;
      // observe o_full's phase j-1 (PV(j-1)) before P(j) lets PV(j) complete
      // phase j: S(j) was issued after PV(j-1), so it has completed (one
      // test_wait).  Only the slow path needs o_full, but an unobserved phase
      // is what compute-sanitizer synccheck reports ("missing wait").
      if (kObservePhases && j > 0 && lane == 0) mbar_observe(obar, uint32_t((j - 1) & 1));
#pragma unroll
      for (int i = 0; i < kHalf / 32; ++i)
        tmem_st16(tS + 16 * i, *reinterpret_cast<uint32_t(*)[16]>(&pk[16 * i]));
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (kPair)  // the leader's barrier (the MMA issuer waits there)
          mbar_arrive_cluster(mapa_shared(pbar, 0));
        else
          mbar_arrive(pbar);
      }
      if (tr) rec(kEvSm0PArrive + 5 * t, j);
      // warp skew of tile 0 (trace builds): W1 = the row partner (wq 0, c 1),
      // W2 / W3 = the two warps on the MMA warp's SMSP (wq 3, c 0 / 1)
      if (kTrace && t == 0 && lane == TA_TRACE_ROW && (wq == 0 ? c == 1 : wq == 3))
        rec(wq == 0 ? kEvSm0ArriveW1 : kEvSm0ArriveW2 + c, j);
    }

    // ------------------------------------------------------ epilogue (split)
    if (my_n_kv > 0) {
      mbar_wait(obar, uint32_t((my_n_kv - 1) & 1));
      tc_fence_after();
    }
    xch[kXL + ((t * 4 + int(wq)) * 2 + c) * 32 + lane] = l_run;
    named_bar_sync(pair_bar, 64);
    const float l_tot = l_run + xch[kXL + ((t * 4 + int(wq)) * 2 + (c ^ 1)) * 32 + lane];
    const int grow = q0 + t * kBM + row;
    const float inv_l = l_tot != 0.f ? 1.f / l_tot : 0.f;  // finalize: l == 0 -> zeros (NaN propagates)
    const int dm = args.head_dim;
    const uint32_t so = sq + t * C::kTileBytes;  // the tile's (dead) Q buffer
#pragma unroll
    for (int h = 0; h < D / 64; ++h) {  // its D / 2 O columns, 32 at a time
      uint32_t orow[32];
      if (my_n_kv > 0) {
        tmem_ld32(tO + h * 32, orow);
        tmem_wait_ld();
        reg_fence(orow);
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) orow[i] = 0u;
      }
      uint32_t packed[16];
#pragma unroll
      for (int i = 0; i < 16; ++i)
        packed[i] = pack2<kBF16>(__uint_as_float(orow[2 * i]) * inv_l,
                                 __uint_as_float(orow[2 * i + 1]) * inv_l);
#pragma unroll
      for (int i = 0; i < 4; ++i) {  // 16-B chunk k of the row's 128-B line, XOR row % 8
        const int gcol = c * (D / 2) + h * 32 + i * 8;
        const uint32_t k = uint32_t((gcol & 63) >> 3);
        st_shared_v4(so + (gcol >> 6) * C::kRegionBytes + row * 128 + ((k ^ (row & 7)) << 4),
                     packed[4 * i], packed[4 * i + 1], packed[4 * i + 2], packed[4 * i + 3]);
      }
    }
    fence_proxy_async_smem();
    named_bar_sync(9 + t, 2 * kBM);  // the tile's eight softmax warps
    if (row == 0 && c == 0) {
      for (int r = 0; r < C::kRegions; ++r)
        if (r * 64 < dm) tma_store_3d(&tmap_o, sq + t * C::kTileBytes + r * C::kRegionBytes, r * 64,
                                      q0 + t * kBM, bh);
      tma_store_commit();
    }
    if (c == 0 && args.lse != nullptr && grow < S)
      args.lse[size_t(bh) * S + grow] =
          l_tot != 0.f ? (m_run + __log2f(l_tot)) * kLn2 : -INFINITY;
    if (row == 0 && c == 0) tma_store_wait_read0();
    if (kTrace && row == 0 && c == 0) rec(kEvEpilogueDone, t);
  } else {
    // -------------------------------------------------------------- softmax
    if constexpr (R::kSetMaxNReg)
      asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(R::kRegsSoftmax));
    const int t = int(warp) / 4;
    const uint32_t wq = warp & 3;  // TMEM lane quadrant accessible to this warp
    const int row = int(wq * 32 + lane);
    const uint32_t lane_off = (wq * 32u) << 16;
    const uint32_t tS0 = tmem + lane_off + C::kTmemS + t * kBN;
    const uint32_t tO = tmem + lane_off + C::kTmemO + t * D;
    const float sl2 = args.scale_log2;
    const uint32_t sbar = smem_u32(&bars->s_full[t]);
    const uint32_t obar = smem_u32(&bars->o_full[t]);

    float m_run = -INFINITY;  // running max used for the exponent (scaled, log2 units)
    float l_run = 0.f;        // running normaliser relative to m_run

    const int my_n_kv = n_kv_t[t];
    for (int j = 0; j < my_n_kv; ++j) {
      // (rotation traces: warp 0 about to wait for S(j); j = 0 is overwritten
      // by the row-max stamp below)
      if (kTrace && C::kRot && row == TA_TRACE_ROW) rec(kEvSm0Max + 5 * t, j);
      mbar_wait(sbar, uint32_t(j & 1));
      // observe PV(j-1)'s o_full / o_half phases (synccheck "missing wait"):
      // without the rotation S(j) follows PV(j-1) in issue order, so both are
      // complete (never blocks); with it (S(j+1) is issued before PV(j)) this
      // happens before P(j)'s first hand-off, below
      if (kObservePhases && !C::kRot && j > 0 && lane == 0) {
        mbar_observe(obar, uint32_t((j - 1) & 1));
        if (kStale) mbar_observe(smem_u32(&bars->o_half[t]), uint32_t((j - 1) & 1));
      }
      tc_fence_after();
      const bool tr = kTrace && row == TA_TRACE_ROW;
      if (tr) rec(kEvSm0SReady + 5 * t, j);
      // (one-tile rotation traces: S ready / loaded as seen by warps 1..3)
      if (kTrace && C::kRot && wq > 0 && lane == 0) rec(kEvSm1SReady + int(wq) - 1, j);
      const uint32_t tS = tS0 + C::s_col(j);  // S(j)
      const uint32_t tP = tS0 + C::p_col(j);  // P(j)
      uint32_t sr[4][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32(tS + c * 32, sr[c]);
      tmem_wait_ld();
      if constexpr (C::kRot) {  // S(j) is in registers: its columns may take S(j+1)
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&bars->s_read));
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) reg_fence(sr[c]);
      if (tr) rec(kEvSm0Loaded + 5 * t, j);
      if (kTrace && C::kRot && wq == 3 && lane == 0) rec(kEvSm1Exp, j);  // (warp 3 loaded)
      float s[128];
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int i = 0; i < 32; ++i) s[c * 32 + i] = __uint_as_float(sr[c][i]);

      {
        // last admitted column of this row in the tile: the ragged tail
        // (keys >= S, zero-filled by TMA, or >= valid_len[b]) and, on the
        // causal diagonal tile, key q0 + 128 t + i admitted iff i <= row (q0
        // is a multiple of the key tile, so the offsets cancel)
        int lim = kBN - 1;
        if (j == n_kv_seq - 1) lim = min(lim, kv_len - j * kBN - 1);
        if (args.mask == kMaskCausal && j == diag0 + t) lim = min(lim, row);
        if (lim < kBN - 1) {
#pragma unroll
          for (int i = 0; i < 128; ++i)
            if (i > lim) s[i] = -INFINITY;
        }
      }
      // row max (8 independent chains); with kStale only on the first
      // tile: later tiles exponentiate against the running max directly and
      // the half-row sum guards the lazy-rescale invariant (below)
      if (!kStale || j == 0) {
      float mx8[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) mx8[i] = s[i];
#pragma unroll
      for (int i = 8; i < 128; ++i) mx8[i & 7] = fmaxf(mx8[i & 7], s[i]);
      const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                             fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
      const float m_new = mx * sl2;
      if (tr) rec(kEvSm0Max + 5 * t, j);
      const bool need = m_new > m_run + kRescaleThreshold;
      const float alpha = need ? ex2(m_run - m_new) : 1.f;  // 0 on the first tile
      if (need) {
        l_run *= alpha;
        m_run = m_new;
      }
      if (j > 0 && __any_sync(0xffffffffu, need)) {
        // O correction (rare with the lazy threshold): wait until PV(j-1) has
        // landed in TMEM and rescale in place; PV(j) is not issued before this
        // warpgroup signals the first half of P(j).
        mbar_wait(obar, uint32_t((j - 1) & 1));
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          uint32_t orow[32];
          tmem_ld32(tO + c * 32, orow);
          tmem_wait_ld();
          reg_fence(orow);
#pragma unroll
          for (int i = 0; i < 32; ++i)
            orow[i] = __float_as_uint(__uint_as_float(orow[i]) * alpha);
          tmem_st32(tO + c * 32, orow);
        }
      }
      }
      float m_use = m_run == -INFINITY ? 0.f : m_run;
      // x = s * scale*log2e - m as packed FFMA2; exp2 split between the MUFU
      // and the FMA pipe (kEmu16 of every 16 columns, emulated in pairs);
      // row sum as packed FADD2 into 4 pair accumulators.
      const uint64_t sl2x2 = f2(sl2, sl2);
      // exps of the row in kPParts parts
#pragma unroll
      for (int h = 0; h < kPParts; ++h) {
        constexpr int kCols = kBN / kPParts;  // key columns per P part
        uint32_t pk[kCols / 32][16];
        uint64_t acc[4];
        auto part_exps = [&]() {
        const uint64_t negm2 = f2(-m_use, -m_use);
        acc[0] = acc[1] = acc[2] = acc[3] = 0ull;
#pragma unroll
        for (int g = 0; g < kCols / 8; ++g) {  // groups of 8 columns
          const int c0 = h * kCols + g * 8;
          uint64_t x[4];
#pragma unroll
          for (int u = 0; u < 4; ++u)
            x[u] = ffma2(f2(s[c0 + 2 * u], s[c0 + 2 * u + 1]), sl2x2, negm2);
          float p[8];
          // emulated pairs are the last ones of the group: of the kEmu16/2
          // pairs per 16 columns, even groups take the larger half
          const int emu_pairs = (g & 1) ? kEmu16 / 4 : kEmu16 / 2 - kEmu16 / 4;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
#ifdef TA_DEBUG_NO_EXP  // timing ablation only: wrong results
            if (true) {
              f2_split(x[u], p[2 * u], p[2 * u + 1]);
            } else
#endif
            if (u >= 4 - emu_pairs) {
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
            acc[u] = fadd2(acc[u], f2(p[2 * u], p[2 * u + 1]));
            pk[(g * 4 + u) / 16][(g * 4 + u) % 16] = pack2<kBF16>(p[2 * u], p[2 * u + 1]);
          }
        }
        };
        part_exps();
        float psum;
        {
          const uint64_t a01 = fadd2(acc[0], acc[1]);
          const uint64_t a23 = fadd2(acc[2], acc[3]);
          float lo, hi;
          f2_split(fadd2(a01, a23), lo, hi);
          psum = lo + hi;
        }
        if (kStale && j > 0 && __any_sync(0xffffffffu, !(psum <= kSumGuard))) {
          // rare: some p of this part may exceed 2^8 (or overflowed): move
          // m_run to the part's max, rescale l and O, redo the part.  O is
          // stable here: PV(j-1) (part 0) or PV(j) over the earlier parts
          // (o_half) has landed; this part is not yet handed off.
          float hm4[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) hm4[i] = s[h * kCols + i];
#pragma unroll
          for (int i = 4; i < kCols; ++i) hm4[i & 3] = fmax_nan(hm4[i & 3], s[h * kCols + i]);
          const float m_part = fmax_nan(fmax_nan(hm4[0], hm4[1]), fmax_nan(hm4[2], hm4[3])) * sl2;
          const bool need = !(psum <= kSumGuard) && m_part > m_run;
          const float alpha = need ? ex2(m_run - m_part) : 1.f;
          if (need) {
            l_run *= alpha;
            m_run = m_part;
            m_use = m_run;
          }
          // (with the S/P rotation S(j) done only implies PV(j-2) done:
          // PV(j-1) complete first makes the o_half parity unambiguous)
          if (h == 0 || C::kRot) mbar_wait(obar, uint32_t((j - 1) & 1));
          if (h != 0) mbar_wait(smem_u32(&bars->o_half[t]), uint32_t(j & 1));
          tc_fence_after();
#pragma unroll 1
          for (int c = 0; c < D / 16; ++c) {
            uint32_t orow[16];
            tmem_ld16(tO + c * 16, orow);
            tmem_wait_ld();
            reg_fence(orow);
#pragma unroll
            for (int i = 0; i < 16; ++i)
              orow[i] = __float_as_uint(__uint_as_float(orow[i]) * alpha);
            tmem_st16(tO + c * 16, orow);
          }
          part_exps();
          const uint64_t a01 = fadd2(acc[0], acc[1]);
          const uint64_t a23 = fadd2(acc[2], acc[3]);
          float lo, hi;
          f2_split(fadd2(a01, a23), lo, hi);
          psum = lo + hi;
          // a NaN score reaches this path on every row it hits (MUFU gives
          // NaN, the FMA-pipe emulation saturates at 2^127); the NaN-
          // propagating part max carries it: l NaN -> O, LSE NaN
          if (kEmu16 > 0 && m_part != m_part) psum = __int_as_float(0x7fffffff);
        }
        l_run += psum;
#pragma unroll
        for (int i = 0; i < kCols / 32; ++i) tmem_st16(tP + h * (kCols / 2) + i * 16, pk[i]);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (kObservePhases && C::kRot && h == 0 && j > 0 && lane == 0) {
          // rotation: observe PV(j-1)'s o_full / o_half phases before P(j)
          // can let PV(j) complete the next ones (parity stays unambiguous;
          // PV(j-1) depends only on P(j-1), already handed off)
          mbar_observe(obar, uint32_t((j - 1) & 1));
          if (kStale) mbar_observe(smem_u32(&bars->o_half[t]), uint32_t((j - 1) & 1));
        }
        if (lane == 0) {
          if constexpr (kPair)  // the leader's barrier (the MMA issuer waits there)
            mbar_arrive_cluster(mapa_shared(smem_u32(&bars->p_full[C::p_bar(t, j)][h]), 0));
          else
            mbar_arrive(smem_u32(&bars->p_full[C::p_bar(t, j)][h]));
        }
        if (h == 0 && tr) rec(kEvSm0Exp + 5 * t, j);
        if (kTrace && h == kPParts - 1 && t == 0 && wq > 0 && lane == 0)
          rec(kEvSm0ArriveW1 + int(wq) - 1, j);
      }
      if (tr) rec(kEvSm0PArrive + 5 * t, j);
    }

    // ------------------------------------------------------------- epilogue
    // rows with no admitted key (padding valid_len == 0) are exact zeros
    // with LSE = -inf (finalize, tiled.hpp:231-233); their O was never written
    // (kRot: when the softmax finishes, S(n-1) done only implies PV(n-3)
    // done, so o_full's phase parity is ambiguous; o_last completes once)
    if (my_n_kv > 0) {
      if constexpr (C::kRot)
        mbar_wait(smem_u32(&bars->o_last), 0u);
      else
        mbar_wait(obar, uint32_t((my_n_kv - 1) & 1));
      tc_fence_after();
    }
    const int grow = q0 + t * kBM + row;
    const float inv_l = l_run != 0.f ? 1.f / l_run : 0.f;  // finalize: l == 0 -> zeros (NaN propagates)
    const int dm = args.head_dim;  // stored columns (<= D)
    uint16_t* orow_g = reinterpret_cast<uint16_t*>(args.o) + (size_t(bh) * S + grow) * dm;
    // TMA-store epilogue: the tile's rows go to its (now dead) Q buffer in the
    // 128B-swizzled layout the O tensor map expects, then one thread stores
    // the tile (rows >= S and columns >= D clipped by the map)
    const uint32_t so = sq + t * C::kTileBytes;
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
      uint32_t orow[32];
      if (my_n_kv > 0) {
        tmem_ld32(tO + c * 32, orow);
        tmem_wait_ld();
        reg_fence(orow);
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) orow[i] = 0u;
      }
      uint32_t packed[16];
#pragma unroll
      for (int i = 0; i < 16; ++i)
        packed[i] = pack2<kBF16>(__uint_as_float(orow[2 * i]) * inv_l,
                                 __uint_as_float(orow[2 * i + 1]) * inv_l);
      if constexpr (kTmaStoreO) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {  // 16-B chunk k of the row's 128-B line, XOR row % 8
          const uint32_t k = uint32_t((c & 1) * 4 + i);
          st_shared_v4(so + (c >> 1) * C::kRegionBytes + row * 128 + ((k ^ (row & 7)) << 4),
                       packed[4 * i], packed[4 * i + 1], packed[4 * i + 2], packed[4 * i + 3]);
        }
      } else if (grow < S) {
        uint4* dst = reinterpret_cast<uint4*>(orow_g + c * 32);
#pragma unroll
        for (int i = 0; i < 4; ++i)  // 16-B pieces of 8 columns; dm is a multiple of 8
          if (c * 32 + i * 8 < dm)
            dst[i] = make_uint4(packed[4 * i], packed[4 * i + 1], packed[4 * i + 2],
                                packed[4 * i + 3]);
      }
    }
    if constexpr (kTmaStoreO) {
      fence_proxy_async_smem();
      named_bar_sync(1 + t, kBM);  // the tile's four softmax warps
      if (row == 0) {
        for (int r = 0; r < C::kRegions; ++r)
          if (r * 64 < dm) tma_store_3d(&tmap_o, so + r * C::kRegionBytes, r * 64, q0 + t * kBM, bh);
        tma_store_commit();
      }
    }
    if (args.lse != nullptr && grow < S)
      args.lse[size_t(bh) * S + grow] =
          l_run != 0.f ? (m_run + __log2f(l_run)) * kLn2 : -INFINITY;
    if (kTmaStoreO && row == 0) tma_store_wait_read0();  // smem stays valid until read
    if (kTrace && row == 0) rec(kEvEpilogueDone, t);
  }

  tc_fence_before();
  if constexpr (kPair) cluster_sync_all(); else __syncthreads();
  tc_fence_after();
  if (warp == kWarpAlloc) {
    if constexpr (kPair) tmem_dealloc_pair<R::kTmemCols>(tmem);
    else tmem_dealloc<R::kTmemCols>(tmem);
  }
}

#include "sdpa_d64_sm100.cuh"

// ----------------------------------------------------------------------------
// Descriptor self-test: one 128x128x128 UMMA product, checked on the host.
//   mode 0: D = A * B^T, A [128][128] K-major, B [128 n][128 k] K-major (QK^T)
//   mode 1: D = A * B,   A K-major, B [128 k][128 n] MN-major       (PV, SS)
//   mode 2: as mode 1 but A staged in TMEM via tcgen05.st (TS-MMA)  (PV, TS)
// ----------------------------------------------------------------------------
template <bool kBF16>
__global__ void __launch_bounds__(128, 1)
    umma_selftest_kernel(const __grid_constant__ CUtensorMap tmap_a,
                         const __grid_constant__ CUtensorMap tmap_b, const uint16_t* a_glob,
                         float* d_out, int mode) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const uint32_t sa = smem_u32(smem);
  const uint32_t sb = sa + 32768;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 65536);
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + 65536 + 64);
  const uint32_t warp = warp_id(), lane = lane_id();
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar[0]), 1);
    mbar_init(smem_u32(&bar[1]), 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<256>(smem_u32(tmem_holder));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(smem_u32(&bar[0]), 65536);
    for (int r = 0; r < 2; ++r) {
      tma_load_3d(sa + r * 16384, &tmap_a, smem_u32(&bar[0]), r * 64, 0, 0);
      tma_load_3d(sb + r * 16384, &tmap_b, smem_u32(&bar[0]), r * 64, 0, 0);
    }
  }
  if (mode == 2) {
    // row = thread; A row (128 x 16-bit = 64 x b32) into TMEM cols 128..191
    const int row = int(threadIdx.x);
    const uint32_t* src = reinterpret_cast<const uint32_t*>(a_glob + size_t(row) * 128);
    uint32_t r0[32], r1[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      r0[i] = src[i];
      r1[i] = src[32 + i];
    }
    const uint32_t base = tmem + ((warp * 32u) << 16) + 128;
    tmem_st32(base, r0);
    tmem_st32(base + 32, r1);
    tmem_wait_st();
  }
  mbar_wait(smem_u32(&bar[0]), 0);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t idesc = make_idesc_f16(kBF16, 128, 128, false, mode != 0);
    for (int ks = 0; ks < 8; ++ks) {
      const uint32_t koff = (ks >> 2) * 16384 + (ks & 3) * 32;
      const uint64_t adesc = sdesc_sw128(sa + koff, 16, 1024);
      if (mode == 0) {
        umma_ss(tmem, adesc, sdesc_sw128(sb + koff, 16, 1024), idesc, ks > 0);
      } else if (mode == 1) {
        umma_ss(tmem, adesc, sdesc_sw128(sb + ks * 2048, 16384, 1024), idesc, ks > 0);
      } else {
        umma_ts(tmem, tmem + 128 + ks * 8, sdesc_sw128(sb + ks * 2048, 16384, 1024), idesc,
                ks > 0);
      }
    }
    umma_commit(smem_u32(&bar[1]));
  }
  mbar_wait(smem_u32(&bar[1]), 0);
  tc_fence_after();
  const int row = int(warp * 32 + lane);
  for (int c = 0; c < 4; ++c) {
    uint32_t r[32];
    tmem_ld32(tmem + ((warp * 32u) << 16) + c * 32, r);
    tmem_wait_ld();
    reg_fence(r);
    for (int i = 0; i < 32; ++i) d_out[size_t(row) * 128 + c * 32 + i] = __uint_as_float(r[i]);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<256>(tmem);
}

// exp2 unit under test: mode 0 = ex2_poly2 (the FMA-pipe emulation the
// softmax uses for part of the columns), mode 1 = MUFU ex2.approx.ftz
__global__ void exp2_unit_kernel(const float* __restrict__ x, float* __restrict__ y, int64_t n,
                                 int mode) {
  const int64_t i = 2 * (int64_t(blockIdx.x) * blockDim.x + threadIdx.x);
  if (i >= n) return;
  const float a = x[i], b = i + 1 < n ? x[i + 1] : 0.f;
  float p0, p1;
  if (mode == 0) {
    ex2_poly2(f2(a, b), p0, p1);
  } else {
    p0 = ex2(a);
    p1 = ex2(b);
  }
  y[i] = p0;
  if (i + 1 < n) y[i + 1] = p1;
}

template <int D, bool kBF16, int kBN = kBN128, bool kPair = false>
cudaError_t launch_typed(const FwdLaunch& L) {
  constexpr int kQT = kQTilesFor<D>;
  using C = Cfg<D, kQT, kBN, kPair>;
  auto kern = L.args.trace != nullptr ? sdpa_fwd_kernel<D, kBF16, true, kQT, kBN, kPair>
                                      : sdpa_fwd_kernel<D, kBF16, false, kQT, kBN, kPair>;
  // the dynamic shared-memory opt-in, once per device and instantiation
  // (idempotent: concurrent first calls may both set it)
  static std::atomic<bool> attr_set[64][2] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  const int tr = L.args.trace != nullptr;
  if (dev >= 64 || !attr_set[dev][tr].load(std::memory_order_acquire)) {
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    if (e != cudaSuccess) return e;
    if (dev < 64) attr_set[dev][tr].store(true, std::memory_order_release);
  }
  const int rows_per_cta = kBM * kQT;
  int64_t qblocks = (L.args.seq_len + rows_per_cta - 1) / rows_per_cta;
  if (kPair) qblocks = (qblocks + 1) & ~int64_t(1);  // whole pairs
  const int64_t ctas = qblocks * L.bh;
  if (ctas > 0x7FFFFFFF) return cudaErrorInvalidConfiguration;
  const dim3 grid(static_cast<unsigned int>(ctas), 1u, 1u);
  if constexpr (kPair) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(RolesFor<D, kQT, kBN>::kThreads, 1, 1);
    cfg.dynamicSmemBytes = C::kSmemBytes;
    cfg.stream = static_cast<cudaStream_t>(L.stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, *L.tmap_q, *L.tmap_k, *L.tmap_v, *L.tmap_o, L.args);
  }
  kern<<<grid, RolesFor<D, kQT, kBN>::kThreads, C::kSmemBytes, static_cast<cudaStream_t>(L.stream)>>>(
      *L.tmap_q, *L.tmap_k, *L.tmap_v, *L.tmap_o, L.args);
  return cudaGetLastError();
}

}  // namespace

// 64-key K/V tiles exist for the D=128 split-softmax kernel (TileSchedule
// t_n <= 64, reference tiled.hpp:26-37); every other kernel runs 128 keys
constexpr bool kHasBN64 = kQTilesFor<128> == 2;

// CTA-pair (cta_group::2) D=128 kernel for 128-key tiles without the causal
// mask (TA_PAIR; the pair streams one K/V sequence for both CTAs)
#ifndef TA_PAIR
#define TA_PAIR 0
#endif
constexpr bool kHasPair = TA_PAIR != 0 && kQTilesFor<128> == 2;

bool fwd_use_pair(int64_t D, int block_n, int mask) {
  return kHasPair && D > 64 && D <= 128 && block_n == 128 && mask != kMaskCausal;
}

int fwd_block_n(int64_t D, int t_n) { return kHasBN64 && D > 64 && D <= 128 && t_n <= 64 ? 64 : 128; }

FwdGeometry fwd_geometry(int64_t S, int64_t BH, int64_t D, int block_n) {
  const int qt = D <= 64 ? kQTilesFor<64> : D <= 128 ? kQTilesFor<128> : 1;  // NOLINT
  FwdGeometry g;
  g.block_m = kBM;
  g.block_n = block_n;
  g.q_tiles_per_cta = qt;
  g.threads = D <= 64    ? RolesFor<64, kQTilesFor<64>>::kThreads
              : D <= 128 ? (block_n == 64 ? RolesFor<128, kQTilesFor<128>, 64>::kThreads
                                          : RolesFor<128, kQTilesFor<128>>::kThreads)
                         : RolesFor<256, 1>::kThreads;
  g.ctas = ((S + kBM * qt - 1) / (kBM * qt)) * BH;
  return g;
}

int fwd_ring_slots(int D, int block_n) {
  if (D > 64 && D <= 128 && block_n == 64) return Cfg<128, kQTilesFor<128>, (kHasBN64 ? 64 : 128)>::kSlots;
  return D > 192 ? Cfg<256>::kSlots : D > 128 ? Cfg<192>::kSlots
         : D > 64 ? Cfg<128>::kSlots : Cfg<64>::kSlots;
}

int fwd_kernel_head_dim(int64_t D) { return D <= 64 ? 64 : D <= 128 ? 128 : D <= 192 ? 192 : 256; }

// D=64: persistent CTAs (two per SM) over the (head, query block) items
// (sdpa_d64_sm100.cuh); TA_D64_PERSIST=0 keeps the one-item-per-CTA grid
#ifndef TA_D64_PERSIST
#define TA_D64_PERSIST 0
#endif

template <bool kBF16>
cudaError_t launch_d64_persistent(const FwdLaunch& L) {
  auto kern = L.args.trace != nullptr ? sdpa_d64_persistent_kernel<kBF16, true>
                                      : sdpa_d64_persistent_kernel<kBF16, false>;
  constexpr int kSmem = 2 * Cfg<64, 1>::kTileBytes + Cfg<64, 1>::kSlots * Cfg<64, 1>::kTileBytes +
                        1024 /*barriers*/ + 1024 /*align pad*/;
  static_assert(sizeof(BarriersD64) <= 1024, "barrier block");
  static std::atomic<bool> attr_set[64][2] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  const int tr = L.args.trace != nullptr;
  if (dev >= 64 || !attr_set[dev][tr].load(std::memory_order_acquire)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    if (e != cudaSuccess) return e;
    if (dev < 64) attr_set[dev][tr].store(true, std::memory_order_release);
  }
  int sms = 0;
  cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  const int64_t items = int64_t((L.args.seq_len + kBM - 1) / kBM) * L.bh;
  if (items > 0x7FFFFFFF) return cudaErrorInvalidConfiguration;
  const int64_t slots = int64_t(sms) * Roles<1>::kMinBlocks;
  const unsigned grid = unsigned(items < slots ? items : slots);
  FwdArgs a = L.args;
  a.bh_count = int(L.bh);
  kern<<<grid, Roles<1>::kThreads, kSmem, static_cast<cudaStream_t>(L.stream)>>>(
      *L.tmap_q, *L.tmap_k, *L.tmap_v, *L.tmap_o, a);
  return cudaGetLastError();
}

cudaError_t launch_sdpa_fwd(const FwdLaunch& L) {
  if (L.head_dim == 128) {
    if constexpr (kHasBN64) {
      if (L.block_n == 64)
        return L.bf16 ? launch_typed<128, true, 64>(L) : launch_typed<128, false, 64>(L);
    }
    if constexpr (kHasPair) {
      if (L.pair)
        return L.bf16 ? launch_typed<128, true, 128, true>(L) : launch_typed<128, false, 128, true>(L);
    }
    return L.bf16 ? launch_typed<128, true>(L) : launch_typed<128, false>(L);
  }
  if (L.head_dim == 64) {
#if TA_D64_PERSIST != 0  // (compiled only when selected)
    if constexpr (kQTilesFor<64> == 1 && TA_D64_ROT)
      return L.bf16 ? launch_d64_persistent<true>(L) : launch_d64_persistent<false>(L);
#endif
    return L.bf16 ? launch_typed<64, true>(L) : launch_typed<64, false>(L);
  }
  if (L.head_dim == 192) return L.bf16 ? launch_typed<192, true>(L) : launch_typed<192, false>(L);
  if (L.head_dim == 256) return L.bf16 ? launch_typed<256, true>(L) : launch_typed<256, false>(L);
  return cudaErrorInvalidValue;
}

cudaError_t launch_exp2_unit(const float* x, float* y, int64_t n, int mode, void* stream) {
  const int64_t pairs = (n + 1) / 2;
  const unsigned blocks = unsigned((pairs + 255) / 256);
  if (blocks > 0)
    exp2_unit_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(x, y, n, mode);
  return cudaGetLastError();
}

cudaError_t launch_umma_selftest(const CUtensorMap* ta_map, const CUtensorMap* tb_map,
                                 const void* a_glob, float* d_out, int mode, bool bf16,
                                 void* stream) {
  const int smem = 65536 + 1024 + 1024;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (bf16) {
    cudaFuncSetAttribute(umma_selftest_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         smem);
    umma_selftest_kernel<true><<<1, 128, smem, st>>>(
        *ta_map, *tb_map, static_cast<const uint16_t*>(a_glob), d_out, mode);
  } else {
    cudaFuncSetAttribute(umma_selftest_kernel<false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    umma_selftest_kernel<false><<<1, 128, smem, st>>>(
        *ta_map, *tb_map, static_cast<const uint16_t*>(a_glob), d_out, mode);
  }
  return cudaGetLastError();
}

}  // namespace ta
