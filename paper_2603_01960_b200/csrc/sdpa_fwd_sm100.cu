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
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "ptx_sm100.cuh"
#include "sdpa_fwd_sm100.h"

namespace ta {
namespace {

constexpr int kBM = 128;        // rows per Q tile (UMMA M)
constexpr int kBN = 128;        // keys per K/V tile (UMMA N of QK^T, K of PV)
constexpr int kQTiles = 2;      // Q tiles per CTA (ping-pong)
constexpr int kNumSoftmaxWarps = 16;  // 8 per Q tile
constexpr int kThreads = 576;         // 18 warps: 16 softmax + TMA + MMA
// Warp roles.  The SM's warp arbiter favours the highest warp id among
// eligible warps, so the latency-critical single-thread roles (TMA, MMA
// issue) take the top ids and are never starved by the softmax stream.
// 576 threads leave 112 registers per thread for every warp (no setmaxnreg).
constexpr int kWarpTma = 16;  // also allocates / frees TMEM
constexpr int kWarpMma = 17;
constexpr uint32_t kTmemCols = 512;
constexpr float kLn2 = 0.69314718055994530942f;
// lazy rescale threshold in log2 units: exps may reach 2^8 before O is
// rescaled (fp32 accumulators, 16-bit P: both fine).
constexpr float kRescaleThreshold = 8.0f;
// exp2 work split: of every 4 column pairs a thread holds per row, kEmuPer4
// pairs use the FMA-pipe polynomial (ex2_poly2) and the rest the MUFU
// (measured 16 exp2/clk/SM).
#ifndef TA_EMU_PER4
#define TA_EMU_PER4 1
#endif
constexpr int kEmuPer4 = TA_EMU_PER4;
// P is handed to the PV MMAs in two halves of 64 keys.
constexpr int kPParts = 2;

template <int D>
struct Cfg {
  static constexpr int kRegions = D / 64;                   // 128-B swizzle atoms along D
  static constexpr int kTileBytes = kBM * D * 2;            // one Q / K / V tile
  static constexpr int kRegionBytes = kBM * 128;            // 128 rows x 128 B
  static constexpr int kSlots = D == 128 ? 4 : 8;           // K/V ring depth
  static constexpr int kSmemData = kQTiles * kTileBytes + kSlots * kTileBytes;
  static constexpr int kSmemBytes = kSmemData + 3072 /*barriers+epilogue*/ + 1024 /*align*/;
  static constexpr uint32_t kTmemS = 0;      // S0 at col 0, S1 at col 128 (fp32)
  static constexpr uint32_t kTmemO = 256;    // O0 at 256, O1 at 256 + D (fp32)
};

struct Barriers {
  uint64_t q_full;
  uint64_t s_full[kQTiles];
  uint64_t p_full[kQTiles][2];  // P key columns [64h, 64h+64) written (8 warp arrivals)
  uint64_t o_full[kQTiles];
  uint64_t slot_full[8];
  uint64_t slot_empty[8];
  uint32_t tmem_base;
  alignas(16) float row_l[kQTiles][128];  // epilogue: per-row normaliser
  alignas(16) float row_m[kQTiles][128];  // epilogue: per-row running max (log2 units)
};
static_assert(sizeof(Barriers) <= 3072, "barrier area overflows its smem budget");

template <int D, bool kBF16>
__global__ void __launch_bounds__(kThreads, 1)
    sdpa_fwd_kernel(const __grid_constant__ CUtensorMap tmap_q,
                    const __grid_constant__ CUtensorMap tmap_k,
                    const __grid_constant__ CUtensorMap tmap_v, FwdArgs args) {
  using C = Cfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const uint32_t sq = smem_u32(smem);                          // Q tiles
  const uint32_t sring = sq + kQTiles * C::kTileBytes;         // K/V ring
  Barriers* bars = reinterpret_cast<Barriers*>(smem + C::kSmemData);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const int S = args.seq_len;
  const int bh = blockIdx.y;
  const int q0 = blockIdx.x * (kBM * kQTiles);
  const int n_kv = (S + kBN - 1) / kBN;
  long long* const trace =
      (args.trace != nullptr && blockIdx.x == 0 && blockIdx.y == 0) ? args.trace : nullptr;
  auto rec = [&](int ev, int j) {
    if (trace != nullptr && j < kTraceIters) trace[ev * kTraceIters + j] = clock64();
  };

  if (threadIdx.x == kWarpMma * 32) {
    mbar_init(smem_u32(&bars->q_full), 1);
    for (int t = 0; t < kQTiles; ++t) {
      mbar_init(smem_u32(&bars->s_full[t]), 1);
      mbar_init(smem_u32(&bars->p_full[t][0]), 8);  // one arrive per softmax warp of the tile
      mbar_init(smem_u32(&bars->p_full[t][1]), 8);
      mbar_init(smem_u32(&bars->o_full[t]), 1);
    }
    for (int s = 0; s < C::kSlots; ++s) {
      mbar_init(smem_u32(&bars->slot_full[s]), 1);
      mbar_init(smem_u32(&bars->slot_empty[s]), 1);
    }
    fence_barrier_init();
  }
  if (warp == kWarpTma) tmem_alloc<kTmemCols>(smem_u32(&bars->tmem_base));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  if (warp == kWarpTma) {
    // ------------------------------------------------------------------ TMA
    if (lane == 0) {
      tma_prefetch_desc(&tmap_q);
      tma_prefetch_desc(&tmap_k);
      tma_prefetch_desc(&tmap_v);
      const uint32_t qbar = smem_u32(&bars->q_full);
      mbar_arrive_expect_tx(qbar, kQTiles * C::kTileBytes);
      for (int t = 0; t < kQTiles; ++t)
        for (int r = 0; r < C::kRegions; ++r)
          tma_load_3d(sq + t * C::kTileBytes + r * C::kRegionBytes, &tmap_q, qbar, r * 64,
                      q0 + t * kBM, bh);
      int slot = 0;
      uint32_t phase = 0;
      for (int j = 0; j < n_kv; ++j) {
        for (int kv = 0; kv < 2; ++kv) {
          mbar_wait(smem_u32(&bars->slot_empty[slot]), phase ^ 1);
          const uint32_t fbar = smem_u32(&bars->slot_full[slot]);
          mbar_arrive_expect_tx(fbar, C::kTileBytes);
          const CUtensorMap* map = kv == 0 ? &tmap_k : &tmap_v;
          for (int r = 0; r < C::kRegions; ++r)
            tma_load_3d(sring + slot * C::kTileBytes + r * C::kRegionBytes, map, fbar, r * 64,
                        j * kBN, bh);
          if (++slot == C::kSlots) {
            slot = 0;
            phase ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == kWarpMma) {
    // ------------------------------------------------------------------ MMA
    // The whole warp runs this loop (uniform control flow, descriptors in
    // uniform registers); one elected lane issues each tcgen05 instruction.
    // Order per K/V step j: PV0(j-1), S0(j), PV1(j-1), S1(j) — the tensor core
    // alternates between the Q tiles while the other tile's softmax runs.
    constexpr uint32_t idesc_qk = make_idesc_f16(kBF16, kBM, kBN, false, false);
    constexpr uint32_t idesc_pv = make_idesc_f16(kBF16, kBM, D, false, true);
    // ring position r (K_j at 2j, V_j at 2j+1) -> slot / phase
    auto slot_of = [](int r) { return r % C::kSlots; };
    auto phase_of = [](int r) { return uint32_t((r / C::kSlots) & 1); };
    auto wait_full = [&](int r) {
      mbar_wait(smem_u32(&bars->slot_full[slot_of(r)]), phase_of(r));
      tc_fence_after();
    };
    auto release = [&](int r) { umma_commit_warp(smem_u32(&bars->slot_empty[slot_of(r)])); };
    // descriptors: base built once, K-step offsets added to the start-address
    // field (addr >> 4; smem addresses < 256 KB never carry out of 14 bits)
    const uint64_t qdesc = sdesc_sw128(sq, 16, 1024);
    const uint64_t kvdesc_k = sdesc_sw128(sring, 16, 1024);
    const uint64_t kvdesc_v = sdesc_sw128(sring, C::kRegionBytes, 1024);
    auto issue_qk = [&](int t, int r) {
      uint64_t qd = qdesc + uint64_t((t * C::kTileBytes) >> 4);
      uint64_t kd = kvdesc_k + uint64_t((slot_of(r) * C::kTileBytes) >> 4);
      // opaque to the optimiser: stops 2 x 8 per-K-step descriptors being
      // hoisted out of the K/V loop into (spilled) registers
      asm volatile("" : "+l"(qd), "+l"(kd));
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks) {
        const uint32_t off = ((ks >> 2) * C::kRegionBytes + (ks & 3) * 32) >> 4;
        umma_ss_warp(tmem + C::kTmemS + t * kBN, qd + off, kd + off, idesc_qk, ks > 0);
      }
      umma_commit_warp(smem_u32(&bars->s_full[t]));
    };
    // PV in two halves of 64 keys, each issued as soon as all 8 softmax warps
    // of the tile have written that half of P (P aliases S in TMEM).
    auto issue_pv = [&](int t, int r, bool accumulate, int j) {
      uint64_t vd = kvdesc_v + uint64_t((slot_of(r) * C::kTileBytes) >> 4);
      asm volatile("" : "+l"(vd));
#pragma unroll
      for (int h = 0; h < kPParts; ++h) {
        mbar_wait(smem_u32(&bars->p_full[t][h]), uint32_t(j & 1));
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < kBN / 16 / kPParts; ++kk) {
          const int ks = h * (kBN / 16 / kPParts) + kk;
          umma_ts_warp(tmem + C::kTmemO + t * D, tmem + C::kTmemS + t * kBN + ks * 8,
                       vd + uint64_t((ks * 16 * 128) >> 4), idesc_pv,
                       (accumulate || ks > 0) ? 1u : 0u);
        }
      }
      umma_commit_warp(smem_u32(&bars->o_full[t]));
    };

    mbar_wait(smem_u32(&bars->q_full), 0);
    tc_fence_after();
    wait_full(0);
    issue_qk(0, 0);
    issue_qk(1, 0);
    release(0);
    for (int j = 1; j < n_kv; ++j) {
      const int rk = 2 * j, rv = 2 * j - 1;
      wait_full(rv);
      if (lane == 0) rec(kEvMmaWaitP0, j);
      issue_pv(0, rv, j > 1, j - 1);
      wait_full(rk);
      issue_qk(0, rk);
      if (lane == 0) rec(kEvMmaIssuedPV0, j);
      if (lane == 0) rec(kEvMmaWaitP1, j);
      issue_pv(1, rv, j > 1, j - 1);
      release(rv);
      issue_qk(1, rk);
      release(rk);
      if (lane == 0) rec(kEvMmaIssuedPV1, j);
    }
    const int rv = 2 * n_kv - 1;
    wait_full(rv);
    issue_pv(0, rv, n_kv > 1, n_kv - 1);
    issue_pv(1, rv, n_kv > 1, n_kv - 1);
    release(rv);
  } else {
    // -------------------------------------------------------------- softmax
    // 8 warps per Q tile.  Warp w works on TMEM lane quadrant q = w % 4 (the
    // only lanes it may access) and, within it, the 16 rows of row-half
    // rh = (w / 4) % 2.  With the 16x256b TMEM shape each thread holds two
    // rows (r, r + 8) x 32 columns (16 adjacent pairs), so a row's max / sum
    // is reduced over the 4 threads sharing it with two xor-shuffles.
    const int t = int(warp) / 8;
    const int wq = int(warp) & 3;
    const int rh = (int(warp) >> 2) & 1;
    const int t0 = int(lane) & 3;             // column-pair slot within a 256-bit chunk
    const int r_lo = wq * 32 + rh * 16 + int(lane >> 2);  // my rows: r_lo, r_lo + 8
    const uint32_t lane_base = uint32_t(wq * 32 + rh * 16) << 16;
    const uint32_t tS = tmem + lane_base + C::kTmemS + t * kBN;
    const uint32_t tO = tmem + lane_base + C::kTmemO + t * D;
    const float sl2 = args.scale_log2;
    const uint32_t sbar = smem_u32(&bars->s_full[t]);
    const uint32_t obar = smem_u32(&bars->o_full[t]);
    const uint64_t sl2x2 = f2(sl2, sl2);
    const bool tr = (warp == 0 || warp == 8) && lane == 0;

    float m_run[2] = {-INFINITY, -INFINITY};  // running max per row (scaled, log2 units)
    float l_run[2] = {0.f, 0.f};              // my partial normaliser per row

    for (int j = 0; j < n_kv; ++j) {
      mbar_wait(sbar, uint32_t(j & 1));
      tc_fence_after();
      if (tr) rec(kEvSm0SReady + 5 * t, j);
      uint32_t sr[64];
      tmem_ld_16x256b_x16(tS, sr);
      tmem_wait_ld();
      reg_fence(sr);
      if (tr) rec(kEvSm0Loaded + 5 * t, j);
      // sv[row][c][k]: row lo/hi, chunk c, column 8c + 2*t0 + k
      float sv[2][16][2];
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        sv[0][c][0] = __uint_as_float(sr[4 * c + 0]);
        sv[0][c][1] = __uint_as_float(sr[4 * c + 1]);
        sv[1][c][0] = __uint_as_float(sr[4 * c + 2]);
        sv[1][c][1] = __uint_as_float(sr[4 * c + 3]);
      }
      if (j == n_kv - 1) {
        const int valid = S - j * kBN;  // keys past S were zero-filled by TMA
        if (valid < kBN) {
#pragma unroll
          for (int c = 0; c < 16; ++c)
#pragma unroll
            for (int k = 0; k < 2; ++k)
              if (8 * c + 2 * t0 + k >= valid) {
                sv[0][c][k] = -INFINITY;
                sv[1][c][k] = -INFINITY;
              }
        }
      }
      // row max: 32 local values per row, then across the 4 threads of the row
      float mx[2];
#pragma unroll
      for (int rr = 0; rr < 2; ++rr) {
        float a = fmaxf(sv[rr][0][0], sv[rr][0][1]), b = fmaxf(sv[rr][1][0], sv[rr][1][1]);
#pragma unroll
        for (int c = 2; c < 16; c += 2) {
          a = fmaxf(a, fmaxf(sv[rr][c][0], sv[rr][c][1]));
          b = fmaxf(b, fmaxf(sv[rr][c + 1][0], sv[rr][c + 1][1]));
        }
        mx[rr] = fmaxf(a, b);
      }
#pragma unroll
      for (int rr = 0; rr < 2; ++rr) {
        mx[rr] = fmaxf(mx[rr], __shfl_xor_sync(0xffffffffu, mx[rr], 1));
        mx[rr] = fmaxf(mx[rr], __shfl_xor_sync(0xffffffffu, mx[rr], 2));
      }
      if (tr) rec(kEvSm0Max + 5 * t, j);
      float alpha[2];
      bool need_any = false;
#pragma unroll
      for (int rr = 0; rr < 2; ++rr) {
        const float m_new = mx[rr] * sl2;
        const bool need = m_new > m_run[rr] + kRescaleThreshold;
        alpha[rr] = need ? ex2(m_run[rr] - m_new) : 1.f;  // 0 on the first tile
        if (need) {
          l_run[rr] *= alpha[rr];
          m_run[rr] = m_new;
        }
        need_any |= need;
      }
      if (j > 0 && __any_sync(0xffffffffu, need_any)) {
        // O correction (rare with the lazy threshold): wait until PV(j-1) has
        // landed in TMEM and rescale my two rows in place; PV(j) is not issued
        // before every softmax warp of the tile signals the first half of P(j).
        mbar_wait(obar, uint32_t((j - 1) & 1));
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < D / 32; ++c) {
          uint32_t orow[16];
          tmem_ld_16x256b_x4(tO + c * 32, orow);
          tmem_wait_ld();
          reg_fence(orow);
#pragma unroll
          for (int i = 0; i < 16; ++i)
            orow[i] = __float_as_uint(__uint_as_float(orow[i]) * alpha[(i >> 1) & 1]);
          tmem_st_16x256b_x4(tO + c * 32, orow);
        }
      }
      const uint64_t negm[2] = {f2(m_run[0] == -INFINITY ? 0.f : -m_run[0],
                                   m_run[0] == -INFINITY ? 0.f : -m_run[0]),
                                f2(m_run[1] == -INFINITY ? 0.f : -m_run[1],
                                   m_run[1] == -INFINITY ? 0.f : -m_run[1])};
      uint64_t acc[2] = {0ull, 0ull};
#pragma unroll
      for (int h = 0; h < kPParts; ++h) {
        // P words for the 16x128b store: pk[2*cc] = row lo, pk[2*cc+1] = row hi
        uint32_t pk[16];
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) {
          const int c = h * 8 + cc;
#pragma unroll
          for (int rr = 0; rr < 2; ++rr) {
            const uint64_t x = ffma2(f2(sv[rr][c][0], sv[rr][c][1]), sl2x2, negm[rr]);
            float p0, p1;
#ifdef TA_DEBUG_NO_EXP  // timing ablation only: wrong results
            f2_split(x, p0, p1);
#else
            if ((c & 3) < kEmuPer4) {
              ex2_poly2(x, p0, p1);
            } else {
              float a, b;
              f2_split(x, a, b);
              p0 = ex2(a);
              p1 = ex2(b);
            }
#endif
            acc[rr] = fadd2(acc[rr], f2(p0, p1));
            pk[2 * cc + rr] = pack2<kBF16>(p0, p1);
          }
        }
        tmem_st_16x128b_x8(tS + h * 32, pk);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&bars->p_full[t][h]));
        if (h == 0 && tr) rec(kEvSm0Exp + 5 * t, j);
      }
#pragma unroll
      for (int rr = 0; rr < 2; ++rr) {
        float lo, hi;
        f2_split(acc[rr], lo, hi);
        l_run[rr] += lo + hi;
      }
      if (tr) rec(kEvSm0PArrive + 5 * t, j);
    }

    // ------------------------------------------------------------- epilogue
    // full row sums; one thread per row publishes l and m for the
    // 32x32b-shaped epilogue (thread == row, warp pair splits the columns).
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      l_run[rr] += __shfl_xor_sync(0xffffffffu, l_run[rr], 1);
      l_run[rr] += __shfl_xor_sync(0xffffffffu, l_run[rr], 2);
    }
    if (t0 == 0) {
      bars->row_l[t][r_lo] = l_run[0];
      bars->row_l[t][r_lo + 8] = l_run[1];
      bars->row_m[t][r_lo] = m_run[0];
      bars->row_m[t][r_lo + 8] = m_run[1];
    }
    named_bar_sync(1 + t * 4 + wq, 64);  // the quadrant's two row-half warps
    const int row = wq * 32 + int(lane);
    const float l = bars->row_l[t][row];
    const float m = bars->row_m[t][row];
    mbar_wait(obar, uint32_t((n_kv - 1) & 1));
    tc_fence_after();
    constexpr int kDh = D / 2;  // my O columns: [rh * kDh, rh * kDh + kDh)
    const uint32_t tO32 = tmem + (uint32_t(wq * 32) << 16) + C::kTmemO + t * D + rh * kDh;
    const int grow = q0 + t * kBM + row;
    const float inv_l = l > 0.f ? 1.f / l : 0.f;
    uint16_t* orow_g =
        reinterpret_cast<uint16_t*>(args.o) + (size_t(bh) * S + grow) * D + rh * kDh;
#pragma unroll
    for (int c = 0; c < kDh / 32; ++c) {
      uint32_t orow[32];
      tmem_ld32(tO32 + c * 32, orow);
      tmem_wait_ld();
      reg_fence(orow);
      uint32_t packed[16];
#pragma unroll
      for (int i = 0; i < 16; ++i)
        packed[i] = pack2<kBF16>(__uint_as_float(orow[2 * i]) * inv_l,
                                 __uint_as_float(orow[2 * i + 1]) * inv_l);
      if (grow < S) {
        uint4* dst = reinterpret_cast<uint4*>(orow_g + c * 32);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          dst[i] = make_uint4(packed[4 * i], packed[4 * i + 1], packed[4 * i + 2],
                              packed[4 * i + 3]);
      }
    }
    if (rh == 0 && args.lse != nullptr && grow < S)
      args.lse[size_t(bh) * S + grow] = l > 0.f ? (m + __log2f(l)) * kLn2 : -INFINITY;
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == kWarpTma) tmem_dealloc<kTmemCols>(tmem);
}

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

template <int D, bool kBF16>
cudaError_t launch_typed(const FwdLaunch& L) {
  using C = Cfg<D>;
  auto kern = sdpa_fwd_kernel<D, kBF16>;
  static bool attr_set[64] = {};  // per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !attr_set[dev]) {
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    if (e != cudaSuccess) return e;
    attr_set[dev] = true;
  }
  const int rows_per_cta = kBM * kQTiles;
  dim3 grid((L.args.seq_len + rows_per_cta - 1) / rows_per_cta, L.bh);
  kern<<<grid, kThreads, C::kSmemBytes, static_cast<cudaStream_t>(L.stream)>>>(
      *L.tmap_q, *L.tmap_k, *L.tmap_v, L.args);
  return cudaGetLastError();
}

}  // namespace

FwdGeometry fwd_geometry(int64_t S, int64_t BH) {
  FwdGeometry g;
  g.block_m = kBM;
  g.block_n = kBN;
  g.q_tiles_per_cta = kQTiles;
  g.threads = kThreads;
  g.ctas = ((S + kBM * kQTiles - 1) / (kBM * kQTiles)) * BH;
  return g;
}

int fwd_ring_slots(int D) { return D == 128 ? Cfg<128>::kSlots : Cfg<64>::kSlots; }

cudaError_t launch_sdpa_fwd(const FwdLaunch& L) {
  if (L.head_dim == 128) return L.bf16 ? launch_typed<128, true>(L) : launch_typed<128, false>(L);
  if (L.head_dim == 64) return L.bf16 ? launch_typed<64, true>(L) : launch_typed<64, false>(L);
  return cudaErrorInvalidValue;
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
