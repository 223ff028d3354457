// tileattn_b200.hpp — C++ mirror of the reference entry point over the C-ABI.
//
//   std::vector<float> tileattn_b200::sdpa_tiled(const AttnInput&, const MaskSpec&,
//       const ScaleSpec&, const TileSchedule&, PlanCache&, const TiledOptions& = {});
//
// Same types, argument meaning and error classes as the reference
// (proj/include/tileattn/types.hpp, tiled.hpp:21-88,244-277): the input is a
// borrowed f32-on-the-16-bit-grid tensor, the output is returned by value and
// snapped to the dtype grid (tiled.cpp:216-220); std::invalid_argument for bad
// shapes / masks / scales, UnsupportedScheduleError for bad schedules and for
// what the sm_100a kernel does not cover (F32 / F64 accumulation, D not a
// multiple of 8 or above 256).  Header-only: include it and link
// libtileattn_b200.so.
#pragma once

#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <new>
#include <optional>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "tileattn_b200.h"

namespace tileattn_b200 {

enum class DType { F32, F16Emu, BF16Emu };                  // types.hpp:15
enum class MaskKind { None, Causal, Padding };              // types.hpp:41
enum class TileLayout { RowPacked, ColPacked };             // tiled.hpp:21
enum class AccumMode { F32, F64 };                          // tiled.hpp:244

struct Shape {                                              // types.hpp:27-36
  int64_t b = 1, h = 1, s = 1, d = 1;
  int64_t bh() const { return b * h; }
  int64_t elems() const { return b * h * s * d; }
  bool operator==(const Shape&) const = default;
};

struct MaskSpec {                                           // types.hpp:48-67
  MaskKind kind = MaskKind::None;
  std::vector<int64_t> valid_len;
  static MaskSpec none() { return {}; }
  static MaskSpec causal() { return {MaskKind::Causal, {}}; }
  static MaskSpec padding(std::vector<int64_t> lens) { return {MaskKind::Padding, std::move(lens)}; }
};

struct ScaleSpec {                                          // types.hpp:78-86
  std::optional<double> value;
};

struct AttnInput {                                          // types.hpp:88-104
  Shape shape;
  DType dtype = DType::F32;
  std::vector<float> q, k, v;
};

struct TileSchedule {                                       // tiled.hpp:30-37
  int t_m = 64;
  int t_n = 128;
  int stages = 2;
  TileLayout layout = TileLayout::RowPacked;
  bool operator==(const TileSchedule&) const = default;
};

struct UnsupportedScheduleError : std::runtime_error {      // tiled.hpp:39-41
  using std::runtime_error::runtime_error;
};

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct KernelStats {                                        // tiled.hpp:247-257
  std::atomic<uint64_t> kv_tiles_visited{0};
  std::atomic<uint64_t> peak_scratch_elems{0};  // GPU: 0 (no host scratch)
  int block_m = 0, block_n = 0, stages = 0;     // executed GPU tiling
};

struct TiledOptions {                                       // tiled.hpp:259-263
  int threads = 0;            // accepted, unused: one CUDA launch per call
  AccumMode accum = AccumMode::F32;
  KernelStats* stats = nullptr;
};

inline bool schedule_supported(const TileSchedule& s) {    // tiled.cpp:21-27
  return ta_schedule_supported(ta_schedule{s.t_m, s.t_n, s.stages,
                                           s.layout == TileLayout::ColPacked ? 1 : 0}) != 0;
}

// PlanCache (tiled.hpp:74-86): memo keyed by (t_m, t_n, D, dtype, causal);
// the GPU plan itself lives in the library's process-wide cache, this object
// keeps the reference's per-instance hit / construction accounting.
class PlanCache {
 public:
  void note(const TileSchedule& s, int64_t d, DType dt, bool causal) {
    const auto key = std::make_tuple(s.t_m, s.t_n, d, int(dt), causal);
    std::lock_guard<std::mutex> lock(mu_);
    if (seen_.emplace(key, true).second)
      constructions_.fetch_add(1);
    else
      hits_.fetch_add(1);
  }
  uint64_t hits() const { return hits_.load(); }
  uint64_t constructions() const { return constructions_.load(); }

 private:
  std::mutex mu_;
  std::map<std::tuple<int, int, int64_t, int, bool>, bool> seen_;
  std::atomic<uint64_t> hits_{0}, constructions_{0};
};

namespace detail {

// exact re-encoding of f32 values lying on the 16-bit grid (RNE for safety)
inline uint16_t to_bf16_bits(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return uint16_t(u >> 16);
}

// float -> IEEE half bits, round to nearest even, integer-only (the harness
// converts every element of q/k/v per call, so this sits on the host path)
inline uint16_t to_f16_bits(float f) {
  uint32_t x;
  std::memcpy(&x, &f, 4);
  const uint16_t sign = uint16_t((x >> 16) & 0x8000u);
  const uint32_t a = x & 0x7FFFFFFFu;
  if (a > 0x7F800000u) return uint16_t(sign | 0x7E00u);   // NaN
  if (a >= 0x477FF000u) return uint16_t(sign | 0x7C00u);  // |f| >= 65520 -> inf
  if (a >= 0x38800000u) {  // normal half: rebias the exponent, round 13 bits
    const uint32_t r = a - 0x38000000u;
    return uint16_t(sign | ((r + 0xFFFu + ((r >> 13) & 1u)) >> 13));
  }
  if (a <= 0x33000000u) return sign;  // |f| <= 2^-25 -> 0 (the tie rounds to even)
  // subnormal half: |f| * 2^24 rounded to nearest even (carries into the
  // smallest normal on round-up from 0x3FF)
  const uint32_t e = a >> 23, m = (a & 0x7FFFFFu) | 0x800000u;
  const uint32_t shift = 126u - e;  // 14..24
  const uint32_t q = m >> shift, rem = m & ((1u << shift) - 1u), half = 1u << (shift - 1u);
  return uint16_t(sign | (q + ((rem > half || (rem == half && (q & 1u))) ? 1u : 0u)));
}

inline float from_bits(uint16_t h, DType dt) {
  uint32_t u;
  if (dt == DType::BF16Emu) {
    u = uint32_t(h) << 16;
  } else {
    const uint32_t sign = uint32_t(h & 0x8000u) << 16, ex = (h >> 10) & 0x1Fu, man = h & 0x3FFu;
    if (ex == 31) {
      u = sign | 0x7F800000u | (man << 13);  // inf / NaN
    } else if (ex != 0) {
      u = sign | ((ex + 112u) << 23) | (man << 13);
    } else {
      const float v = float(man) * 0x1.0p-24f;  // subnormal (exact)
      std::memcpy(&u, &v, 4);
      u |= sign;
    }
  }
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

[[noreturn]] inline void raise(ta_status st) {
  const std::string msg = ta_last_error();
  switch (st) {
    case TA_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case TA_ERR_UNSUPPORTED: throw UnsupportedScheduleError(msg);
    case TA_ERR_OOM: throw std::bad_alloc();
    default: throw CudaError(msg);
  }
}

}  // namespace detail

inline double effective_scale(const ScaleSpec& scale, int64_t d) {  // types.cpp:108-116
  double out = 0.0;
  const ta_status st = ta_effective_scale(scale.value ? 1 : 0, scale.value.value_or(0.0), d, &out);
  if (st != TA_OK) detail::raise(st);
  return out;
}

// sdpa_tiled on the B200: validation in the reference order (shape -> mask ->
// schedule -> scale, tiled.cpp:256-259) happens inside the library before any
// device work; the call is synchronous like the reference's.
inline std::vector<float> sdpa_tiled(const AttnInput& input, const MaskSpec& mask,
                                     const ScaleSpec& scale, const TileSchedule& sched,
                                     PlanCache& cache, const TiledOptions& options = {}) {
  const Shape& sh = input.shape;
  const ta_dtype dt = input.dtype == DType::BF16Emu ? TA_BF16
                    : input.dtype == DType::F16Emu  ? TA_F16 : TA_F32;
  const ta_mask_kind mk = mask.kind == MaskKind::Causal  ? TA_MASK_CAUSAL
                        : mask.kind == MaskKind::Padding ? TA_MASK_PADDING : TA_MASK_NONE;
  const ta_schedule ts{sched.t_m, sched.t_n, sched.stages,
                       sched.layout == TileLayout::ColPacked ? 1 : 0};
  if (mk == TA_MASK_PADDING && int64_t(mask.valid_len.size()) != sh.b && sh.b >= 1 &&
      sh.h >= 1 && sh.s >= 1 && sh.d >= 1)
    throw std::invalid_argument("padding mask needs one valid_len per batch");
  const int has_scale = scale.value ? 1 : 0;
  const double scale_v = scale.value.value_or(0.0);
  const int64_t* vl = mk == TA_MASK_PADDING ? mask.valid_len.data() : nullptr;
  ta_status rc = ta_sdpa_check(ta_shape{sh.b, sh.h, sh.s, sh.d}, dt, mk, vl, has_scale, scale_v, ts);
  if (rc != TA_OK) detail::raise(rc);
  if (options.accum == AccumMode::F64)
    throw UnsupportedScheduleError("AccumMode::F64 has no sm_100a tensor-core path");
  const size_t n = size_t(sh.elems());
  if (input.q.size() != n || input.k.size() != n || input.v.size() != n)
    throw std::invalid_argument("q/k/v sizes do not match the shape");
  std::vector<uint16_t> q(n), k(n), v(n), o(n);
  auto conv = dt == TA_BF16 ? detail::to_bf16_bits : detail::to_f16_bits;
  for (size_t i = 0; i < n; ++i) {
    q[i] = conv(input.q[i]);
    k[i] = conv(input.k[i]);
    v[i] = conv(input.v[i]);
  }
  ta_kernel_stats st{};
  rc = ta_sdpa_fwd_host(q.data(), k.data(), v.data(), o.data(), nullptr,
                        ta_shape{sh.b, sh.h, sh.s, sh.d}, dt, mk, vl, has_scale, scale_v, ts,
                        nullptr, &st);
  if (rc != TA_OK) detail::raise(rc);
  cache.note(sched, sh.d, input.dtype, mk == TA_MASK_CAUSAL);
  if (options.stats) {
    options.stats->kv_tiles_visited.fetch_add(st.kv_tiles_visited);
    options.stats->block_m = st.block_m;
    options.stats->block_n = st.block_n;
    options.stats->stages = st.stages;
  }
  std::vector<float> out(n);
  for (size_t i = 0; i < n; ++i) out[i] = detail::from_bits(o[i], input.dtype);
  return out;
}

}  // namespace tileattn_b200
