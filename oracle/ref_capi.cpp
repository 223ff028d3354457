// TEST INFRASTRUCTURE ONLY — extern "C" shim over the UNMODIFIED reference
// sources (/root/reference/proj/src/{types,reference,tiled}.cpp), compiled by
// oracle/Makefile into oracle/_ref/libtileattn_ref*.so.  Used (a) to pin the
// oracle restatement in oracle/oracle.c, (b) to generate tests/golden/, and
// (c) as bench.py's CPU baseline ("kind": "reference") and `--impl reference`
// arm.  The product library never links it.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <vector>

#include "tileattn/reference.hpp"
#include "tileattn/tiled.hpp"
#include "tileattn/types.hpp"

using namespace tileattn;

namespace {

thread_local char g_err[512];

int fail(const std::exception& e, int code) {
  std::strncpy(g_err, e.what(), sizeof(g_err) - 1);
  return code;
}

DType to_dtype(int d) {
  return d == 1 ? DType::F16Emu : d == 2 ? DType::BF16Emu : DType::F32;
}

MaskSpec to_mask(int kind, const int64_t* valid_len, int64_t b) {
  if (kind == 1) return MaskSpec::causal();
  if (kind == 2) return MaskSpec::padding(std::vector<int64_t>(valid_len, valid_len + b));
  return MaskSpec::none();
}

AttnInput wrap(const float* q, const float* k, const float* v, int64_t B, int64_t H, int64_t S,
               int64_t D, int dtype) {
  AttnInput in;
  in.shape = Shape{B, H, S, D};
  in.dtype = to_dtype(dtype);
  const size_t n = size_t(B * H * S * D);
  in.q.assign(q, q + n);
  in.k.assign(k, k + n);
  in.v.assign(v, v + n);
  return in;
}

}  // namespace

extern "C" {

__attribute__((visibility("default"))) const char* ref_last_error() { return g_err; }

// types.cpp:151-164
__attribute__((visibility("default"))) int ref_make_input(int64_t B, int64_t H, int64_t S,
                                                          int64_t D, int dtype, uint64_t seed,
                                                          float* q, float* k, float* v) {
  try {
    AttnInput in = make_input(Shape{B, H, S, D}, to_dtype(dtype), seed);
    std::memcpy(q, in.q.data(), in.q.size() * 4);
    std::memcpy(k, in.k.data(), in.k.size() * 4);
    std::memcpy(v, in.v.data(), in.v.size() * 4);
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(e, 1);
  }
}

// types.cpp:52-78
__attribute__((visibility("default"))) float ref_snap(float v, int dtype) {
  return snap_to_dtype(v, to_dtype(dtype));
}

// types.cpp:108-116; returns NaN and sets the error on invalid_argument.
__attribute__((visibility("default"))) double ref_effective_scale(int has_value, double value,
                                                                  int64_t d) {
  try {
    ScaleSpec s;
    if (has_value) s.value = value;
    return effective_scale(s, d);
  } catch (const std::invalid_argument& e) {
    fail(e, 1);
    return std::nan("");
  }
}

// reference.cpp:8-55 (o in double, row_sums)
__attribute__((visibility("default"))) int ref_sdpa_reference(
    const float* q, const float* k, const float* v, int64_t B, int64_t H, int64_t S, int64_t D,
    int dtype, int has_scale, double scale, int mask_kind, const int64_t* valid_len, double* o,
    double* row_sums) {
  try {
    AttnInput in = wrap(q, k, v, B, H, S, D, dtype);
    ScaleSpec sc;
    if (has_scale) sc.value = scale;
    RefOutput r = sdpa_reference(in, to_mask(mask_kind, valid_len, B), sc);
    std::memcpy(o, r.o.data(), r.o.size() * 8);
    std::memcpy(row_sums, r.row_sums.data(), r.row_sums.size() * 8);
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(e, 1);
  }
}

// tiled.cpp:253-272 — the reference CPU hot path itself.
// layout 0 = RowPacked, 1 = ColPacked; accum 0 = F32, 1 = F64.
// Returns 0 ok, 1 invalid_argument, 2 UnsupportedScheduleError.
__attribute__((visibility("default"))) int ref_sdpa_tiled(
    const float* q, const float* k, const float* v, int64_t B, int64_t H, int64_t S, int64_t D,
    int dtype, int has_scale, double scale, int mask_kind, const int64_t* valid_len, int t_m,
    int t_n, int stages, int layout, int threads, int accum, float* out,
    uint64_t* kv_tiles_visited) {
  try {
    AttnInput in = wrap(q, k, v, B, H, S, D, dtype);
    ScaleSpec sc;
    if (has_scale) sc.value = scale;
    TileSchedule sched{t_m, t_n, stages,
                       layout == 1 ? TileLayout::ColPacked : TileLayout::RowPacked};
    PlanCache cache;
    KernelStats stats;
    TiledOptions opt;
    opt.threads = threads;
    opt.accum = accum == 1 ? AccumMode::F64 : AccumMode::F32;
    opt.stats = &stats;
    std::vector<float> o = sdpa_tiled(in, to_mask(mask_kind, valid_len, B), sc, sched, cache, opt);
    std::memcpy(out, o.data(), o.size() * 4);
    if (kv_tiles_visited) *kv_tiles_visited = stats.kv_tiles_visited.load();
    return 0;
  } catch (const UnsupportedScheduleError& e) {
    return fail(e, 2);
  } catch (const std::invalid_argument& e) {
    return fail(e, 1);
  }
}

// Timing entry for the CPU baseline: the input is built once by the caller
// (already an AttnInput-shaped f32 copy), so only sdpa_tiled is timed.
struct RefHandle {
  AttnInput in;
  PlanCache cache;
};

__attribute__((visibility("default"))) void* ref_handle_new(const float* q, const float* k,
                                                            const float* v, int64_t B, int64_t H,
                                                            int64_t S, int64_t D, int dtype) {
  auto* h = new RefHandle;
  h->in = wrap(q, k, v, B, H, S, D, dtype);
  return h;
}

__attribute__((visibility("default"))) void ref_handle_free(void* h) {
  delete static_cast<RefHandle*>(h);
}

__attribute__((visibility("default"))) int ref_handle_run(void* hv, int t_m, int t_n,
                                                          int stages, int layout, int threads,
                                                          float* out_first /*nullable*/) {
  auto* h = static_cast<RefHandle*>(hv);
  try {
    TileSchedule sched{t_m, t_n, stages,
                       layout == 1 ? TileLayout::ColPacked : TileLayout::RowPacked};
    TiledOptions opt;
    opt.threads = threads;
    std::vector<float> o = sdpa_tiled(h->in, MaskSpec::none(), ScaleSpec{}, sched, h->cache, opt);
    if (out_first) *out_first = o[0];
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 2);
  }
}

// LSE via the reference's own header-only primitives (tiled.hpp:149-221):
// drive score_tile<double> + online_update<double> over t_n-wide K/V tiles
// exactly as run_tiled does (tiled.cpp:185-214, no mask), read st.m / st.l
// before finalize, LSE = m + ln(l). Heads [bh_begin, bh_end).
__attribute__((visibility("default"))) int ref_lse_via_primitives(
    const float* q, const float* k, const float* v, int64_t B, int64_t H, int64_t S, int64_t D,
    int has_scale, double scale, int t_n, int64_t bh_begin, int64_t bh_end, double* lse) {
  try {
    ScaleSpec sc;
    if (has_scale) sc.value = scale;
    const double s = effective_scale(sc, D);
    (void)B;
    (void)H;
    std::vector<double> scores(static_cast<size_t>(t_n));
    for (int64_t bh = bh_begin; bh < bh_end; ++bh) {
      for (int64_t i = 0; i < S; ++i) {
        SoftmaxState<double> st;
        st.reset(1, D);
        const float* qi = q + (bh * S + i) * D;
        for (int64_t c0 = 0; c0 < S; c0 += t_n) {
          const int cols = int(std::min<int64_t>(t_n, S - c0));
          const float* kt = k + (bh * S + c0) * D;
          const float* vt = v + (bh * S + c0) * D;
          score_tile<double>(qi, 1, D, kt, cols, TileLayout::RowPacked, s, scores.data());
          online_update<double>(st, scores.data(), cols, vt);
        }
        lse[bh * S + i] = st.l[0] == 0.0 ? -INFINITY : st.m[0] + std::log(st.l[0]);
      }
    }
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(e, 1);
  }
}

// Reference's fast_expf (tiled.hpp:98-113), exposed for the exp2-emulation KAT.
__attribute__((visibility("default"))) float ref_fast_expf(float x) { return fast_expf(x); }

}  // extern "C"
