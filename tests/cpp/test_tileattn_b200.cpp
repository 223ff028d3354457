// C++ parity tests of tileattn_b200::sdpa_tiled (include/tileattn_b200.hpp),
// written the way the reference's own tests are (proj/tests/test_tiled.cpp,
// test_reference.cpp): same cases, same tolerances, against the oracle
// (oracle/oracle.c, a restatement of reference.cpp:8-55; test infrastructure).
//
//   built and run by tests/test_cpp_api.py:  ./test_tileattn_b200 [--cpu-only]
// --cpu-only runs the cases that need no GPU (validation / error classes).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "tileattn_b200.hpp"

extern "C" {
void oracle_make_input(int64_t n, int dtype, uint64_t seed, float* q, float* k, float* v);
int oracle_sdpa_reference(const float* q, const float* k, const float* v, int64_t B, int64_t H,
                          int64_t S, int64_t D, double scale, int mask_kind,
                          const int64_t* valid_len, int64_t bh_begin, int64_t bh_end, double* o,
                          double* row_sums, double* row_max, double* lse);
}

using namespace tileattn_b200;

static int g_checks = 0, g_failures = 0;
#define CHECK(cond)                                                                   \
  do {                                                                                \
    ++g_checks;                                                                       \
    if (!(cond)) {                                                                    \
      ++g_failures;                                                                   \
      std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #cond);  \
    }                                                                                 \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                       \
  do {                                                    \
    bool thrown = false;                                  \
    try {                                                 \
      (void)(expr);                                       \
    } catch (const type&) {                               \
      thrown = true;                                      \
    } catch (...) {                                       \
    }                                                     \
    ++g_checks;                                           \
    if (!thrown) {                                        \
      ++g_failures;                                       \
      std::fprintf(stderr, "%s:%d: expected %s from %s\n", __FILE__, __LINE__, #type, #expr); \
    }                                                     \
  } while (0)

static int dtype_code(DType dt) { return dt == DType::F16Emu ? 1 : dt == DType::BF16Emu ? 2 : 0; }

static AttnInput make_input(const Shape& sh, DType dt, uint64_t seed) {  // types.cpp:151-164
  AttnInput in;
  in.shape = sh;
  in.dtype = dt;
  const size_t n = size_t(sh.elems());
  in.q.resize(n);
  in.k.resize(n);
  in.v.resize(n);
  oracle_make_input(int64_t(n), dtype_code(dt), seed, in.q.data(), in.k.data(), in.v.data());
  return in;
}

static std::vector<double> oracle_o(const AttnInput& in, const MaskSpec& m, double scale = 0) {
  const Shape& sh = in.shape;
  std::vector<double> o(size_t(sh.elems())), rs(size_t(sh.bh() * sh.s)), rm(rs.size()),
      lse(rs.size());
  const int mk = m.kind == MaskKind::Causal ? 1 : m.kind == MaskKind::Padding ? 2 : 0;
  const double sc = scale > 0 ? scale : 1.0 / std::sqrt(double(sh.d));
  oracle_sdpa_reference(in.q.data(), in.k.data(), in.v.data(), sh.b, sh.h, sh.s, sh.d, sc, mk,
                        m.valid_len.data(), 0, sh.bh(), o.data(), rs.data(), rm.data(),
                        lse.data());
  return o;
}

static double max_abs_diff(const std::vector<float>& got, const std::vector<double>& want) {
  double m = 0.0;
  for (size_t i = 0; i < got.size(); ++i) {
    const double d = std::abs(double(got[i]) - want[i]);
    if (std::isnan(d)) return INFINITY;  // NaN fails loudly (bench.cpp:79-84)
    m = std::max(m, d);
  }
  return m;
}

static double dtype_tol(DType dt) {  // bench.cpp:56-63
  return dt == DType::F16Emu ? 5e-3 : dt == DType::BF16Emu ? 2e-2 : 1e-4;
}

// ---------------------------------------------------------------- CPU cases
static void test_unsupported_schedules_are_rejected() {  // test_tiled.cpp:256-271
  CHECK(schedule_supported(TileSchedule{64, 128, 2, TileLayout::RowPacked}));
  CHECK(!schedule_supported(TileSchedule{48, 128, 2, TileLayout::RowPacked}));
  CHECK(!schedule_supported(TileSchedule{64, 512, 2, TileLayout::RowPacked}));
  CHECK(!schedule_supported(TileSchedule{64, 128, 0, TileLayout::RowPacked}));
  CHECK(!schedule_supported(TileSchedule{64, 128, 5, TileLayout::RowPacked}));
  PlanCache cache;
  const AttnInput in = make_input(Shape{1, 1, 32, 64}, DType::BF16Emu, 1);
  CHECK_THROWS_AS(sdpa_tiled(in, MaskSpec::none(), ScaleSpec{},
                             TileSchedule{64, 64, 7, TileLayout::RowPacked}, cache),
                  UnsupportedScheduleError);
  CHECK(cache.constructions() == 0);
}

// the host conversions the mirror applies to every element (harness inputs
// are float): bit-exact round-to-nearest-even against a frexp/nearbyint
// restatement on a strided sweep of every float bit pattern, and every half
// round-trips through from_bits
static uint16_t f16_bits_slow(float f) {
  uint32_t x;
  std::memcpy(&x, &f, 4);
  const uint16_t sign = uint16_t((x >> 16) & 0x8000u);
  const float a = std::fabs(f);
  if (std::isnan(f)) return uint16_t(sign | 0x7E00u);
  if (a >= 65520.0f) return uint16_t(sign | 0x7C00u);
  if (a < 0x1.0p-14f) return uint16_t(sign | uint16_t(std::nearbyint(double(a) * 0x1.0p24)));
  int e;
  double m = std::nearbyint(std::frexp(double(a), &e) * 2048.0);
  if (m >= 2048.0) {
    m /= 2.0;
    ++e;
  }
  return uint16_t(sign | uint16_t((e + 14) << 10) | (uint16_t(m) & 0x3FFu));
}

static void test_host_f16_conversions() {
  int bad = 0;
  for (uint64_t i = 0; i < (uint64_t(1) << 32); i += 4093) {
    const uint32_t u = uint32_t(i);
    float f;
    std::memcpy(&f, &u, 4);
    bad += tileattn_b200::detail::to_f16_bits(f) != f16_bits_slow(f);
  }
  for (uint32_t u : {0x38800000u, 0x387FFFFFu, 0x33000000u, 0x33000001u, 0x477FEFFFu,
                     0x477FF000u, 0x7F800000u, 0x7FC00000u, 0x80000000u, 0xB3800000u}) {
    float f;
    std::memcpy(&f, &u, 4);
    bad += tileattn_b200::detail::to_f16_bits(f) != f16_bits_slow(f);
  }
  CHECK(bad == 0);
  int trip = 0;
  for (uint32_t h = 0; h < 65536; ++h) {
    if (((h >> 10) & 0x1Fu) == 31 && (h & 0x3FFu)) continue;  // NaN payloads
    trip += tileattn_b200::detail::to_f16_bits(
                tileattn_b200::detail::from_bits(uint16_t(h), DType::F16Emu)) != h;
  }
  CHECK(trip == 0);
}

static void test_validation_order_and_classes() {  // tiled.cpp:256-259, types.cpp:80-116
  PlanCache cache;
  AttnInput bad = make_input(Shape{1, 1, 32, 64}, DType::BF16Emu, 1);
  bad.shape.h = 0;  // shape is checked first, even with a bad schedule
  CHECK_THROWS_AS(sdpa_tiled(bad, MaskSpec::none(), ScaleSpec{}, TileSchedule{48, 64, 1}, cache),
                  std::invalid_argument);
  const AttnInput in = make_input(Shape{2, 1, 32, 64}, DType::BF16Emu, 1);
  CHECK_THROWS_AS(sdpa_tiled(in, MaskSpec::padding({4}), ScaleSpec{}, TileSchedule{}, cache),
                  std::invalid_argument);
  CHECK_THROWS_AS(sdpa_tiled(in, MaskSpec::padding({4, 33}), ScaleSpec{}, TileSchedule{}, cache),
                  std::invalid_argument);
  CHECK_THROWS_AS(sdpa_tiled(in, MaskSpec::none(), ScaleSpec{-1.0}, TileSchedule{}, cache),
                  std::invalid_argument);
  CHECK_THROWS_AS(effective_scale(ScaleSpec{0.0}, 64), std::invalid_argument);
  CHECK(effective_scale(ScaleSpec{}, 64) == 0.125);
  // not covered by the tensor-core kernel -> "unsupported" (bench.cpp:290-292)
  const AttnInput f32 = make_input(Shape{1, 1, 32, 64}, DType::F32, 1);
  CHECK_THROWS_AS(sdpa_tiled(f32, MaskSpec::none(), ScaleSpec{}, TileSchedule{}, cache),
                  UnsupportedScheduleError);
  for (int64_t d : {44, 264}) {  // not a multiple of 8 / above 256
    const AttnInput odd = make_input(Shape{1, 2, 32, d}, DType::BF16Emu, 77);
    CHECK_THROWS_AS(sdpa_tiled(odd, MaskSpec::none(), ScaleSpec{}, TileSchedule{}, cache),
                    UnsupportedScheduleError);
  }
  TiledOptions f64;
  f64.accum = AccumMode::F64;
  CHECK_THROWS_AS(sdpa_tiled(in, MaskSpec::none(), ScaleSpec{}, TileSchedule{}, cache, f64),
                  UnsupportedScheduleError);
}

// ---------------------------------------------------------------- GPU cases
static void test_tiled_kernel_matches_the_reference_oracle() {  // test_tiled.cpp:273-291
  PlanCache cache;
  for (int64_t s : {32, 130}) {
    for (DType dt : {DType::F16Emu, DType::BF16Emu}) {
      for (int64_t d : {64, 96, 128, 160, 256}) {
        const AttnInput in = make_input(Shape{1, 2, s, d}, dt, 77);
        for (const MaskSpec& mask : {MaskSpec::none(), MaskSpec::causal(),
                                     MaskSpec::padding({std::max<int64_t>(1, s / 2)})}) {
          const std::vector<double> ref = oracle_o(in, mask);
          for (TileLayout lay : {TileLayout::RowPacked, TileLayout::ColPacked}) {
            const std::vector<float> got =
                sdpa_tiled(in, mask, ScaleSpec{}, TileSchedule{64, 64, 2, lay}, cache);
            CHECK(max_abs_diff(got, ref) <= dtype_tol(dt));
          }
        }
      }
    }
  }
}

static void test_plan_cache_hits_and_constructions() {  // test_tiled.cpp:234-254
  PlanCache cache;
  const AttnInput in = make_input(Shape{1, 1, 64, 64}, DType::BF16Emu, 3);
  const TileSchedule sched{64, 64, 2, TileLayout::RowPacked};
  (void)sdpa_tiled(in, MaskSpec::none(), ScaleSpec{}, sched, cache);
  CHECK(cache.constructions() == 1 && cache.hits() == 0);
  (void)sdpa_tiled(in, MaskSpec::none(), ScaleSpec{}, sched, cache);
  CHECK(cache.constructions() == 1 && cache.hits() == 1);
  (void)sdpa_tiled(in, MaskSpec::causal(), ScaleSpec{}, sched, cache);
  CHECK(cache.constructions() == 2);
}

static void test_causal_tiles_above_the_diagonal_are_never_visited() {  // test_tiled.cpp:305-334
  PlanCache cache;
  const AttnInput ragged = make_input(Shape{1, 1, 1000, 64}, DType::F16Emu, 3);
  KernelStats rs;
  TiledOptions opt;
  opt.stats = &rs;
  (void)sdpa_tiled(ragged, MaskSpec::causal(), ScaleSpec{}, TileSchedule{64, 128, 2}, cache, opt);
  // the executed query tile is block_m rows; the formula is the reference's
  uint64_t want = 0;
  for (int64_t r0 = 0; r0 < 1000; r0 += rs.block_m) {
    const int64_t last = std::min<int64_t>(r0 + rs.block_m - 1, 999);
    want += uint64_t((last + 1 + rs.block_n - 1) / rs.block_n);
  }
  CHECK(rs.kv_tiles_visited.load() == want);
}

static void test_causal_outputs_independent_of_future_keys() {  // test_tiled.cpp:336-357
  PlanCache cache;
  const Shape sh{1, 1, 256, 64};
  const AttnInput in = make_input(sh, DType::BF16Emu, 8);
  const std::vector<float> base = sdpa_tiled(in, MaskSpec::causal(), ScaleSpec{}, TileSchedule{}, cache);
  std::mt19937_64 rng(12);
  for (int trial = 0; trial < 10; ++trial) {
    const int64_t i = int64_t(rng() % 255);
    const int64_t j = i + 1 + int64_t(rng() % uint64_t(256 - i - 1));
    AttnInput mutated = in;
    for (int64_t d = 0; d < sh.d; ++d) {
      mutated.k[size_t(j * sh.d + d)] += 3.5f;
      mutated.v[size_t(j * sh.d + d)] -= 1.25f;
    }
    const std::vector<float> out =
        sdpa_tiled(mutated, MaskSpec::causal(), ScaleSpec{}, TileSchedule{}, cache);
    CHECK(std::memcmp(out.data(), base.data(), size_t((i + 1) * sh.d) * sizeof(float)) == 0);
  }
}

static void test_padding_rows_past_valid_len_produce_zero_rows() {  // test_tiled.cpp:359-370
  PlanCache cache;
  const AttnInput in = make_input(Shape{2, 1, 40, 64}, DType::BF16Emu, 6);
  const std::vector<float> out =
      sdpa_tiled(in, MaskSpec::padding({0, 20}), ScaleSpec{}, TileSchedule{}, cache);
  bool zero = true;
  for (int64_t i = 0; i < 40 * 64; ++i) zero &= out[size_t(i)] == 0.0f;
  CHECK(zero);
  CHECK(max_abs_diff(out, oracle_o(in, MaskSpec::padding({0, 20}))) <= dtype_tol(DType::BF16Emu));
}

static void test_worker_count_does_not_change_the_output_bytes() {  // test_tiled.cpp:387-400
  const AttnInput in = make_input(Shape{2, 2, 96, 64}, DType::F16Emu, 456);
  PlanCache c1, c2;
  TiledOptions one, four;
  one.threads = 1;
  four.threads = 4;
  const auto a = sdpa_tiled(in, MaskSpec::causal(), ScaleSpec{}, TileSchedule{32, 32, 3}, c1, one);
  const auto b = sdpa_tiled(in, MaskSpec::causal(), ScaleSpec{}, TileSchedule{32, 32, 3}, c2, four);
  CHECK(std::memcmp(a.data(), b.data(), a.size() * sizeof(float)) == 0);
}

static void test_single_key_and_zero_queries() {  // test_reference.cpp:77-103
  PlanCache cache;
  const AttnInput s1 = make_input(Shape{1, 1, 1, 64}, DType::BF16Emu, 3);
  const auto o1 = sdpa_tiled(s1, MaskSpec::none(), ScaleSpec{}, TileSchedule{}, cache);
  CHECK(std::memcmp(o1.data(), s1.v.data(), 64 * sizeof(float)) == 0);  // O = v exactly
  AttnInput z = make_input(Shape{1, 1, 6, 64}, DType::F16Emu, 1);
  std::fill(z.q.begin(), z.q.end(), 0.0f);
  const auto oz = sdpa_tiled(z, MaskSpec::none(), ScaleSpec{}, TileSchedule{}, cache);
  double err = 0;
  for (int64_t d = 0; d < 64; ++d) {
    double mean = 0;
    for (int64_t j = 0; j < 6; ++j) mean += z.v[size_t(j * 64 + d)] / 6.0;
    for (int64_t i = 0; i < 6; ++i) err = std::max(err, std::abs(oz[size_t(i * 64 + d)] - mean));
  }
  CHECK(err <= dtype_tol(DType::F16Emu));
}

int main(int argc, char** argv) {
  const bool cpu_only = argc > 1 && std::string(argv[1]) == "--cpu-only";
  std::vector<std::pair<const char*, std::function<void()>>> cases = {
      {"unsupported schedules are rejected", test_unsupported_schedules_are_rejected},
      {"validation order and error classes", test_validation_order_and_classes},
      {"host f16 conversions round to nearest even", test_host_f16_conversions},
  };
  if (!cpu_only) {
    cases.insert(cases.end(), {
        {"tiled kernel matches the reference oracle", test_tiled_kernel_matches_the_reference_oracle},
        {"plan cache hits and constructions", test_plan_cache_hits_and_constructions},
        {"causal K/V tiles above the diagonal are never visited",
         test_causal_tiles_above_the_diagonal_are_never_visited},
        {"causal outputs are bitwise independent of future keys",
         test_causal_outputs_independent_of_future_keys},
        {"padding rows past valid_len produce zero rows",
         test_padding_rows_past_valid_len_produce_zero_rows},
        {"worker count does not change the output bytes",
         test_worker_count_does_not_change_the_output_bytes},
        {"single key and zero queries", test_single_key_and_zero_queries},
    });
  }
  for (auto& [name, fn] : cases) {
    const int before = g_failures;
    try {
      fn();
    } catch (const std::exception& e) {
      ++g_failures;
      std::fprintf(stderr, "[%s] unexpected exception: %s\n", name, e.what());
    }
    std::printf("[%s] %s\n", g_failures == before ? "PASS" : "FAIL", name);
  }
  std::printf("%d checks, %d failures\n", g_checks, g_failures);
  return g_failures == 0 ? 0 : 1;
}
