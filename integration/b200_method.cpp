// The B200 operator registered in the reference's benchmark harness (see
// b200_method.hpp).  Built against the reference headers and linked with the
// reference's own harness translation units plus libtileattn_b200.so by
// oracle/Makefile (target b200_grid) — the reference sources are compiled
// where they lie, never copied.
#include "b200_method.hpp"

#include <cmath>
#include <limits>
#include <new>
#include <stdexcept>
#include <utility>
#include <vector>

#include "tileattn/analysis.hpp"
#include "tileattn_b200.hpp"  // the C++ mirror of sdpa_tiled over the C-ABI

namespace tileattn_b200_harness {
namespace {

namespace ref = tileattn;
namespace gpu = tileattn_b200;

gpu::DType to_gpu(ref::DType dt) {
  switch (dt) {
    case ref::DType::F16Emu: return gpu::DType::F16Emu;
    case ref::DType::BF16Emu: return gpu::DType::BF16Emu;
    default: return gpu::DType::F32;
  }
}

gpu::MaskSpec to_gpu(const ref::MaskSpec& m) {
  switch (m.kind) {
    case ref::MaskKind::Causal: return gpu::MaskSpec::causal();
    case ref::MaskKind::Padding: return gpu::MaskSpec::padding(m.valid_len);
    default: return gpu::MaskSpec::none();
  }
}

gpu::TileSchedule to_gpu(const ref::TileSchedule& s) {
  return gpu::TileSchedule{s.t_m, s.t_n, s.stages,
                           s.layout == ref::TileLayout::ColPacked ? gpu::TileLayout::ColPacked
                                                                  : gpu::TileLayout::RowPacked};
}

// one plan-cache accounting object per process, like the harness's PlanCache
gpu::PlanCache& gpu_cache() {
  static gpu::PlanCache cache;
  return cache;
}

// status-annotated NaN row (the reference's convention for failed points)
void fail_point(ref::BenchRecord& rec, ref::BenchStatus status, std::string why) {
  constexpr double nan = std::numeric_limits<double>::quiet_NaN();
  rec.status = status;
  rec.status_detail = std::move(why);
  rec.median_ms = rec.p95_ms = rec.tokens_per_s = rec.bw_proxy = nan;
}

}  // namespace

std::vector<float> run_b200(const ref::Workload& workload, const ref::TileSchedule& sched) {
  gpu::AttnInput in;
  const ref::Shape& sh = workload.input.shape;
  in.shape = gpu::Shape{sh.b, sh.h, sh.s, sh.d};
  in.dtype = to_gpu(workload.input.dtype);
  in.q = workload.input.q;
  in.k = workload.input.k;
  in.v = workload.input.v;
  gpu::ScaleSpec scale{workload.scale.value};
  try {
    return gpu::sdpa_tiled(in, to_gpu(workload.mask), scale, to_gpu(sched), gpu_cache());
  } catch (const gpu::UnsupportedScheduleError& e) {
    // the harness records these as status=unsupported rows (bench.cpp:290-292)
    throw ref::UnsupportedScheduleError(e.what());
  }
}

ref::RunResult run_grid_b200(const ref::GridConfig& config) {
  {  // the reference's config validation, minus its registry check for "b200"
    ref::GridConfig others = config;
    std::erase(others.methods, std::string(kMethodName));
    if (others.methods.empty()) others.methods = {"tiled"};
    ref::validate(others);
  }
  ref::RunResult out;
  out.manifest = ref::make_manifest(config);
  out.manifest.artifact_version += " + tileattn_b200 (sm_100a)";
  ref::PlanCache cpu_cache;

  for (const std::string& name : config.methods) {
    const bool ours = name == kMethodName;
    const ref::MethodDesc* desc = ours ? nullptr : ref::find_method(name);
    if (!ours && desc == nullptr) throw std::invalid_argument("unknown method: " + name);
    const bool by_schedule = ours || desc->schedule_dependent;
    const std::vector<ref::TileSchedule> schedules =
        by_schedule ? config.schedules : std::vector<ref::TileSchedule>{ref::TileSchedule{}};

    auto method = [&](const ref::TileSchedule& sched) {
      return [&, sched](const ref::Workload& w) {
        return ours ? run_b200(w, sched)
                    : ref::run_method(name, w, sched, cpu_cache, config.threads);
      };
    };

    for (const ref::TileSchedule& sched : schedules)
      for (int64_t s : config.s_values)
        for (int64_t d : config.d_values)
          for (ref::DType dtype : config.dtypes)
            for (ref::MaskKind kind : config.masks) {
              ref::BenchRecord rec;
              rec.method = name;
              rec.b = config.b;
              rec.h = config.h;
              rec.s = s;
              rec.d = d;
              rec.dtype = dtype;
              rec.causal = kind == ref::MaskKind::Causal;
              if (by_schedule) rec.schedule = sched;
              if (!ours && !desc->available) {
                fail_point(rec, ref::BenchStatus::Unsupported,
                           "method not available on this backend");
                out.records.push_back(std::move(rec));
                continue;
              }
              const auto runner = method(sched);
              auto workload = [&](int64_t seq) {
                const ref::Shape shape{config.b, config.h, seq, d};
                return ref::Workload{ref::make_input(shape, dtype, config.seed),
                                     ref::make_mask(kind, shape), ref::ScaleSpec{}};
              };
              try {
                // correctness gate against the reference oracle (on the
                // S = 256 twin for longer sequences), then device timing of
                // the full point through the same call
                const int64_t gate_s = s < 256 ? s : 256;
                const ref::CheckResult chk =
                    ref::check_correctness(runner, workload(gate_s), dtype);
                if (!chk.passed) {
                  fail_point(rec, ref::BenchStatus::CheckFailed,
                             "max_abs_err=" + std::to_string(chk.max_abs_err) + " exceeds tol=" +
                                 std::to_string(chk.tol_used) + " (twin S=" +
                                 std::to_string(gate_s) + ")");
                } else {
                  const ref::Workload w = workload(s);
                  const ref::TimingStats t =
                      ref::time_method([&] { (void)runner(w); }, config.n_warmup, config.n_timed);
                  rec.median_ms = t.median_ms;
                  rec.p95_ms = t.p95_ms;
                  rec.tokens_per_s = ref::tokens_per_second(config.b, config.h, s, t.median_ms);
                  rec.bw_proxy = ref::bandwidth_proxy(config.b, config.h, s, d,
                                                      ref::bytes_per_elem(dtype), t.median_ms);
                  rec.status = ref::BenchStatus::Ok;
                }
              } catch (const ref::UnsupportedScheduleError& e) {
                fail_point(rec, ref::BenchStatus::Unsupported, e.what());
              } catch (const std::bad_alloc&) {
                fail_point(rec, ref::BenchStatus::Oom, "allocation failure");
              }
              out.records.push_back(std::move(rec));
            }
  }
  return out;
}

}  // namespace tileattn_b200_harness
