// The B200 operator as a method of the reference's own benchmark harness
// (reference proj/include/tileattn/bench.hpp): the translation unit a
// maintainer adds next to proj/src/bench.cpp.  It uses only the reference's
// public harness API (Workload, check_correctness, time_method, BenchRecord,
// write_records / write_manifest, make_mask) and the C-ABI of
// libtileattn_b200.so — no reference source is modified.
//
//   run_b200()        = the body of run_method("b200", ...)  (bench.cpp:111-142)
//   run_grid_b200()   = run_grid (bench.cpp:235-331) with "b200" registered
//                       next to the reference's methods
#pragma once

#include <string>
#include <vector>

#include "tileattn/bench.hpp"

namespace tileattn_b200_harness {

// Name the method is registered under in the grid.
inline constexpr const char* kMethodName = "b200";

// One forward through ta_sdpa_fwd_host: the f32-on-grid workload is encoded
// to 16-bit storage bits (exact), run on the current CUDA device, decoded
// back (exact).  Errors map to the reference's exception classes:
// invalid_argument, UnsupportedScheduleError, bad_alloc, runtime_error.
std::vector<float> run_b200(const tileattn::Workload& workload,
                            const tileattn::TileSchedule& sched);

// The reference's grid cross product (method-major, then schedule for
// schedule-dependent methods, then S, D, dtype, mask) with "b200" available
// as a schedule-dependent method; every other name goes to
// tileattn::run_method.  Same per-point protocol: correctness gate (S <= 256
// directly, else on the S = 256 twin), then time_method, then metrics;
// failures become status-annotated NaN rows.
tileattn::RunResult run_grid_b200(const tileattn::GridConfig& config);

}  // namespace tileattn_b200_harness
