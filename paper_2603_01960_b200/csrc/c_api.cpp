// C-ABI host layer (include/tileattn_b200.h): validation with the reference's
// order and error classes, the plan cache, TMA descriptor encoding and the
// launch of the sm_100a kernel.  No CPU fallback: every compute call either
// runs the CUDA kernel or returns an error.
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/tileattn_b200.h"
#include "sdpa_fwd_sm100.h"

namespace {

thread_local std::string g_last_error;

ta_status fail(ta_status st, const std::string& msg) {
  g_last_error = msg;
  return st;
}

ta_status cuda_fail(cudaError_t e, const char* what) {
  return fail(e == cudaErrorMemoryAllocation ? TA_ERR_OOM : TA_ERR_CUDA,
              std::string(what) + ": " + cudaGetErrorString(e));
}

// ---------------------------------------------------------------------------
// Validation — restates types.cpp:80-116 and tiled.cpp:21-35.
// ---------------------------------------------------------------------------
bool schedule_ok(const ta_schedule& s) {
  const bool tm = s.t_m == 16 || s.t_m == 32 || s.t_m == 64 || s.t_m == 128;
  const bool tn = s.t_n == 16 || s.t_n == 32 || s.t_n == 64 || s.t_n == 128 || s.t_n == 256;
  return tm && tn && s.stages >= 1 && s.stages <= 4 && (s.layout == 0 || s.layout == 1);
}

ta_schedule resolve_schedule(ta_schedule s) {
  if (s.t_m == 0 && s.t_n == 0 && s.stages == 0 && s.layout == 0)
    return ta_schedule{64, 128, 2, 0};  // TileSchedule{} default (tiled.hpp:30-37)
  return s;
}

ta_status validate_common(ta_shape sh, ta_mask_kind mask, const int64_t* valid_len,
                          ta_schedule sched, int has_scale, double scale, double* eff_scale) {
  // shape (types.cpp:80-83)
  if (sh.b < 1 || sh.h < 1 || sh.s < 1 || sh.d < 1)
    return fail(TA_ERR_INVALID_ARGUMENT, "shape extents must all be >= 1");
  // mask (types.cpp:99-106)
  if (mask != TA_MASK_NONE && mask != TA_MASK_CAUSAL && mask != TA_MASK_PADDING)
    return fail(TA_ERR_INVALID_ARGUMENT, "unknown mask kind");
  if (mask == TA_MASK_PADDING) {
    if (valid_len == nullptr)
      return fail(TA_ERR_INVALID_ARGUMENT, "padding mask needs one valid_len per batch");
    for (int64_t b = 0; b < sh.b; ++b)
      if (valid_len[b] < 0 || valid_len[b] > sh.s)
        return fail(TA_ERR_INVALID_ARGUMENT, "padding valid_len out of [0,S]");
  }
  // schedule (tiled.cpp:29-35)
  if (!schedule_ok(sched))
    return fail(TA_ERR_UNSUPPORTED, "unsupported schedule: t_m=" + std::to_string(sched.t_m) +
                                        " t_n=" + std::to_string(sched.t_n) +
                                        " stages=" + std::to_string(sched.stages));
  // scale (types.cpp:108-116)
  if (has_scale) {
    // the reference predicate (types.cpp:108-116 throws for *scale <= 0.0):
    // NaN passes, as there, and propagates into O / LSE
    if (scale <= 0.0)
      return fail(TA_ERR_INVALID_ARGUMENT, "effective_scale: explicit scale must be > 0");
    *eff_scale = scale;
  } else {
    *eff_scale = 1.0 / std::sqrt(double(sh.d));
  }
  return TA_OK;
}

ta_status validate_device_support(ta_shape sh, ta_dtype dt, ta_mask_kind mask) {
  if (dt == TA_F32)
    return fail(TA_ERR_UNSUPPORTED, "dtype f32 is not a tensor-core input; use f16 or bf16");
  if (dt != TA_F16 && dt != TA_BF16) return fail(TA_ERR_INVALID_ARGUMENT, "unknown dtype");
  // D runs on the smallest kernel of 64 / 128 / 192 / 256 columns that
  // holds it: the TMA boxes zero-fill the columns past D (they add nothing to
  // Q.K^T and give zero O columns, which are not stored).  Rows must be 16-B
  // aligned for TMA.  D > 256 would need more than the 512 TMEM columns.
  if (sh.d > 256 || sh.d % 8 != 0)
    return fail(TA_ERR_UNSUPPORTED, "head dim " + std::to_string(sh.d) +
                                        " not supported (D a multiple of 8, D <= 256)");
  if (sh.s > (int64_t(1) << 30)) return fail(TA_ERR_UNSUPPORTED, "S too large");
  if (ta::fwd_geometry(sh.s, sh.b * sh.h, sh.d).ctas > 0x7FFFFFFF)
    return fail(TA_ERR_UNSUPPORTED, "more than 2^31 - 1 CTAs (B*H*ceil(S/rows per CTA))");
  return TA_OK;
}

// ---------------------------------------------------------------------------
// Plan cache: the reference's PlanCache (tiled.cpp:37-70) keyed by
// (t_m, t_n, D, dtype, causal).  The plan records the executed GPU tiling.
// ---------------------------------------------------------------------------
struct Plan {
  int block_m, block_n, stages, q_tiles, threads;
};

struct PlanCache {
  std::mutex mu;
  std::map<std::tuple<int, int, int64_t, int, int>, std::shared_ptr<const Plan>> plans;
  std::atomic<uint64_t> hits{0}, constructions{0};
};

PlanCache& plan_cache() {
  static PlanCache c;
  return c;
}

std::shared_ptr<const Plan> get_plan(const ta_schedule& s, int64_t d, ta_dtype dt, bool causal) {
  PlanCache& c = plan_cache();
  const auto key = std::make_tuple(s.t_m, s.t_n, d, int(dt), int(causal));
  {
    std::lock_guard<std::mutex> lock(c.mu);
    auto it = c.plans.find(key);
    if (it != c.plans.end()) {
      c.hits.fetch_add(1, std::memory_order_relaxed);
      return it->second;
    }
  }
  // the schedule's t_n selects the executed K/V tile (64 keys for t_n <= 64
  // where a 64-key kernel exists, else 128); t_m is a hint: the tcgen05 M
  // tile is 128 rows (two per CTA at D <= 128)
  const int bn = ta::fwd_block_n(d, s.t_n);
  auto g = ta::fwd_geometry(1, 1, d, bn);
  auto plan = std::make_shared<const Plan>(
      Plan{g.block_m, g.block_n, ta::fwd_ring_slots(int(d), bn), g.q_tiles_per_cta, g.threads});
  c.constructions.fetch_add(1, std::memory_order_relaxed);
  std::lock_guard<std::mutex> lock(c.mu);
  auto [it, inserted] = c.plans.emplace(key, std::move(plan));
  return it->second;
}

// ---------------------------------------------------------------------------
// TMA descriptors (driver entry point fetched through the runtime, so the
// library does not link libcuda and loads on GPU-less hosts).
// ---------------------------------------------------------------------------
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return EncodeTiledFn(nullptr);
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// [BH][rows][cols] 16-bit tensor, boxes of 64 cols (128 B, SWIZZLE_128B) x box_rows.
ta_status encode_tmap(CUtensorMap* m, const void* ptr, bool bf16, int64_t bh, int64_t rows,
                      int64_t cols, uint32_t box_rows) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(TA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (driver too old?)");
  cuuint64_t dims[3] = {cuuint64_t(cols), cuuint64_t(rows), cuuint64_t(bh)};
  cuuint64_t strides[2] = {cuuint64_t(cols * 2), cuuint64_t(rows * cols * 2)};
  cuuint32_t box[3] = {64, box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                   3, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(TA_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
  return TA_OK;
}

// Per-thread memo of recent tensor maps (the same q/k/v buffers recur call
// after call; a map is a pure function of these fields), so the small-shape
// host path pays no encode.
ta_status make_tmap(CUtensorMap* m, const void* ptr, bool bf16, int64_t bh, int64_t rows,
                    int64_t cols, uint32_t box_rows) {
  struct Entry {
    const void* ptr = nullptr;
    int64_t bh = 0, rows = 0, cols = 0;
    uint32_t box_rows = 0;
    bool bf16 = false;
    CUtensorMap map;
  };
  constexpr int kEntries = 8;
  thread_local Entry memo[kEntries];
  thread_local int next = 0;
  for (const Entry& e : memo)
    if (e.ptr == ptr && e.ptr != nullptr && e.bh == bh && e.rows == rows && e.cols == cols &&
        e.box_rows == box_rows && e.bf16 == bf16) {
      *m = e.map;
      return TA_OK;
    }
  ta_status st = encode_tmap(m, ptr, bf16, bh, rows, cols, box_rows);
  if (st != TA_OK) return st;
  Entry& e = memo[next];
  next = (next + 1) % kEntries;
  e.ptr = ptr;
  e.bh = bh;
  e.rows = rows;
  e.cols = cols;
  e.box_rows = box_rows;
  e.bf16 = bf16;
  e.map = *m;
  return TA_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int device_cc(int dev) {
  static std::mutex mu;
  static std::map<int, int> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int major = 0, minor = 0;
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  return cache[dev] = major * 10 + minor;
}

ta_status check_device() {
  int dev = -1;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(TA_ERR_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
  }
  if (device_cc(dev) != 100)
    return fail(TA_ERR_CUDA, "device " + std::to_string(dev) +
                                 " is not sm_100 (this library carries sm_100a code only)");
  return TA_OK;
}

// KernelStats::kv_tiles_visited (tiled.hpp:246-257) for the executed 128-row
// query tiles: causal visits kv_end = last_row / t_n + 1 tiles (tiled.cpp:159),
// padding ceil(valid_len / t_n).
void fill_stats(ta_kernel_stats* st, const Plan& p, ta_shape sh, ta_mask_kind mask,
                const int64_t* valid_len) {
  if (!st) return;
  const int64_t bh = sh.b * sh.h;
  const int64_t q_tiles = (sh.s + p.block_m - 1) / p.block_m;
  const int64_t kv_tiles = (sh.s + p.block_n - 1) / p.block_n;
  const auto g = ta::fwd_geometry(sh.s, bh, sh.d, p.block_n);
  uint64_t visited = 0;
  if (mask == TA_MASK_CAUSAL) {
    for (int64_t qt = 0; qt < q_tiles; ++qt) {
      const int64_t last = std::min<int64_t>((qt + 1) * p.block_m, sh.s) - 1;
      visited += uint64_t(last / p.block_n + 1);
    }
    visited *= uint64_t(bh);
  } else if (mask == TA_MASK_PADDING) {
    for (int64_t b = 0; b < sh.b; ++b)
      visited += uint64_t(sh.h * q_tiles * ((valid_len[b] + p.block_n - 1) / p.block_n));
  } else {
    visited = uint64_t(bh * q_tiles * kv_tiles);
  }
  st->kv_tiles_visited = visited;
  st->block_m = p.block_m;
  st->block_n = p.block_n;
  st->stages = p.stages;
  st->q_tiles_per_cta = p.q_tiles;
  st->ctas = g.ctas;
  st->threads_per_cta = p.threads;
  st->reserved = 0;
}

// Device copies of padding lengths for B > kInlinePadding: a per-device pool
// of (pinned host, device, event) slots.  A slot is taken when its last
// launch has completed (event query), so steady-state calls allocate nothing
// and the copy source is pinned (asynchronous).
struct PaddingSlot {
  int* host = nullptr;
  int* dev = nullptr;
  size_t cap = 0;
  cudaEvent_t done = nullptr;
  std::atomic<bool> busy{false};  // taken under the pool mutex, released by its user
};

struct PaddingPool {
  std::mutex mu;
  std::vector<std::unique_ptr<PaddingSlot>> slots;
};

PaddingPool& padding_pool(int dev) {
  static std::mutex mu;
  static std::map<int, std::unique_ptr<PaddingPool>> pools;
  std::lock_guard<std::mutex> lock(mu);
  auto& p = pools[dev];
  if (!p) p = std::make_unique<PaddingPool>();
  return *p;
}

void release_padding_pool(int dev) {
  PaddingPool& pool = padding_pool(dev);
  std::lock_guard<std::mutex> lock(pool.mu);
  for (auto& sl : pool.slots) {
    if (sl->done) cudaEventSynchronize(sl->done);
    if (sl->dev) cudaFree(sl->dev);
    if (sl->host) cudaFreeHost(sl->host);
    if (sl->done) cudaEventDestroy(sl->done);
  }
  pool.slots.clear();
}

ta_status padding_slot(size_t n, PaddingSlot** out) {
  int dev = 0;
  cudaGetDevice(&dev);
  PaddingPool& pool = padding_pool(dev);
  std::lock_guard<std::mutex> lock(pool.mu);
  PaddingSlot* pick = nullptr;
  for (auto& sl : pool.slots) {
    if (sl->busy.load(std::memory_order_acquire) || sl->cap < n) continue;
    const cudaError_t q = cudaEventQuery(sl->done);
    if (q == cudaSuccess) {
      pick = sl.get();
      break;
    }
    if (q != cudaErrorNotReady) return cuda_fail(q, "padding slot event");
  }
  if (pick == nullptr) {
    auto sl = std::make_unique<PaddingSlot>();
    const size_t cap = std::max<size_t>(n, 1024);
    cudaError_t e;
    if ((e = cudaMallocHost(reinterpret_cast<void**>(&sl->host), cap * sizeof(int))) != cudaSuccess ||
        (e = cudaMalloc(reinterpret_cast<void**>(&sl->dev), cap * sizeof(int))) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&sl->done, cudaEventDisableTiming)) != cudaSuccess) {
      if (sl->host) cudaFreeHost(sl->host);
      if (sl->dev) cudaFree(sl->dev);
      cudaGetLastError();
      return cuda_fail(e, "padding lengths (pool slot)");
    }
    sl->cap = cap;
    pick = sl.get();
    pool.slots.push_back(std::move(sl));
  }
  pick->busy.store(true, std::memory_order_relaxed);
  *out = pick;
  return TA_OK;
}

struct MaskArgs {
  ta_mask_kind kind = TA_MASK_NONE;
  const int64_t* valid_len = nullptr;  // host, [B] (padding)
  int64_t heads = 1;                   // H of the caller's [B,H,S,D] view
  int64_t bh_offset = 0;               // first flattened head of this launch
  int64_t batches = 1;
};

ta_status run_device(const void* q, const void* k, const void* v, void* o, float* lse,
                     ta_shape sh, ta_dtype dt, double scale, const Plan& plan, void* stream,
                     const MaskArgs& mask_args, long long* trace = nullptr) {
  const bool bf16 = dt == TA_BF16;
  const int64_t bh = sh.b * sh.h;
  CUtensorMap mq, mk, mv;
  ta_status st;
  if ((st = make_tmap(&mq, q, bf16, bh, sh.s, sh.d, 128)) != TA_OK) return st;
  const uint32_t kv_rows = uint32_t(plan.block_n);  // one TMA box = one K/V tile row block
  // CTA pair: each CTA loads half of a K tile's keys (boxes of block_n / 2 rows)
  const bool pair = ta::fwd_use_pair(ta::fwd_kernel_head_dim(sh.d), plan.block_n, int(mask_args.kind));
  if ((st = make_tmap(&mk, k, bf16, bh, sh.s, sh.d, pair ? kv_rows / 2 : kv_rows)) != TA_OK) return st;
  if ((st = make_tmap(&mv, v, bf16, bh, sh.s, sh.d, kv_rows)) != TA_OK) return st;
  CUtensorMap mo;
  if ((st = make_tmap(&mo, o, bf16, bh, sh.s, sh.d, 128)) != TA_OK) return st;
  ta::FwdLaunch L{};
  L.tmap_q = &mq;
  L.tmap_k = &mk;
  L.tmap_v = &mv;
  L.tmap_o = &mo;
  L.args.o = o;
  L.args.lse = lse;
  L.args.seq_len = int(sh.s);
  L.args.scale_log2 = float(scale * 1.4426950408889634074);
  L.args.trace = trace;
  L.args.mask = int(mask_args.kind);
  L.args.heads = int(mask_args.heads);
  L.args.bh_offset = int(mask_args.bh_offset);
  // padding lengths: inline for B <= kInlinePadding, else a device array
  // from the per-device pool (pinned staging, stream-ordered copy; a slot is
  // reused once the launch that read it has completed)
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  PaddingSlot* slot = nullptr;
  if (mask_args.kind == TA_MASK_PADDING) {
    if (mask_args.batches <= ta::kInlinePadding) {
      for (int64_t b = 0; b < mask_args.batches; ++b)
        L.args.valid_len[b] = int(mask_args.valid_len[b]);
    } else {
      // the pool's pinned staging and event queries cannot live in a CUDA
      // graph (a replay would read whatever the slot holds then): refuse
      cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
      if (cudaStreamIsCapturing(cs, &cap) == cudaSuccess && cap != cudaStreamCaptureStatusNone)
        return fail(TA_ERR_UNSUPPORTED,
                    "padding masks with more than 32 batches cannot be captured in a CUDA graph");
      ta_status pst = padding_slot(size_t(mask_args.batches), &slot);
      if (pst != TA_OK) return pst;
      for (int64_t b = 0; b < mask_args.batches; ++b) slot->host[b] = int(mask_args.valid_len[b]);
      cudaError_t e = cudaMemcpyAsync(slot->dev, slot->host, size_t(mask_args.batches) * sizeof(int),
                                      cudaMemcpyHostToDevice, cs);
      if (e != cudaSuccess) {
        slot->busy.store(false, std::memory_order_release);
        return cuda_fail(e, "padding lengths (copy)");
      }
      L.args.valid_len_dev = slot->dev;
    }
  }
  L.bh = bh;
  L.head_dim = ta::fwd_kernel_head_dim(sh.d);  // kernel instantiation
  L.block_n = plan.block_n;
  L.pair = pair;
  L.args.head_dim = int(sh.d);         // row length of q/k/v/o in memory
  L.bf16 = bf16;
  L.stream = stream;

  cudaError_t e = ta::launch_sdpa_fwd(L);
  if (slot != nullptr) {
    // the slot is free again once this launch (which read it) completes
    cudaError_t er = cudaEventRecord(slot->done, cs);
    slot->busy.store(false, std::memory_order_release);  // after the record
    if (e == cudaSuccess && er != cudaSuccess) e = er;
  }
  if (e != cudaSuccess) return cuda_fail(e, "sdpa_fwd launch");
  return TA_OK;
}

// per-device workspace for the host-buffer entry: device buffers plus the
// copy streams / events of the chunked H2D -> compute -> D2H pipeline
struct Workspace {
  static constexpr int kMaxChunks = 64;
  std::mutex mu;
  void* ptr = nullptr;
  size_t bytes = 0;
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t ev_in[kMaxChunks] = {}, ev_out[kMaxChunks] = {};
  cudaEvent_t ev_compute_done = nullptr;

  ta_status ensure_streams() {
    if (h2d) return TA_OK;
    cudaError_t e;
    if ((e = cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&ev_compute_done, cudaEventDisableTiming)) != cudaSuccess)
      return cuda_fail(e, "workspace streams");
    for (int i = 0; i < kMaxChunks; ++i)
      if ((e = cudaEventCreateWithFlags(&ev_in[i], cudaEventDisableTiming)) != cudaSuccess ||
          (e = cudaEventCreateWithFlags(&ev_out[i], cudaEventDisableTiming)) != cudaSuccess)
        return cuda_fail(e, "workspace events");
    return TA_OK;
  }
};

Workspace& workspace(int dev) {
  static std::mutex mu;
  static std::map<int, std::unique_ptr<Workspace>> ws;
  std::lock_guard<std::mutex> lock(mu);
  auto& w = ws[dev];
  if (!w) w = std::make_unique<Workspace>();
  return *w;
}

}  // namespace

extern "C" {

const char* ta_last_error(void) { return g_last_error.c_str(); }

int ta_abi_version(void) { return TA_ABI_VERSION; }

int ta_schedule_supported(ta_schedule sched) { return schedule_ok(sched) ? 1 : 0; }

ta_status ta_effective_scale(int has_scale, double scale, int64_t d, double* out) {
  if (d < 1) return fail(TA_ERR_INVALID_ARGUMENT, "effective_scale: D must be >= 1");
  if (has_scale) {
    if (scale <= 0.0)  // reference predicate: NaN is accepted (types.cpp:108-116)
      return fail(TA_ERR_INVALID_ARGUMENT, "effective_scale: explicit scale must be > 0");
    if (out) *out = scale;
    return TA_OK;
  }
  if (out) *out = 1.0 / std::sqrt(double(d));
  return TA_OK;
}

void ta_plan_cache_stats(uint64_t* hits, uint64_t* constructions) {
  if (hits) *hits = plan_cache().hits.load();
  if (constructions) *constructions = plan_cache().constructions.load();
}

void ta_plan_cache_clear(void) {
  PlanCache& c = plan_cache();
  std::lock_guard<std::mutex> lock(c.mu);
  c.plans.clear();
  c.hits = 0;
  c.constructions = 0;
}

ta_status ta_sdpa_check(ta_shape shape, ta_dtype dtype, ta_mask_kind mask,
                        const int64_t* valid_len, int has_scale, double scale,
                        ta_schedule sched) {
  sched = resolve_schedule(sched);
  double eff = 0.0;
  ta_status st = validate_common(shape, mask, valid_len, sched, has_scale, scale, &eff);
  if (st != TA_OK) return st;
  return validate_device_support(shape, dtype, mask);
}

int ta_device_supported(int device) { return device_cc(device) == 100 ? 1 : 0; }

ta_status ta_sdpa_fwd(const void* q, const void* k, const void* v, void* o, float* lse,
                      ta_shape shape, ta_dtype dtype, ta_mask_kind mask,
                      const int64_t* valid_len, int has_scale, double scale,
                      ta_schedule sched, void* stream, ta_kernel_stats* stats) {
  sched = resolve_schedule(sched);
  double eff = 0.0;
  ta_status st = validate_common(shape, mask, valid_len, sched, has_scale, scale, &eff);
  if (st != TA_OK) return st;
  if (!q || !k || !v || !o) return fail(TA_ERR_INVALID_ARGUMENT, "null tensor pointer");
  if ((st = validate_device_support(shape, dtype, mask)) != TA_OK) return st;
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o))
    return fail(TA_ERR_INVALID_ARGUMENT, "q/k/v/o must be 16-byte aligned");
  if ((st = check_device()) != TA_OK) return st;
  auto plan = get_plan(sched, shape.d, dtype, mask == TA_MASK_CAUSAL);
  MaskArgs mk{mask, valid_len, shape.h, 0, shape.b};
  if ((st = run_device(q, k, v, o, lse, shape, dtype, eff, *plan, stream, mk)) != TA_OK)
    return st;
  fill_stats(stats, *plan, shape, mask, valid_len);
  return TA_OK;
}

ta_status ta_sdpa_fwd_host(const void* q, const void* k, const void* v, void* o, float* lse,
                           ta_shape shape, ta_dtype dtype, ta_mask_kind mask,
                           const int64_t* valid_len, int has_scale, double scale,
                           ta_schedule sched, void* stream, ta_kernel_stats* stats) {
  sched = resolve_schedule(sched);
  double eff = 0.0;
  ta_status st = validate_common(shape, mask, valid_len, sched, has_scale, scale, &eff);
  if (st != TA_OK) return st;
  if (!q || !k || !v || !o) return fail(TA_ERR_INVALID_ARGUMENT, "null tensor pointer");
  if ((st = validate_device_support(shape, dtype, mask)) != TA_OK) return st;
  if ((st = check_device()) != TA_OK) return st;
  int dev = 0;
  cudaGetDevice(&dev);
  const size_t n = size_t(shape.b * shape.h * shape.s * shape.d);
  const size_t tbytes = (n * 2 + 255) & ~size_t(255);
  const size_t lbytes = lse ? ((size_t(shape.b * shape.h * shape.s) * 4 + 255) & ~size_t(255)) : 0;
  const size_t need = 4 * tbytes + lbytes;
  Workspace& ws = workspace(dev);
  std::lock_guard<std::mutex> lock(ws.mu);
  if (ws.bytes < need) {
    if (ws.ptr) cudaFree(ws.ptr);
    ws.ptr = nullptr;
    ws.bytes = 0;
    cudaError_t e = cudaMalloc(&ws.ptr, need);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return cuda_fail(e, "workspace cudaMalloc");
    }
    ws.bytes = need;
  }
  char* base = static_cast<char*>(ws.ptr);
  char* dq = base;
  char* dk = base + tbytes;
  char* dv = base + 2 * tbytes;
  char* dout = base + 3 * tbytes;
  float* dl = lse ? reinterpret_cast<float*>(base + 4 * tbytes) : nullptr;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  auto plan = get_plan(sched, shape.d, dtype, mask == TA_MASK_CAUSAL);
  // Pipeline over head chunks: H2D of chunk c+1 and D2H of chunk c-1 run on
  // the workspace's copy streams while chunk c computes on the caller's
  // stream (heads are independent and contiguous in [B*H, S, D]).
  const int64_t bh = shape.b * shape.h;
  const size_t head_elems = size_t(shape.s * shape.d);
  // ~64 MiB+ tensors: up to 64 chunks (the pipeline fill and drain are one
  // chunk's H2D and one chunk's compute + D2H; the H2D stream itself runs at
  // the PCIe rate the whole time), never below 8 MiB per input chunk
  const int64_t max_chunks = std::max<int64_t>(1, int64_t(n * 2 / (size_t(8) << 20)));
  const int n_chunks = int(n * 2 >= (size_t(64) << 20)
                               ? std::min<int64_t>({bh, int64_t(Workspace::kMaxChunks), max_chunks})
                               : 1);
  if ((st = ws.ensure_streams()) != TA_OK) return st;
  // enqueue the whole pipeline; on a failure part-way, drain every stream
  // before returning so no copy still reads the caller's q/k/v or writes o
  // (and the next call cannot reuse the workspace under them)
  auto enqueue = [&]() -> ta_status {
    int64_t h0 = 0;
    for (int c = 0; c < n_chunks; ++c) {
      const int64_t h1 = bh * (c + 1) / n_chunks;
      const int64_t hc = h1 - h0;
      if (hc == 0) continue;
      const size_t off = size_t(h0) * head_elems * 2, bytes = size_t(hc) * head_elems * 2;
      // inputs of this chunk, ordered after the previous call's use of the
      // workspace (the compute stream's last event)
      if ((e = cudaStreamWaitEvent(ws.h2d, ws.ev_compute_done, 0)) != cudaSuccess ||
          (e = cudaMemcpyAsync(dq + off, static_cast<const char*>(q) + off, bytes,
                               cudaMemcpyHostToDevice, ws.h2d)) != cudaSuccess ||
          (e = cudaMemcpyAsync(dk + off, static_cast<const char*>(k) + off, bytes,
                               cudaMemcpyHostToDevice, ws.h2d)) != cudaSuccess ||
          (e = cudaMemcpyAsync(dv + off, static_cast<const char*>(v) + off, bytes,
                               cudaMemcpyHostToDevice, ws.h2d)) != cudaSuccess ||
          (e = cudaEventRecord(ws.ev_in[c], ws.h2d)) != cudaSuccess ||
          (e = cudaStreamWaitEvent(s, ws.ev_in[c], 0)) != cudaSuccess)
        return cuda_fail(e, "H2D copy");
      const ta_shape cs{1, hc, shape.s, shape.d};
      MaskArgs mk{mask, valid_len, shape.h, h0, shape.b};
      ta_status rst = run_device(dq + off, dk + off, dv + off, dout + off,
                                 dl ? dl + size_t(h0) * size_t(shape.s) : nullptr, cs, dtype, eff,
                                 *plan, stream, mk);
      if (rst != TA_OK) return rst;
      if ((e = cudaEventRecord(ws.ev_out[c], s)) != cudaSuccess ||
          (e = cudaStreamWaitEvent(ws.d2h, ws.ev_out[c], 0)) != cudaSuccess ||
          (e = cudaMemcpyAsync(static_cast<char*>(o) + off, dout + off, bytes,
                               cudaMemcpyDeviceToHost, ws.d2h)) != cudaSuccess)
        return cuda_fail(e, "D2H copy");
      if (lse && (e = cudaMemcpyAsync(lse + size_t(h0) * size_t(shape.s),
                                      dl + size_t(h0) * size_t(shape.s),
                                      size_t(hc) * size_t(shape.s) * 4, cudaMemcpyDeviceToHost,
                                      ws.d2h)) != cudaSuccess)
        return cuda_fail(e, "D2H copy");
      h0 = h1;
    }
    return TA_OK;
  };
  st = enqueue();
  if (st != TA_OK) {
    const std::string msg = g_last_error;
    cudaStreamSynchronize(ws.h2d);
    cudaStreamSynchronize(ws.d2h);
    cudaStreamSynchronize(s);
    cudaEventRecord(ws.ev_compute_done, s);
    g_last_error = msg;
    return st;
  }
  if ((e = cudaEventRecord(ws.ev_compute_done, s)) != cudaSuccess)
    return cuda_fail(e, "event record");
  if ((e = cudaStreamSynchronize(ws.d2h)) != cudaSuccess) return cuda_fail(e, "D2H sync");
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_fail(e, "stream sync");
  fill_stats(stats, *plan, shape, mask, valid_len);
  return TA_OK;
}

ta_status ta_release_workspace(int device) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return cuda_fail(e, "release workspace");
  }
  if (device < 0 || device >= n) return fail(TA_ERR_INVALID_ARGUMENT, "no such device");
  int prev = 0;
  cudaGetDevice(&prev);
  if ((e = cudaSetDevice(device)) != cudaSuccess) return cuda_fail(e, "release workspace");
  {
    Workspace& ws = workspace(device);
    std::lock_guard<std::mutex> lock(ws.mu);
    if (ws.h2d) cudaStreamSynchronize(ws.h2d);
    if (ws.d2h) cudaStreamSynchronize(ws.d2h);
    if (ws.ev_compute_done) cudaEventSynchronize(ws.ev_compute_done);
    if (ws.ptr) e = cudaFree(ws.ptr);
    ws.ptr = nullptr;
    ws.bytes = 0;
  }
  release_padding_pool(device);
  cudaSetDevice(prev);
  if (e != cudaSuccess) return cuda_fail(e, "release workspace");
  return TA_OK;
}

ta_status ta_debug_sdpa_trace(const void* q, const void* k, const void* v, void* o,
                              ta_shape shape, ta_dtype dtype, long long* trace, void* stream) {
  double eff = 0.0;
  ta_schedule sched = resolve_schedule(ta_schedule{0, 0, 0, 0});
  ta_status st = validate_common(shape, TA_MASK_NONE, nullptr, sched, 0, 0.0, &eff);
  if (st != TA_OK) return st;
  if ((st = validate_device_support(shape, dtype, TA_MASK_NONE)) != TA_OK) return st;
  if ((st = check_device()) != TA_OK) return st;
  auto plan = get_plan(sched, shape.d, dtype, false);
  if ((st = run_device(q, k, v, o, nullptr, shape, dtype, eff, *plan, stream, MaskArgs{},
                       trace)) != TA_OK)
    return st;
  cudaError_t e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "trace sync");
  return TA_OK;
}

ta_status ta_debug_exp2(const float* x, float* y, int64_t n, int mode, void* stream) {
  if (mode < 0 || mode > 1) return fail(TA_ERR_INVALID_ARGUMENT, "mode must be 0 or 1");
  if (n < 0 || (n > 0 && (!x || !y))) return fail(TA_ERR_INVALID_ARGUMENT, "x, y, n");
  ta_status st;
  if ((st = check_device()) != TA_OK) return st;
  cudaError_t e = ta::launch_exp2_unit(x, y, n, mode, stream);
  if (e != cudaSuccess) return cuda_fail(e, "exp2 unit launch");
  if ((e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream))) != cudaSuccess)
    return cuda_fail(e, "exp2 unit sync");
  return TA_OK;
}

ta_status ta_debug_umma_gemm(int mode, ta_dtype dtype, const void* a, const void* b, float* d,
                             void* stream) {
  if (mode < 0 || mode > 2) return fail(TA_ERR_INVALID_ARGUMENT, "mode must be 0, 1 or 2");
  if (dtype != TA_F16 && dtype != TA_BF16) return fail(TA_ERR_UNSUPPORTED, "dtype");
  ta_status st;
  if ((st = check_device()) != TA_OK) return st;
  CUtensorMap ma, mb;
  const bool bf16 = dtype == TA_BF16;
  if ((st = make_tmap(&ma, a, bf16, 1, 128, 128, 128)) != TA_OK) return st;
  if ((st = make_tmap(&mb, b, bf16, 1, 128, 128, 128)) != TA_OK) return st;
  cudaError_t e = ta::launch_umma_selftest(&ma, &mb, a, d, mode, bf16, stream);
  if (e != cudaSuccess) return cuda_fail(e, "selftest launch");
  if ((e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream))) != cudaSuccess)
    return cuda_fail(e, "selftest sync");
  return TA_OK;
}

}  // extern "C"
