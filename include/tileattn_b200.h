/*
 * tileattn_b200.h — C-ABI of the B200-native SDPA forward operator.
 *
 * Drop-in for the reference hot path
 *     std::vector<float> tileattn::sdpa_tiled(const AttnInput&, const MaskSpec&,
 *         const ScaleSpec&, const TileSchedule&, PlanCache&, const TiledOptions&)
 *     (reference proj/include/tileattn/tiled.hpp:274-277, proj/src/tiled.cpp:253-272)
 * reduced to plain pointers and sizes so that any FFI (ctypes, cgo, JNI, a
 * C++ caller such as the reference's run_method, bench.cpp:130-142) can bind
 * it.  No torch or C++ types cross this boundary.
 *
 * Library: paper_2603_01960_b200/_lib/libtileattn_b200.so (sm_100a only).
 * See INTEGRATION.md for the reference-side bindings.
 */
#ifndef TILEATTN_B200_H_
#define TILEATTN_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TA_ABI_VERSION 1

#if defined(__GNUC__)
#define TA_API __attribute__((visibility("default")))
#else
#define TA_API
#endif

/* Status codes.  Mirror the reference's error channels:
 *   std::invalid_argument     (types.cpp:80-116)       -> TA_ERR_INVALID_ARGUMENT
 *   UnsupportedScheduleError  (tiled.cpp:29-35,42-43)  -> TA_ERR_UNSUPPORTED
 *   std::bad_alloc -> BenchStatus::Oom (bench.cpp:293-297) -> TA_ERR_OOM
 *   (new) CUDA runtime failure / no sm_100 device      -> TA_ERR_CUDA
 * The message of the last failure on the calling thread is ta_last_error(). */
typedef enum ta_status {
  TA_OK = 0,
  TA_ERR_INVALID_ARGUMENT = 1,
  TA_ERR_UNSUPPORTED = 2,
  TA_ERR_OOM = 3,
  TA_ERR_CUDA = 4
} ta_status;

/* DType (types.hpp:15).  The device path computes on 16-bit storage; F32 is
 * accepted by the validator and reported as TA_ERR_UNSUPPORTED. */
typedef enum ta_dtype { TA_F32 = 0, TA_F16 = 1, TA_BF16 = 2 } ta_dtype;

/* MaskKind (types.hpp:41-76). */
typedef enum ta_mask_kind { TA_MASK_NONE = 0, TA_MASK_CAUSAL = 1, TA_MASK_PADDING = 2 } ta_mask_kind;

/* TileLayout (tiled.hpp:21). */
typedef enum ta_layout { TA_LAYOUT_ROW = 0, TA_LAYOUT_COL = 1 } ta_layout;

/* TileSchedule (tiled.hpp:30-37): t_m in {16,32,64,128}, t_n in
 * {16,32,64,128,256}, stages in [1,4] — validated exactly like
 * schedule_supported (tiled.cpp:21-27).  On the GPU the values are a hint:
 * the executed tile (128-row UMMA tiles, 128-key K/V tiles, ring depth) is
 * reported in ta_kernel_stats.  All-zero = the reference default {64,128,2,row}. */
typedef struct ta_schedule {
  int32_t t_m;
  int32_t t_n;
  int32_t stages;
  int32_t layout;
} ta_schedule;

/* Shape (types.hpp:27-36): [B,H,S,D] row-major, D innermost.  The kernels
 * cover D a multiple of 8 up to 256 (D runs on the 64 / 128 / 192 / 256-column
 * instantiation that holds it, TMA zero-fill past D); other D ->
 * TA_ERR_UNSUPPORTED. */
typedef struct ta_shape {
  int64_t b, h, s, d;
} ta_shape;

/* KernelStats (tiled.hpp:247-257) plus the executed GPU tiling. */
typedef struct ta_kernel_stats {
  uint64_t kv_tiles_visited;  /* sum over 128-row query tiles of K/V tiles streamed */
  int32_t block_m;            /* executed rows per UMMA Q tile */
  int32_t block_n;            /* executed keys per K/V tile */
  int32_t stages;             /* executed smem ring depth (K and V tiles) */
  int32_t q_tiles_per_cta;    /* Q tiles ping-ponged per CTA */
  int64_t ctas;               /* CTAs launched */
  int32_t threads_per_cta;
  int32_t reserved;
} ta_kernel_stats;

/* ---------------------------------------------------------------------------
 * Device entry (the hot path).  Asynchronous on `stream` (a cudaStream_t; NULL
 * = legacy default stream); no implicit synchronisation, no allocation.
 *
 *   q, k, v : device, [B,H,S,D] contiguous, 16-bit (dtype), 16-B aligned
 *   o       : device, [B,H,S,D] contiguous, same dtype (finalize + RNE cvt,
 *             tiled.hpp:223-238, tiled.cpp:216-220)
 *   lse     : device, [B,H,S] fp32 natural-log log-sum-exp of the scaled
 *             scores (m + ln l); -inf for rows with no admitted key; NULL = skip
 *             (a NaN input propagates to the O and LSE of the rows whose
 *             scores it reaches, as the reference's arithmetic does; padded
 *             K/V rows (>= valid_len) never contribute, like the reference's
 *             zero-weight skip; one divergence: under the causal mask a NaN /
 *             inf in V at key k also reaches the rows of k's 128-key tile that
 *             precede k -- P V on the tensor core multiplies it by weight 0)
 *   valid_len : HOST array of B entries, MaskKind::Padding only (else NULL);
 *             B <= 32 travels in the kernel parameters, larger B through a
 *             per-device pool of pinned/device slots (allocated on first
 *             use, reused once the launch that read a slot has completed;
 *             not capturable in a CUDA graph: TA_ERR_UNSUPPORTED there)
 *   has_scale/scale : ScaleSpec (types.hpp:78-86); has_scale = 0 -> 1/sqrt(D)
 *   stats   : optional out-parameter (KernelStats analogue), may be NULL
 *
 * Validation order follows sdpa_tiled (tiled.cpp:256-259):
 *   shape -> mask -> schedule -> scale, then device-support checks.
 * ------------------------------------------------------------------------- */
TA_API ta_status ta_sdpa_fwd(const void* q, const void* k, const void* v, void* o, float* lse,
                      ta_shape shape, ta_dtype dtype, ta_mask_kind mask,
                      const int64_t* valid_len, int has_scale, double scale,
                      ta_schedule sched, void* stream, ta_kernel_stats* stats);

/* Host-buffer entry (the end-to-end path): q/k/v/o/lse are HOST pointers
 * (pinned for full PCIe bandwidth and for the chunked H2D / compute / D2H
 * overlap; pageable works, but each pageable copy blocks the host, which
 * serialises the pipeline).  Copies in, runs the device entry, copies O (and
 * LSE) back, and synchronises `stream`; on an error part-way every stream is
 * drained before returning.  Device workspace (4 tensors + LSE) is cached
 * per device and grown on demand; ta_release_workspace frees it. */
TA_API ta_status ta_sdpa_fwd_host(const void* q, const void* k, const void* v, void* o, float* lse,
                           ta_shape shape, ta_dtype dtype, ta_mask_kind mask,
                           const int64_t* valid_len, int has_scale, double scale,
                           ta_schedule sched, void* stream, ta_kernel_stats* stats);

/* Free the per-device workspace of ta_sdpa_fwd_host and the padding-length
 * pool (after draining their streams).  The next call re-allocates. */
TA_API ta_status ta_release_workspace(int device);

/* Validation only: the status ta_sdpa_fwd / ta_sdpa_fwd_host would return for
 * these arguments before touching any device (reference order shape -> mask ->
 * schedule -> scale, then what the sm_100a kernel covers).  Lets a harness
 * record status=unsupported rows (bench.cpp:290-292) without allocating. */
TA_API ta_status ta_sdpa_check(ta_shape shape, ta_dtype dtype, ta_mask_kind mask,
                               const int64_t* valid_len, int has_scale, double scale,
                               ta_schedule sched);

/* Thread-local message for the last non-OK status (exception what()). */
TA_API const char* ta_last_error(void);

/* TA_ABI_VERSION of the loaded library. */
TA_API int ta_abi_version(void);

/* schedule_supported (tiled.cpp:21-27): 1 if valid, else 0. */
TA_API int ta_schedule_supported(ta_schedule sched);

/* effective_scale (types.cpp:108-116).  Returns TA_ERR_INVALID_ARGUMENT for
 * d < 1 or an explicit scale <= 0. */
TA_API ta_status ta_effective_scale(int has_scale, double scale, int64_t d, double* out);

/* PlanCache counters (tiled.hpp:74-86): one process-wide cache keyed by
 * (t_m, t_n, D, dtype, causal). */
TA_API void ta_plan_cache_stats(uint64_t* hits, uint64_t* constructions);
TA_API void ta_plan_cache_clear(void);

/* 1 if `device` is an sm_100 part this library has code for, else 0. */
TA_API int ta_device_supported(int device);

/* Diagnostics: one 128x128x128 tcgen05 product checked by tests
 *   mode 0: d = a * b^T  (a [128][128] K-major, b [128 n][128 k] K-major)
 *   mode 1: d = a * b    (b [128 k][128 n] MN-major, SS operands)
 *   mode 2: d = a * b    (a staged in TMEM: TS-MMA)
 * a, b: device 16-bit; d: device fp32 [128][128].  Synchronous. */
TA_API ta_status ta_debug_umma_gemm(int mode, ta_dtype dtype, const void* a, const void* b, float* d,
                             void* stream);

/* Diagnostics: y[i] = 2^x[i] on the device with the softmax's exp2 units
 *   mode 0: ex2_poly2, the FMA-pipe emulation (tiled.hpp:94-118 fast_expf
 *           construction in base 2: round-to-nearest split, degree-3
 *           polynomial, exponent insertion by integer add)
 *   mode 1: MUFU ex2.approx.ftz
 * x, y: device fp32 [n].  Synchronous. */
TA_API ta_status ta_debug_exp2(const float* x, float* y, int64_t n, int mode, void* stream);

/* Diagnostics: run the forward once with a cycle-timeline trace of CTA (0,0):
 * trace (device, int64[24 * 64]) receives clock64 stamps per event and K/V
 * iteration (event ids: see TraceEvent in csrc/sdpa_fwd_sm100.h).  Synchronous. */
TA_API ta_status ta_debug_sdpa_trace(const void* q, const void* k, const void* v, void* o,
                                     ta_shape shape, ta_dtype dtype, long long* trace,
                                     void* stream);

#ifdef __cplusplus
}
#endif

#endif /* TILEATTN_B200_H_ */
