// capi.cu — the C-ABI entry points (include/tb_pairwise.h): the runtime
// tile planner that replaces the reference's compile-time memory tiler
// (PassConfig pipeline.py:18-41, plan_split split.py:285-301) and the
// stream-ordered drivers of the kNN pipeline.
#include <cstring>
#include <cmath>
#include <string>
#include <mutex>
#include <cstdlib>
#include <vector>

#include "tb_common.cuh"
#include "knn_internal.h"

namespace tb {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

// B200: 148 SMs.  The planner is device-agnostic arithmetic (it must run on
// a CPU-only host for tests and dry planning); the run checks the device.
constexpr int kPlanSms = 148;
constexpr int64_t kAlign = 256;
// engine chosen for TB_ENGINE_AUTO: the fp16 single pass with the measured-
// residual bound (tc1) certifies C2/C3 with no fallback at 1/3 of tc3's MMAs
constexpr int kAutoEngine = TB_ENGINE_TC1;

static int64_t elem_size(int dtype) { return dtype == TB_F32 ? 4 : 8; }

// Lowest-cost slice count for a grid of `qt` query tiles x S slices over
// `tiles` row tiles: minimise waves * tiles-per-slice; ties -> fewer slices.
static int choose_slices(int64_t qt, int64_t tiles, int ctas_per_sm, int max_slices) {
  const int64_t conc = (int64_t)kPlanSms * ctas_per_sm;
  int best = 1;
  int64_t best_cost = INT64_MAX;
  const int64_t smax = std::min<int64_t>(std::max<int64_t>(tiles, 1), max_slices);
  for (int64_t s = 1; s <= smax; ++s) {
    const int64_t waves = ceil_div(qt * s, conc);
    const int64_t per = ceil_div(tiles, s);
    const int64_t cost = waves * per;
    if (cost < best_cost) {
      best_cost = cost;
      best = (int)s;
    }
  }
  return best;
}

struct Carve {
  int64_t used = 0;
  int64_t take(int64_t bytes) {
    const int64_t o = used;
    used += round_up(std::max<int64_t>(bytes, 0), kAlign);
    return o;
  }
};

static bool device_is_sm100(std::string* why) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    *why = "no CUDA device visible";
    return false;
  }
  int major = 0, minor = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  if (major != 10 || minor != 0) {
    *why = "this library is built for sm_100a (B200); device is sm_" +
           std::to_string(major) + std::to_string(minor);
    return false;
  }
  return true;
}

}  // namespace tb

using namespace tb;

// tb_knn_run_ex body; `ready[c]` (if given) gates database chunk c
static int knn_run_impl(const tb_knn_plan* p, const void* x, const void* q,
                        int64_t index_base, void* out_dist, int64_t* out_idx,
                        void* workspace, int64_t workspace_bytes, cudaStream_t st,
                        void** events, int32_t n_events, void** ready, int32_t n_ready);

namespace tb {
int set_smem_once(const void* kernel, int bytes) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<const void*, int>, int>> done;   // (kernel, dev) -> bytes
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  for (auto& e : done)
    if (e.first.first == kernel && e.first.second == dev) {
      if (e.second >= bytes) return TB_OK;
      TB_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
      e.second = bytes;
      return TB_OK;
    }
  TB_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done.push_back({{kernel, dev}, bytes});
  return TB_OK;
}
}  // namespace tb

// Per-device copy stream and event pool of tb_knn_run_host, created on first
// use and kept for the process (stream and event creation are driver round
// trips; the pool is held only while one call enqueues its work).
struct HostCopyRes {
  cudaStream_t stream = nullptr;
  std::vector<cudaEvent_t> events;
};
static std::mutex g_copy_mu;
static HostCopyRes g_copy_res[64];

extern "C" {

const char* tb_last_error(void) { return g_last_error.c_str(); }

int32_t tb_capabilities(void) {
  return (1 << 16) | 0x1 | 0x2 | 0x4 | 0x8;
}

int tb_knn_plan_create(int64_t n, int64_t m, int64_t d, int64_t k, int32_t metric,
                int32_t dtype, int32_t out_dtype, int32_t engine,
                int64_t memory_limit, int64_t resident_bytes,
                tb_knn_plan* plan) {
  return tb_knn_plan_create_ex(n, m, d, k, metric, dtype, out_dtype, engine, memory_limit,
                               resident_bytes, 0, plan);
}

int tb_knn_plan_create_ex(int64_t n, int64_t m, int64_t d, int64_t k, int32_t metric,
                          int32_t dtype, int32_t out_dtype, int32_t engine,
                          int64_t memory_limit, int64_t resident_bytes,
                          int64_t max_chunk_rows, tb_knn_plan* plan) {
  if (!plan) return fail(TB_ERR_ARG, "plan pointer is null");
  std::memset(plan, 0, sizeof(*plan));
  if (n < 1 || d < 1 || m < 0)
    return fail(TB_ERR_ARG, "n and d must be at least 1 and m non-negative");
  if (k < 1 || k > n)
    return fail(TB_ERR_ARG, "k=" + std::to_string(k) +
                                " must satisfy 1 <= k <= n=" + std::to_string(n));
  if (metric != TB_METRIC_L2 && metric != TB_METRIC_L1 && metric != TB_METRIC_COSINE)
    return fail(TB_ERR_ARG, "metric must be one of ('l2', 'l1', 'cosine')");
  if ((dtype != TB_F32 && dtype != TB_F64) || (out_dtype != TB_F32 && out_dtype != TB_F64))
    return fail(TB_ERR_ARG, "unsupported dtype; only f32/f64 tensors exist");
  if (n >= (int64_t)INT_MAX - 1 || m >= (int64_t)INT_MAX)
    return fail(TB_ERR_UNSUPPORTED, "shard extents must be < 2^31 rows");
  // l1 has no tensor-core form (CUDA-core engine); cosine runs on the
  // tensor-core engines over unit-normalised rows
  if (engine == TB_ENGINE_AUTO)
    engine = metric == TB_METRIC_L1 ? TB_ENGINE_SIMT
             : round_up(d, 64) <= tc_max_dpad() || metric == TB_METRIC_COSINE ? kAutoEngine
                                                                            : TB_ENGINE_SIMT;
  if (engine != TB_ENGINE_TC3 && engine != TB_ENGINE_SIMT && engine != TB_ENGINE_TC1)
    return fail(TB_ERR_ARG, "unknown engine");
  if (metric == TB_METRIC_L1 && engine != TB_ENGINE_SIMT)
    return fail(TB_ERR_UNSUPPORTED, "l1 has no tensor-core form: use engine 'simt' or 'auto'");
  if (metric == TB_METRIC_COSINE && engine == TB_ENGINE_SIMT)
    return fail(TB_ERR_UNSUPPORTED, "cosine runs on the tensor-core engines ('tc3', 'tc1')");
  const bool tc = engine != TB_ENGINE_SIMT;
  if (tc && round_up(d, 64) > tc_max_dpad())
    return fail(TB_ERR_UNSUPPORTED, "tcgen05 engines support d <= " +
                                        std::to_string(tc_max_dpad()));

  // candidates kept beyond k: the single-pass engine and long (d > 128)
  // contractions have wider certified error bounds, so they keep more
  const int64_t margin = round_up(d, 64) > 128 && engine != TB_ENGINE_SIMT ? 22 : 6;
  const int64_t want = k + margin;
  int cand = want <= 16 ? 16 : want <= 32 ? 32 : want <= 64 ? 64 : 0;
  if (!cand) {
    if (k <= 64) cand = 64;
    else return fail(TB_ERR_UNSUPPORTED, "k > 64 is not supported by the register top-k engines");
  }

  plan->n = n; plan->m = m; plan->d = d; plan->k = k;
  plan->metric = metric; plan->dtype = dtype; plan->out_dtype = out_dtype;
  plan->engine = engine; plan->cand = cand;
  plan->memory_limit = memory_limit; plan->resident_bytes = resident_bytes;
  const int64_t qt = ceil_div(std::max<int64_t>(m, 1), 128);
  plan->m_pad = qt * 128;
  plan->d_pad = tc ? round_up(d, 64) : d;
  plan->output_bytes = m * k * (elem_size(out_dtype) + 8);
  // what the caller's allocator charges: dist and idx are two buffers
  const int64_t out_charged = alloc_bytes(m * k * elem_size(out_dtype)) + alloc_bytes(m * k * 8);

  const int tile_rows = tc ? 256 : 128;
  const int ctas_per_sm = 1;
  const int passes = engine == TB_ENGINE_TC1 ? 1 : 3;

  auto layout = [&](int64_t chunk_rows, int slices) -> int64_t {
    Carve c;
    const int64_t chunk_pad = round_up(chunk_rows, tile_rows);
    const int64_t last = n - (ceil_div(n, chunk_rows) - 1) * chunk_rows;
    const int64_t lists =
        tc ? std::max(tc_lists(m, chunk_pad, kPlanSms, passes, plan->d_pad),
                      tc_lists(m, round_up(last, tile_rows), kPlanSms, passes, plan->d_pad))
           : 2 * (int64_t)slices;
    plan->off[kQn64] = c.take(m * 8);
    plan->off[kQnorm] = c.take(m * 4);
    // counters | tc1 centring mean [d] + per-block partials [64][d + 1]
    plan->off[kStats] = c.take(256 + 8 * (plan->d_pad + 64 * (plan->d_pad + 1)));
    plan->off[kFbList] = c.take(fb_region_bytes(m));
    plan->off[kXn] = c.take(chunk_pad * 4);
    plan->off[kCandS] = c.take(lists * m * cand * 4);
    plan->off[kCandI] = c.take(lists * m * cand * 4);
    plan->off[kRunS] = c.take(2 * m * cand * 4);
    plan->off[kRunI] = c.take(2 * m * cand * 4);
    plan->off[kGThr] = c.take(tc_gthr_words(m, cand) * 4);   // thresholds + insertion pools
    if (tc) {
      // tc1 (fp16 single pass) stages one plane per operand
      const int64_t lo = engine == TB_ENGINE_TC1 ? 0 : 1;
      plan->off[kQHi] = c.take(plan->m_pad * plan->d_pad * 2);
      plan->off[kQLo] = c.take(lo * plan->m_pad * plan->d_pad * 2);
      plan->off[kXHi] = c.take(chunk_pad * plan->d_pad * 2);
      plan->off[kXLo] = c.take(lo * chunk_pad * plan->d_pad * 2);
      plan->off[kXExt] = c.take(chunk_pad * 32);
      plan->off[kQln] = c.take(m * 4);
    }
    return c.used;
  };

  const int64_t limit = memory_limit > 0 ? memory_limit : INT64_MAX;
  int64_t chunk = tc ? std::min<int64_t>(n, (int64_t)1 << 22) : n;
  int64_t min_chunk = std::min<int64_t>(n, tile_rows);
  if (max_chunk_rows > 0)   // a strict cap (whole tiles below it), at least one tile
    chunk = std::max(min_chunk,
                     std::min(chunk, std::max<int64_t>(tile_rows, max_chunk_rows / tile_rows * tile_rows)));
  for (;;) {
    const int64_t tiles = ceil_div(chunk, tile_rows);
    int slices = tc ? 1 : choose_slices(qt, tiles, ctas_per_sm, 512);
    int64_t ws = layout(chunk, slices);
    // shrink the candidate fan-out before the chunk if that is what breaks the limit
    while (resident_bytes + alloc_bytes(ws) + out_charged > limit && slices > 1) {
      slices = std::max(1, slices / 2);
      ws = layout(chunk, slices);
    }
    if (resident_bytes + alloc_bytes(ws) + out_charged <= limit) {
      plan->chunk_rows = chunk;
      plan->n_chunks = ceil_div(n, chunk);
      plan->slices = slices;
      plan->workspace_bytes = ws;
      plan->peak_bytes = resident_bytes + alloc_bytes(ws) + out_charged;
      return TB_OK;
    }
    if (chunk <= min_chunk) {
      const int64_t need = resident_bytes + alloc_bytes(ws) + out_charged;
      return fail(TB_ERR_BUDGET,
                  "knn: allocating " + std::to_string(ws + plan->output_bytes) +
                      " bytes would exceed the budget (live=" +
                      std::to_string(resident_bytes) + ", limit=" +
                      std::to_string(memory_limit) + ", smallest plan needs " +
                      std::to_string(need) + ")");
    }
    chunk = std::max<int64_t>(min_chunk, round_up(chunk / 2, tile_rows));
  }
}

int tb_knn_run(const tb_knn_plan* p, const void* x, const void* q,
               int64_t index_base, void* out_dist, int64_t* out_idx,
               void* workspace, int64_t workspace_bytes, void* stream) {
  return tb_knn_run_ex(p, x, q, index_base, out_dist, out_idx, workspace,
                       workspace_bytes, stream, nullptr, 0);
}

int tb_knn_run_ex(const tb_knn_plan* p, const void* x, const void* q,
                  int64_t index_base, void* out_dist, int64_t* out_idx,
                  void* workspace, int64_t workspace_bytes, void* stream,
                  void** events, int32_t n_events) {
  return knn_run_impl(p, x, q, index_base, out_dist, out_idx, workspace, workspace_bytes,
                      (cudaStream_t)stream, events, n_events, nullptr, 0);
}

int tb_knn_run_host(const tb_knn_plan* p, const void* x_host, const void* q_host,
                    int64_t index_base, void* dist_host, int64_t* idx_host, void* x_dev,
                    void* q_dev, void* dist_dev, int64_t* idx_dev, void* workspace,
                    int64_t workspace_bytes, void* stream) {
  if (!p) return fail(TB_ERR_ARG, "plan pointer is null");
  if (!x_host || !q_host || !dist_host || !idx_host || !x_dev || !q_dev || !dist_dev || !idx_dev)
    return fail(TB_ERR_ARG, "null buffer passed to tb_knn_run_host");
  if (p->m == 0) return TB_OK;
  std::string why;
  if (!device_is_sm100(&why)) return fail(TB_ERR_NO_DEVICE, why);
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t es = elem_size(p->dtype);
  // database chunk c is copied on a side stream; chunk c's compute waits only
  // for its own rows, so chunk c+1's host->device copy overlaps chunk c
  int dev = 0;
  TB_CUDA_TRY(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return fail(TB_ERR_ARG, "device ordinal out of range");
  std::lock_guard<std::mutex> lock(g_copy_mu);
  HostCopyRes& res = g_copy_res[dev];
  if (!res.stream) TB_CUDA_TRY(cudaStreamCreateWithFlags(&res.stream, cudaStreamNonBlocking));
  while (res.events.size() < (size_t)p->n_chunks + 1) {
    cudaEvent_t e;
    TB_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    res.events.push_back(e);
  }
  cudaStream_t cp = res.stream;
  std::vector<cudaEvent_t> ready(res.events.begin(), res.events.begin() + p->n_chunks + 1);
  int rc = TB_OK;
  {
    // the copy stream starts after the caller's prior work on `stream`
    cudaEventRecord(ready[p->n_chunks], st);
    cudaStreamWaitEvent(cp, ready[p->n_chunks], 0);
    // the queries go first on the SAME copy stream: host->device copies of
    // two streams share one copy engine, and a query copy queued on `st`
    // could be scheduled behind every database chunk (no overlap at all)
    cudaMemcpyAsync(q_dev, q_host, p->m * p->d * es, cudaMemcpyHostToDevice, cp);
    cudaEventRecord(ready[p->n_chunks], cp);
    cudaStreamWaitEvent(st, ready[p->n_chunks], 0);
    for (int64_t c = 0; c < p->n_chunks; ++c) {
      const int64_t c0 = c * p->chunk_rows, rows = std::min(p->chunk_rows, p->n - c0);
      cudaMemcpyAsync((char*)x_dev + c0 * p->d * es, (const char*)x_host + c0 * p->d * es,
                      rows * p->d * es, cudaMemcpyHostToDevice, cp);
      cudaEventRecord(ready[c], cp);
    }
    std::vector<void*> rv(ready.begin(), ready.end());
    rc = knn_run_impl(p, x_dev, q_dev, index_base, dist_dev, idx_dev, workspace,
                      workspace_bytes, st, nullptr, 0, rv.data(), (int32_t)p->n_chunks);
    if (rc == TB_OK) {
      cudaMemcpyAsync(dist_host, dist_dev, p->m * p->k * elem_size(p->out_dtype),
                      cudaMemcpyDeviceToHost, st);
      cudaMemcpyAsync(idx_host, idx_dev, p->m * p->k * 8, cudaMemcpyDeviceToHost, st);
      const cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) rc = fail(TB_ERR_CUDA, std::string("tb_knn_run_host: ") +
                                                       cudaGetErrorString(e));
    }
  }
  return rc;
}

}  // extern "C"

static int knn_run_impl(const tb_knn_plan* p, const void* x, const void* q,
                        int64_t index_base, void* out_dist, int64_t* out_idx,
                        void* workspace, int64_t workspace_bytes, cudaStream_t st,
                        void** events, int32_t n_events, void** ready, int32_t n_ready) {
  if (!p) return fail(TB_ERR_ARG, "plan pointer is null");
  if (p->m == 0) return TB_OK;
  if (!x || !q || !out_dist || !out_idx || !workspace)
    return fail(TB_ERR_ARG, "null buffer passed to tb_knn_run");
  // the row kernels read x and q with 16-byte vector loads; a misaligned
  // view (e.g. buf[1:] of a float tensor) would fault the whole context
  if (((uintptr_t)x | (uintptr_t)q) & 15)
    return fail(TB_ERR_ARG, "x and q must be 16-byte aligned (copy the view into a fresh buffer)");
  if (workspace_bytes < p->workspace_bytes)
    return fail(TB_ERR_ARG, "workspace smaller than plan->workspace_bytes");
  std::string why;
  if (!device_is_sm100(&why)) return fail(TB_ERR_NO_DEVICE, why);
  char* ws = (char*)workspace;
  auto at = [&](int slot) { return ws + p->off[slot]; };
  double* qn64 = (double*)at(kQn64);
  float* qnorm = (float*)at(kQnorm);
  unsigned* stats = (unsigned*)at(kStats);
  int* fb = (int*)at(kFbList);
  float* xn = (float*)at(kXn);
  float* cs = (float*)at(kCandS);
  int* ci = (int*)at(kCandI);
  float* rs[2] = {(float*)at(kRunS), (float*)at(kRunS) + p->m * p->cand};
  int* ri[2] = {(int*)at(kRunI), (int*)at(kRunI) + p->m * p->cand};
  const bool tc = p->engine != TB_ENGINE_SIMT;
  __nv_bfloat16* qhi = tc ? (__nv_bfloat16*)at(kQHi) : nullptr;
  __nv_bfloat16* qlo = tc ? (__nv_bfloat16*)at(kQLo) : nullptr;
  __nv_bfloat16* xhi = tc ? (__nv_bfloat16*)at(kXHi) : nullptr;
  __nv_bfloat16* xlo = tc ? (__nv_bfloat16*)at(kXLo) : nullptr;
  uint8_t* xext = tc ? (uint8_t*)at(kXExt) : nullptr;
  const int64_t es = elem_size(p->dtype);
  const int tile_rows = tc ? 256 : 128;
  unsigned* gthr = (unsigned*)at(kGThr);

  TB_CUDA_TRY(cudaMemsetAsync(stats, 0, 256, st));
  if (tc) TB_CUDA_TRY(cudaMemsetAsync(gthr, 0xFF, tc_gthr_words(p->m, p->cand) * 4, st));
  const bool f16 = p->engine == TB_ENGINE_TC1;
  float* qln = f16 ? (float*)at(kQln) : nullptr;
  const float* f16p = f16 ? reinterpret_cast<const float*>(stats + kF16Slot) : nullptr;
  int rc = TB_OK;
  // the query prep of tc1 follows the centring decision, which reads the
  // first database rows: it runs once chunk 0 is on the device
  auto query_prep = [&]() -> int {
    if (tc && p->metric == TB_METRIC_L2) {
      const int64_t rows0 = std::min(p->chunk_rows, p->n);
      int r0 = launch_f16_center(p->dtype, x, rows0, p->d, stats, st);
      if (r0) return r0;
    }
    return f16 ? launch_query_prep_f16(p->dtype, p->metric, q, p->m, p->d, qn64, qnorm, qln,
                                       stats, (__half*)qhi, p->m_pad, p->d_pad, st)
               : launch_query_prep(p->dtype, p->metric, q, p->m, p->d, qn64, qnorm, qhi, qlo,
                                   p->m_pad, p->d_pad, st, tc ? stats : nullptr);
  };

  const float* prev_s = nullptr;
  const int* prev_i = nullptr;
  int flip = 0;
  for (int64_t c = 0; c < p->n_chunks; ++c) {
    const int64_t c0 = c * p->chunk_rows;
    const int64_t rows = std::min(p->chunk_rows, p->n - c0);
    const int64_t rows_pad = round_up(rows, tile_rows);
    const char* xc = (const char*)x + c0 * p->d * es;
    if (ready && c < n_ready) TB_CUDA_TRY(cudaStreamWaitEvent(st, (cudaEvent_t)ready[c], 0));
    if (c == 0 && (rc = query_prep())) return rc;
    rc = f16 ? launch_db_prep_f16(p->dtype, p->metric, xc, rows, p->d, xn, stats,
                                  (__half*)xhi, rows_pad, p->d_pad, xext, st)
             : launch_db_prep(p->dtype, p->metric, xc, rows, p->d, xn, stats, xhi, xlo,
                              rows_pad, p->d_pad, xext, st);
    if (rc) return rc;
    const int slices = (int)std::min<int64_t>(p->slices, ceil_div(rows, tile_rows));
    int lists = tc ? tc_lists(p->m, rows_pad, kPlanSms, p->engine == TB_ENGINE_TC1 ? 1 : 3, p->d_pad)
                   : slices * 2;
    const bool prof = events && 2 * c + 1 < n_events;
    if (prof) TB_CUDA_TRY(cudaEventRecord((cudaEvent_t)events[2 * c], st));
    if (tc) {
      rc = launch_knn_tc(p->engine == TB_ENGINE_TC1 ? 1 : 3, p->cand, xhi, xlo,
                         qhi, qlo, xext, rows, rows_pad, p->m, p->m_pad, p->d_pad,
                         lists, (int)c0, cs, ci, gthr, f16p, st);
    } else {
      rc = launch_knn_simt(p->dtype, p->metric, p->cand, xc, q, xn, rows, p->m, p->d,
                           slices, (int)c0, cs, ci, st);
    }
    if (rc) return rc;
    if (prof) TB_CUDA_TRY(cudaEventRecord((cudaEvent_t)events[2 * c + 1], st));
    rc = launch_knn_merge(p->cand, cs, ci, lists, prev_s, prev_i, p->m,
                          rs[flip], ri[flip], st);
    if (rc) return rc;
    prev_s = rs[flip];
    prev_i = ri[flip];
    flip ^= 1;
  }

  // error-bound coefficients of the approximate score
  const double u24 = std::ldexp(1.0, -24);
  double dot_rel;
  if (p->engine == TB_ENGINE_SIMT)
    dot_rel = (double)(p->d + 4) * u24 * (p->dtype == TB_F64 ? 2.0 : 1.0) + 2 * u24;
  else if (p->engine == TB_ENGINE_TC3)
    dot_rel = 4.0 * std::ldexp(1.0, -16) + (double)(3 * p->d_pad + 16) * 2 * u24;
  else  // tc1: fp32 accumulation only; the fp16 rounding enters through the
        // measured residual norms (refine kernel, qln + stats[2])
    dot_rel = (double)(p->d_pad + 32) * u24;
  double c1 = 2.0 * 2.0 * dot_rel;   // 2x safety, 2 for the -2 q.x
  double c2 = 2.0 * 4.0 * u24;        // ||x||^2 rounding + final FMA
  // tc1: ||x||^2 enters the fp32 sum too, and its fp16 split comes from the
  // fp32 norms (relative error <= (d + 2) 2^-24)
  if (f16) c2 += 2.0 * dot_rel + std::ldexp(1.0, -26) + 2.0 * (double)(p->d + 2) * u24;
  if (p->metric == TB_METRIC_L1) {
    // fp32 sum of d non-negative |q-x| terms: relative (d+2)u, plus the
    // rounding of f64 inputs to fp32, u (|q|_1 + |x|_1); 2x safety
    c1 = 2.0 * (double)(p->d + 2) * u24;
    c2 = p->dtype == TB_F64 ? 2.0 * u24 : 0.0;
  }
  // test hook: make every query uncertified to exercise the exact fallback
  if (const char* f = std::getenv("TB_FORCE_FALLBACK"))
    if (f[0] == '1') c1 = c2 = 1e300;
  rc = launch_knn_refine(p->dtype, p->out_dtype, p->metric, p->cand, prev_s, prev_i, x, q,
                         qn64, qnorm, qln, stats, p->n, p->m, p->d, p->k, c1, c2,
                         out_dist, out_idx, index_base, fb, st);
  if (rc) return rc;
  // everything the planner placed from kXn on (norms, candidate and running
  // lists, thresholds, operand and chunk staging) is dead once the re-rank
  // has run: the fallback uses it as scratch (its hit buffers need room on
  // clustered data, where a query's bound can enclose hundreds of rows)
  return launch_knn_fallback(p->dtype, p->out_dtype, p->metric, x, q, p->n, p->m, p->d, p->k, stats, fb,
                             at(kXn), p->workspace_bytes - p->off[kXn], out_dist, out_idx,
                             index_base, st);
}

extern "C" {

int tb_knn_fallback_count(const tb_knn_plan* p, const void* workspace,
                          void* stream, int64_t* count) {
  if (!p || !workspace || !count) return fail(TB_ERR_ARG, "null argument");
  int v = 0;
  const char* ws = (const char*)workspace;
  TB_CUDA_TRY(cudaMemcpyAsync(&v, ws + p->off[kStats] + 4, 4, cudaMemcpyDeviceToHost,
                              (cudaStream_t)stream));
  TB_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
  *count = v;
  return TB_OK;
}

int tb_knn_check(const tb_knn_plan* p, const void* workspace, void* stream) {
  if (!p || !workspace) return fail(TB_ERR_ARG, "null argument");
  if (p->metric != TB_METRIC_COSINE) return TB_OK;
  unsigned v = 0;
  const char* ws = (const char*)workspace;
  TB_CUDA_TRY(cudaMemcpyAsync(&v, ws + p->off[kStats] + 4 * kZeroRowWord, 4,
                              cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  TB_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
  return v ? fail(TB_ERR_ARG, "cosine distance is undefined for zero rows") : TB_OK;
}

int tb_topk_merge(const void* dist_lists, const int64_t* idx_lists,
                  int32_t n_lists, int64_t m, int64_t k, int32_t dtype,
                  void* out_dist, int64_t* out_idx, void* stream) {
  if (n_lists < 1 || k < 1 || m < 0) return fail(TB_ERR_ARG, "bad merge shape");
  if (dtype != TB_F32 && dtype != TB_F64) return fail(TB_ERR_ARG, "bad dtype");
  if (m == 0) return TB_OK;
  std::string why;
  if (!device_is_sm100(&why)) return fail(TB_ERR_NO_DEVICE, why);
  return launch_topk_merge(dist_lists, idx_lists, n_lists, m, k, dtype,
                           out_dist, out_idx, (cudaStream_t)stream);
}

}  // extern "C"
