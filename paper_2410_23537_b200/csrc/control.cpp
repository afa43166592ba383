// Host control plane of the swap scheduler in C++ (SURVEY.md §8(f) row 1): EWT,
// the byte-budget swap planner and the rank -> plan step that drives the KV data
// plane.  Pure host code (no CUDA calls), compiled with -ffp-contract=off so every
// float64 operation rounds exactly as the reference's Python floats do.
//
//   alise_ewt_ms        <- kvmanager.py:276-294  ewt_ms
//   alise_plan_swaps    <- kvmanager.py:297-322  plan_swaps
//   alise_rank_and_plan <- simcore.py:439-462    _Run._ranked_with_grants
//                          (EWT over the global rank, regroup by level ordered by
//                          (EWT, rank position), skip in-flight jobs, plan)
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/alise_b200.h"

namespace alise {
int fail(int code, const char* fmt, ...);
}
using alise::fail;

namespace {

// Python's max(x, 0.0) / min(a, b): the first argument wins unless the second
// compares strictly greater / smaller (keeps the sign of a zero the same way).
inline double py_max0(double x) { return (0.0 > x) ? 0.0 : x; }
inline double py_min(double a, double b) { return (b < a) ? b : a; }

void ewt_core(int64_t n, const int32_t* level, const int64_t* last_promotion_us, const double* remaining_ms,
              double aging_ms, int64_t now_us, double* out) {
  const bool aging_on = !std::isinf(aging_ms);
  double ahead = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double promote = std::numeric_limits<double>::infinity();
    if (aging_on) {
      const double waited = (double)(now_us - last_promotion_us[i]) / 1000.0;
      promote = py_max0((double)level[i] * aging_ms - waited);
    }
    out[i] = py_min(ahead, promote);
    ahead += remaining_ms[i];
  }
}

// actions: 0 denied, 1 granted (resident or no transfer), 2 granted + upload,
// 3 denied + offload (kvmanager.py:310-321)
void plan_core(int64_t m, const int32_t* idx, const int32_t* residency, const int64_t* need, int64_t budget,
               int8_t* action) {
  int64_t used = 0;
  for (int64_t k = 0; k < m; ++k) {
    const int64_t i = idx ? idx[k] : k;
    if (used + need[i] <= budget) {
      used += need[i];
      action[k] = residency[i] == ALISE_RES_CPU ? 2 : 1;
    } else {
      action[k] = residency[i] == ALISE_RES_GPU ? 3 : 0;
    }
  }
}

}  // namespace

extern "C" int alise_ewt_ms(int64_t n, const int32_t* level, const int64_t* last_promotion_us,
                            const double* remaining_ms, double aging_ms, int64_t now_us, double* out_ewt_ms) {
  if (n < 0) return fail(ALISE_EINVAL, "negative job count");
  if (n > 0 && (!level || !last_promotion_us || !remaining_ms || !out_ewt_ms))
    return fail(ALISE_EINVAL, "null argument");
  ewt_core(n, level, last_promotion_us, remaining_ms, aging_ms, now_us, out_ewt_ms);
  return ALISE_OK;
}

extern "C" int alise_plan_swaps(int64_t n, const int32_t* residency, const int64_t* need_gpu_bytes,
                                int64_t budget_bytes, int8_t* out_action) {
  if (n < 0) return fail(ALISE_EINVAL, "negative entry count");
  if (n > 0 && (!residency || !need_gpu_bytes || !out_action)) return fail(ALISE_EINVAL, "null argument");
  plan_core(n, nullptr, residency, need_gpu_bytes, budget_bytes, out_action);
  return ALISE_OK;
}

extern "C" int alise_rank_and_plan(int64_t n, const int32_t* level, const int64_t* last_promotion_us,
                                   const double* remaining_ms, const int32_t* residency,
                                   const int64_t* need_gpu_bytes, double aging_ms, int64_t now_us,
                                   int64_t budget_bytes, double* out_ewt_ms, int32_t* out_order,
                                   int64_t* out_count, int8_t* out_action) {
  if (n < 0) return fail(ALISE_EINVAL, "negative job count");
  if (!out_count) return fail(ALISE_EINVAL, "null argument");
  if (n > 0 && (!level || !last_promotion_us || !remaining_ms || !residency || !need_gpu_bytes ||
                !out_ewt_ms || !out_order || !out_action))
    return fail(ALISE_EINVAL, "null argument");
  ewt_core(n, level, last_promotion_us, remaining_ms, aging_ms, now_us, out_ewt_ms);
  // levels ascending, then (EWT, rank position) within a level (simcore.py:444-450);
  // in-flight jobs are dropped before sorting (they are skipped after it)
  struct Key {
    int32_t level;
    double ewt;
    int32_t pos;
  };
  std::vector<Key> keys;
  keys.reserve((size_t)n);
  for (int64_t i = 0; i < n; ++i)
    if (residency[i] != ALISE_RES_UPLOADING && residency[i] != ALISE_RES_OFFLOADING)
      keys.push_back(Key{level[i], out_ewt_ms[i], (int32_t)i});
  std::sort(keys.begin(), keys.end(), [](const Key& a, const Key& b) {
    if (a.level != b.level) return a.level < b.level;
    if (a.ewt < b.ewt) return true;
    if (b.ewt < a.ewt) return false;
    return a.pos < b.pos;
  });
  int64_t m = 0;
  for (const Key& k : keys) out_order[m++] = k.pos;
  plan_core(m, out_order, residency, need_gpu_bytes, budget_bytes, out_action);
  *out_count = m;
  return ALISE_OK;
}
