// Host-side program planner for engine.compile_batch: SWAP-chain lowering and
// ASAP layering of a batch of programs (native so that batches of 10^3
// circuits x 10^3 gates plan in milliseconds, not seconds of Python).
//
// Lowering follows the reference's per-gate loop exactly (backends.py:47-60):
// a two-qubit gate on (q1, q2) with |q1 - q2| > 1 becomes the SWAP chain of
// MpsState.apply_two_qubit_routed (mps.py:138-157) -- SWAPs on hi-1 .. lo+1,
// the gate on (lo, lo+1) (as SWAP.G.SWAP when q1 > q2), SWAPs back on
// lo+1 .. hi-1. ASAP layering: an op's layer is one past the last layer of any
// op touching its sites, so ops sharing a site keep program order and ops in a
// layer are site-disjoint (they commute bit-exactly in Vidal form).
#include <stdint.h>

#include <vector>

#include "bmps.h"

namespace {

inline void expand_op(int8_t ar, int32_t q1, int32_t q2, int64_t src, int32_t state, int32_t* last,
                      int32_t* xs, int8_t* xa, int32_t* xq, int64_t* xsrc, int32_t* xl,
                      int64_t* xrec, int64_t& k, int64_t& rec) {
  auto put = [&](int8_t a, int32_t site, int64_t s) {
    int32_t L;
    if (a == 1) {
      L = last[site] + 1;
      last[site] = L;
    } else {
      L = (last[site] > last[site + 1] ? last[site] : last[site + 1]) + 1;
      last[site] = L;
      last[site + 1] = L;
    }
    xs[k] = state;
    xa[k] = a;
    xq[k] = site;
    xsrc[k] = s;
    xl[k] = L - 1;
    xrec[k] = a == 2 ? rec++ : -1;
    ++k;
  };
  if (ar == 1) {
    put(1, q1, src);
    return;
  }
  const int32_t lo = q1 < q2 ? q1 : q2, hi = q1 < q2 ? q2 : q1;
  for (int32_t s = hi - 1; s > lo; --s) put(2, s, -1);
  put(2, lo, q1 < q2 ? src : -src - 2);
  for (int32_t s = lo + 1; s < hi; ++s) put(2, s, -1);
}

}  // namespace

extern "C" {

int64_t bmps_plan_expanded_count(const int8_t* arity, const int32_t* q1, const int32_t* q2,
                                 int64_t nops) {
  int64_t k = 0;
  for (int64_t i = 0; i < nops; ++i) {
    if (arity[i] == 1) {
      ++k;
    } else {
      const int64_t d = q1[i] > q2[i] ? q1[i] - q2[i] : q2[i] - q1[i];
      k += d >= 1 ? 2 * d - 1 : 1;
    }
  }
  return k;
}

int32_t bmps_plan_build(int32_t nprogs, const int64_t* prog_off, const int32_t* prog_state,
                        const int8_t* arity, const int32_t* q1, const int32_t* q2, int32_t n,
                        int32_t* x_state, int8_t* x_arity, int32_t* x_site, int64_t* x_src,
                        int32_t* x_layer, int64_t* x_rec, int64_t* err_op) {
  if (nprogs < 0 || n < 1 || !prog_off || !err_op) return BMPS_E_ARG;
  *err_op = -1;
  std::vector<int32_t> last((size_t)n + 1);
  int64_t k = 0, rec = 0;
  for (int32_t p = 0; p < nprogs; ++p) {
    std::fill(last.begin(), last.end(), 0);
    for (int64_t i = prog_off[p]; i < prog_off[p + 1]; ++i) {
      const int32_t a = q1[i], b = arity[i] == 2 ? q2[i] : a;
      if (a < 0 || a >= n || b < 0 || b >= n) {
        *err_op = i;
        return BMPS_PLAN_E_SITE;
      }
      if (arity[i] == 2 && a == b) {
        *err_op = i;
        return BMPS_PLAN_E_SAME_SITE;
      }
      expand_op(arity[i], a, b, i, prog_state[p], last.data(), x_state, x_arity, x_site, x_src,
                x_layer, x_rec, k, rec);
    }
  }
  return BMPS_OK;
}

}  // extern "C"
