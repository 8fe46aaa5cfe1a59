// splitters.cpp -- host port of the skew-resilient splitter search.
//
// Restates skew._minmax_contiguous (/root/reference/pkg/src/mpsm/skew.py
// 180-273) with the cost of skew.compute_splitters (skew.py:302-304,
// split_relevant_cost skew.py:148-153).  The reference runs this in Python
// (~15 ms at B=10, T=8, SURVEY.md finding 6) on the critical path between the
// public sort and the private scatter; here it is microseconds.
//
// Bit-identical bounds: seg_cost uses libm log2 exactly like Python's
// math.log2 and the same operation order; the candidate bound values the
// reference derives with numpy (np.log2 differs from libm log2 in the last ulp
// for some inputs) are computed by the caller with numpy and passed in.
//
// One deliberate difference: the reference raises ValueError when float
// rounding in the CDF makes a bucket span negative by ~1e-13 (skew.py:150-151;
// reproduced by tests/golden "dup_heavy", T=3).  We clamp such spans at 0.

#include <cmath>
#include <cstdint>
#include <vector>

#include "../../include/mpsm_b200.h"

namespace {

struct Costs {
    int64_t n;
    int t;
    const int64_t* prefix;
    const double* edge;
    double seg(int64_t a, int64_t b) const {
        int64_t size = prefix[b] - prefix[a];
        double span = edge[b] - edge[a];
        if (span < 0) span = 0.0;
        double c = size > 0 ? (double)size * std::log2((double)size) : 0.0;
        c = c + (double)((int64_t)t * size);
        return c + span;
    }
    int64_t max_extend(int64_t a, double bound) const {
        int64_t lo = a + 1, hi = n;
        while (lo < hi) {
            int64_t mid = (lo + hi + 1) / 2;
            if (seg(a, mid) <= bound) lo = mid;
            else hi = mid - 1;
        }
        return lo;
    }
    bool feasible(double bound) const {
        if (seg(0, 1) > bound) return false;
        int64_t a = 0;
        int parts = 0;
        while (a < n) {
            if (seg(a, a + 1) > bound) return false;
            a = max_extend(a, bound);
            if (++parts > t) return false;
        }
        return true;
    }
};

}  // namespace

extern "C" int mpsm_minmax_contiguous(int64_t n, int t, const int64_t* prefix, const double* edge_cdf,
                                      const double* cand, int64_t ncand, int64_t* out_bounds) {
    if (n < 1 || t < 1 || !prefix || !edge_cdf || !out_bounds) return MPSM_ERR_ARG;
    if (t > n) return MPSM_ERR_CONFIG;
    if (t == 1) {
        out_bounds[0] = 0;
        out_bounds[1] = n;
        return MPSM_OK;
    }
    Costs C{n, t, prefix, edge_cdf};
    double best;
    if (n <= 256) {  // exact search over the sorted unique candidate costs
        if (ncand < 1) return MPSM_ERR_ARG;
        int64_t lo = 0, hi = ncand - 1;
        while (lo < hi) {
            int64_t mid = (lo + hi) / 2;
            if (C.feasible(cand[mid])) hi = mid;
            else lo = mid + 1;
        }
        best = cand[lo];
    } else {  // float bisection; cand = the n single-bucket costs
        if (ncand < 1) return MPSM_ERR_ARG;
        double lo_c = cand[0];
        for (int64_t i = 1; i < ncand; ++i)
            if (cand[i] > lo_c || std::isnan(lo_c)) lo_c = cand[i];
        double hi_c = C.seg(0, n);
        for (int it = 0; it < 80; ++it) {
            double mid = 0.5 * (lo_c + hi_c);
            if (C.feasible(mid)) hi_c = mid;
            else lo_c = mid;
            if (hi_c - lo_c <= 1e-9 * std::fmax(1.0, std::fabs(hi_c))) break;
        }
        best = hi_c;
    }
    std::vector<int64_t> jump(n), g(n + 1, 0);
    for (int64_t a = 0; a < n; ++a) jump[a] = C.max_extend(a, best);
    for (int64_t a = n - 1; a >= 0; --a) g[a] = 1 + g[jump[a]];
    out_bounds[0] = 0;
    int64_t a = 0;
    for (int p = 1; p < t; ++p) {
        int remaining = t - p;
        int64_t e = a + 1, limit = n - remaining;
        while (e <= limit) {
            if (C.seg(a, e) <= best && g[e] <= remaining) break;
            ++e;
        }
        if (e > limit) return MPSM_ERR_INTERNAL;
        out_bounds[p] = e;
        a = e;
    }
    out_bounds[t] = n;
    return MPSM_OK;
}
