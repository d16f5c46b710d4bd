// Persistence-directed cancellation of an extremum graph (SURVEY
// 8(f) f4).  The paper's tachyon runs it serially after the graph is built
// ("Their implementations in tachyon are serial in nature"), and so does this
// host-side pass over the last graph of a context: a min-priority queue of
// (cost, saddle id) with lazy cost updates (reading L20 in DESIGN.md):
//   cost(s) = min_{m adjacent} f(m) - f(s) for a simple saddle, f(second
//   highest adjacent maximum) - f(s) for a multi-saddle, never for a saddle
//   with one distinct maximum; costs are double differences of the f32 values;
//   pop s, recompute: above tau -> discard (s stays), above the top's cost ->
//   reinsert, else cancel -- every adjacent maximum but the highest (SoS order)
//   is merged into it (their arcs redirected, multiplicities added) and s and
//   the merged maxima leave the graph.  A minimum graph runs in the reversed
//   order (values negated, ties to the lower index).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <queue>
#include <utility>
#include <vector>

#include "eg_impl.h"

namespace eg {

void simplify_graph(int64_t n_max, const int64_t *maxima, const float *fmax, int64_t n_sad, const int64_t *saddles,
                    const int32_t *sbeta, const float *fsad, int64_t n_arc, const int64_t *arc_s,
                    const int64_t *arc_m, const int32_t *arc_mult, double tau, bool minimum, SimplifyResult &out) {
    const double sgn = minimum ? -1.0 : 1.0;
    // maxima by position in the ascending maxima list (binary search); saddles
    // by position in the ascending saddle list (arcs are sorted by saddle)
    auto mi = [&](int64_t id) { return int32_t(std::lower_bound(maxima, maxima + n_max, id) - maxima); };
    std::vector<double> mval(n_max);
    for (int64_t i = 0; i < n_max; ++i) mval[i] = sgn * double(fmax[i]);
    // SoS order of maxima: (value, id), the id reversed for a minimum graph
    auto higher = [&](int32_t a, int32_t b) {     // is maximum a above maximum b?
        if (mval[a] != mval[b]) return mval[a] > mval[b];
        return minimum ? maxima[a] < maxima[b] : maxima[a] > maxima[b];
    };
    std::vector<std::vector<std::pair<int32_t, int32_t>>> sarcs(n_sad);   // (max index, mult)
    std::vector<std::vector<int32_t>> by_max(n_max);                       // saddles adjacent to a maximum
    {
        int64_t j = 0;
        for (int64_t a = 0; a < n_arc; ++a) {
            while (j < n_sad && saddles[j] < arc_s[a]) ++j;
            const int32_t m = mi(arc_m[a]);
            sarcs[j].push_back({m, arc_mult[a]});
            by_max[m].push_back(int32_t(j));
        }
    }
    std::vector<char> sal(n_sad, 1), mal(n_max, 1);
    // cost: the second highest adjacent maximum (the lower one of two) minus
    // the saddle, in one pass over its distinct maxima
    auto cost = [&](int64_t j) -> double {
        const auto &v = sarcs[j];
        if (v.size() < 2) return INFINITY;
        int32_t t1 = v[0].first, t2 = -1;
        for (size_t k = 1; k < v.size(); ++k) {
            const int32_t m = v[k].first;
            if (higher(m, t1)) {
                t2 = t1;
                t1 = m;
            } else if (t2 < 0 || higher(m, t2)) {
                t2 = m;
            }
        }
        return mval[t2] - sgn * double(fsad[j]);
    };
    // (cost, saddle position): positions are in ascending id order, so ties
    // still go to the lower saddle id
    using Item = std::pair<double, int64_t>;
    std::vector<Item> init(static_cast<size_t>(n_sad));
    for (int64_t j = 0; j < n_sad; ++j) init[size_t(j)] = {cost(j), j};
    std::priority_queue<Item, std::vector<Item>, std::greater<Item>> pq(std::greater<Item>(), std::move(init));
    while (!pq.empty()) {
        const int64_t j = pq.top().second;
        pq.pop();
        const double c = cost(j);
        if (c > tau) continue;
        if (!pq.empty() && c > pq.top().first) {
            pq.push({c, j});
            continue;
        }
        // cancel: every maximum of s but the highest merges into the highest
        int32_t top = sarcs[j][0].first;
        for (const auto &p : sarcs[j])
            if (higher(p.first, top)) top = p.first;
        for (const auto &p : sarcs[j]) {
            const int32_t m = p.first;
            if (m == top) continue;
            for (int32_t s2 : by_max[m]) {
                if (s2 == int32_t(j) || !sal[s2]) continue;
                auto &v = sarcs[s2];
                int32_t mult = 0;
                for (size_t k = 0; k < v.size();)
                    if (v[k].first == m) {
                        mult += v[k].second;
                        v[k] = v.back();
                        v.pop_back();
                    } else {
                        ++k;
                    }
                if (!mult) continue;
                bool found = false;
                for (auto &q : v)
                    if (q.first == top) {
                        q.second += mult;
                        found = true;
                    }
                if (!found) {
                    v.push_back({top, mult});
                    by_max[top].push_back(s2);
                }
            }
            by_max[m].clear();
            mal[m] = 0;
        }
        sal[j] = 0;
        sarcs[j].clear();
    }
    out = SimplifyResult{};
    for (int64_t i = 0; i < n_max; ++i)
        if (mal[i]) out.maxima.push_back(maxima[i]);
    for (int64_t j = 0; j < n_sad; ++j) {
        if (!sal[j]) continue;
        out.saddles.push_back(saddles[j]);
        out.saddle_beta.push_back(sbeta[j]);
        std::vector<std::pair<int64_t, int32_t>> a;
        for (const auto &p : sarcs[j]) a.push_back({maxima[p.first], p.second});
        std::sort(a.begin(), a.end());
        for (const auto &p : a) {
            out.arc_s.push_back(saddles[j]);
            out.arc_m.push_back(p.first);
            out.arc_mult.push_back(p.second);
        }
    }
}

// f at the given node ids (device)
__global__ void k_gather_f(const float *__restrict__ f, int64_t f_base, const int64_t *__restrict__ ids, int64_t n,
                           float *out) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) out[i] = __ldg(f + (ids[i] - f_base));
}

cudaError_t launch_gather_f(const float *f, int64_t f_base, const int64_t *ids, int64_t n, float *out,
                            cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    k_gather_f<<<unsigned((n + 255) / 256), 256, 0, st>>>(f, f_base, ids, n, out);
    return cudaGetLastError();
}

}  // namespace eg
