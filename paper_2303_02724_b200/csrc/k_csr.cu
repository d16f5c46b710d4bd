// CSR neighbourhood-graph kernels (reading L14: the link of v is the subgraph
// induced on N(v)).  S1: gradient = highest upper neighbour; S3:
// beta0+ = components of the induced upper link by union-find over
// the link edges, which are found by merging the sorted lists N(a) and U(v);
// a saddle's component representatives are stored by classify (in its own
// row range of a row_ptr-indexed buffer), so S4 only gathers their labels.
// One warp per vertex (k_classify_csr); no degree cap.
#include <algorithm>
#include <cstdlib>

#include "eg_impl.h"

namespace eg {

__device__ __forceinline__ bool csr_higher(int32_t u, float fu, int32_t v, float fv) {
    return fu > fv || (fu == fv && u > v);     // simulated perturbation (L1)
}

// Two warp-per-vertex passes (north_star (b): "warp-level shuffles and
// ballots for link-component labelling"); a warp owns the 32 vertices of one
// bitmap word.
//  S1  (k_csr_upper) lanes take N(v) 32 at a time; U(v) = ballot of the upper
//      neighbours, compacted in order (ascending ids) into the upper list
//      upl[row_ptr[v] ..] (|U(v)| in nup[v]); the gradient is the (value, id)
//      maximum over U by two warp max-reductions of order-preserving keys
//      (ties by id, L1); maximum iff U is empty.
//  S3  (k_csr_link) for |U(v)| >= 2: the link edges inside U(v) (reading L14:
//      the subgraph induced on N(v)).  Every edge {a, b} of U(v) closes a
//      triangle whose lowest vertex is v, and is found once from its lower end
//      a: b in U(a) and b in U(v).  Lane p owns a = U(v)[p] (and p + 32), walks
//      the upper list of a and looks each entry up in a per-warp hash set of
//      U(v) -> a bit in its own adjacency word.  Components by
//      frontier expansion: a step ORs the forward words of the frontier
//      (__reduce_or_sync) and the ballot of the lanes whose word meets the
//      frontier (the backward edges); UpperLinkRep = the component's
//      (value, id) maximum.  |U| > 64 (no degree cap): lane 0 runs a
//      union-find over merged sorted rows (row_ptr-indexed scratch), slow but
//      exact.
constexpr int kCsrWarps = 4;
constexpr int kCsrFast = 64;                  // |U| handled by the warp path
constexpr int kHash = 128;                    // per-warp open-addressing set of U

// order-preserving key of a non-NaN float with -0 == +0 (reading L2)
__device__ __forceinline__ uint32_t fkey(float x) {
    const uint32_t b = x == 0.0f ? 0u : __float_as_uint(x);
    return b ^ ((b & 0x80000000u) ? 0xffffffffu : 0x80000000u);
}

__device__ __forceinline__ uint32_t hslot(int32_t x) { return (uint32_t(x) * 2654435761u) >> 25; }

__global__ void __launch_bounds__(32 * kCsrWarps) k_csr_upper(
    const int64_t *__restrict__ rp, const int32_t *__restrict__ ci, const float *__restrict__ f, int64_t v0,
    int64_t v1, int32_t *ptr, uint32_t *max_bits, int32_t *upl, int32_t *nup, int *nan_flag) {
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    const int64_t n = v1 - v0, words = (n + 31) / 32;
    for (int64_t w = int64_t(blockIdx.x) * kCsrWarps + wib; w < words; w += int64_t(gridDim.x) * kCsrWarps) {
        uint32_t mb = 0;
        int32_t my_ptr = 0, my_nu = 0;
        const int jn = n - w * 32 < 32 ? int(n - w * 32) : 32;
        for (int j = 0; j < jn; ++j) {
            const int32_t v = int32_t(v0 + w * 32 + j);
            const int64_t b0 = rp[v], b1 = rp[v + 1];
            const float fv = __ldg(f + v);
            if (lane == 0 && fv != fv) atomicOr(nan_flag, 1);
            int nu = 0;
            uint32_t bk = 0u;          // lane-local best order key (0: none; every finite key is > 0)
            int32_t bid = -1;
            for (int64_t e0 = b0; e0 < b1; e0 += 32) {
                const int64_t e = e0 + lane;
                const int32_t u = e < b1 ? ci[e] : -1;
                const float fu = u >= 0 ? __ldg(f + u) : 0.f;
                const bool up = u >= 0 && csr_higher(u, fu, v, fv);
                const uint32_t bal = __ballot_sync(0xffffffffu, up);
                if (up) {
                    upl[b0 + nu + __popc(bal & lt)] = u;
                    const uint32_t k = fkey(fu);
                    if (k > bk || (k == bk && u > bid)) {
                        bk = k;
                        bid = u;
                    }
                }
                nu += __popc(bal);
            }
            const uint32_t km = __reduce_max_sync(0xffffffffu, bk);
            const int32_t best = __reduce_max_sync(0xffffffffu, (bk == km && bid >= 0) ? bid : -1);
            if (lane == j) {
                my_ptr = nu == 0 ? v : best;
                my_nu = nu;
            }
            mb |= uint32_t(nu == 0) << j;
        }
        const int64_t i = w * 32 + lane;
        if (lane < jn) {
            ptr[i] = my_ptr;
            nup[v0 + i] = my_nu;
        }
        if (lane == 0 && max_bits) max_bits[w] = mb;
    }
}

__device__ __forceinline__ int uf_find_g(int32_t *par, int x) {
    while (par[x] != x) {
        par[x] = par[par[x]];
        x = par[x];
    }
    return x;
}

// lane 0 only: union-find over U (ascending, in gU) for |U| > kCsrFast, link
// edges by merging the sorted rows N(a) with U.  Returns beta0+; the reps
// (ascending) go to reps_out when non-null.
__device__ __noinline__ int csr_slow_components(const int64_t *__restrict__ rp, const int32_t *__restrict__ ci,
                                                const float *__restrict__ f, const int32_t *gU, int32_t *par, int nu,
                                                int32_t *reps_out) {
    for (int p = 0; p < nu; ++p) par[p] = p;
    for (int p = 0; p < nu; ++p) {
        const int32_t a = gU[p];
        int64_t e = rp[a];
        const int64_t e1 = rp[a + 1];
        int q = p + 1;
        while (e < e1 && q < nu) {
            const int32_t x = ci[e], y = gU[q];
            if (x < y) ++e;
            else if (y < x) ++q;
            else {
                const int ra = uf_find_g(par, p), rb = uf_find_g(par, q);
                if (ra != rb) par[max(ra, rb)] = min(ra, rb);
                ++e;
                ++q;
            }
        }
    }
    int b = 0;
    for (int p = 0; p < nu; ++p) {
        if (uf_find_g(par, p) != p) continue;
        int32_t r = -1;
        float rf = 0.f;
        for (int q = p; q < nu; ++q) {
            if (uf_find_g(par, q) != p) continue;
            const float fq = __ldg(f + gU[q]);
            if (r < 0 || fq >= rf) {   // ascending ids: >= keeps the higher id on ties
                r = gU[q];
                rf = fq;
            }
        }
        if (reps_out) reps_out[b] = r;
        ++b;
    }
    if (reps_out)
        for (int a = 1; a < b; ++a) {
            const int32_t x = reps_out[a];
            int c = a - 1;
            while (c >= 0 && reps_out[c] > x) {
                reps_out[c + 1] = reps_out[c];
                --c;
            }
            reps_out[c + 1] = x;
        }
    return b;
}

struct __align__(16) CsrLinkSmem {
    int32_t hkey[kHash];                      // first: 16-byte aligned for the int4 clear
    int32_t hpos[kHash];
    int32_t rep[kCsrFast];
};

__device__ __forceinline__ void hset_insert(CsrLinkSmem &sm, int32_t u, int pos) {
    uint32_t h = hslot(u);
    while (atomicCAS(&sm.hkey[h], -1, u) != -1) h = (h + 1) & (kHash - 1);
    sm.hpos[h] = pos;
}

__device__ __forceinline__ int hset_find(const CsrLinkSmem &sm, int32_t x) {   // position of x in U, or -1
    uint32_t h = hslot(x);
    for (;;) {
        const int32_t key = sm.hkey[h];
        if (key == x) return sm.hpos[h];
        if (key == -1) return -1;
        h = (h + 1) & (kHash - 1);
    }
}

// |U(v)| <= 32: lane p owns link vertex U[p]; 32-bit adjacency words.
// Returns beta0+; with reps != null the ascending UpperLinkReps of a saddle
// are stored there.
__device__ __forceinline__ int csr_link32(CsrLinkSmem &sm, const int64_t *__restrict__ rp,
                                          const float *__restrict__ f, const int32_t *__restrict__ upl,
                                          const int32_t *__restrict__ nup, const int32_t *U, int nu, int lane,
                                          int32_t *reps) {
    reinterpret_cast<int4 *>(sm.hkey)[lane] = make_int4(-1, -1, -1, -1);
    __syncwarp();
    const int32_t uA = lane < nu ? U[lane] : -1;
    int64_t sA = 0;
    int lA = 0;
    if (uA >= 0) {
        hset_insert(sm, uA, lane);
        sA = rp[uA];
        lA = nup[uA];
    }
    const uint32_t kA = uA >= 0 ? fkey(__ldg(f + uA)) : 0u;
    __syncwarp();
    // forward link edges {a, b}, b in U(a) and b in U(v); four loads in flight
    uint32_t adj = 0u;
    for (int k = 0; k < lA; k += 4) {
        int32_t x[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) x[i] = k + i < lA ? upl[sA + k + i] : -1;
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (x[i] >= 0) {
                const int q = hset_find(sm, x[i]);
                if (q >= 0) adj |= 1u << q;
            }
    }
    const uint32_t all = nu == 32 ? 0xffffffffu : ((1u << nu) - 1u);
    uint32_t seen = 0u;
    int beta = 0;
    int32_t my_rep = -1;
    while (seen != all) {
        uint32_t comp = (all & ~seen) & (0u - (all & ~seen));     // lowest unseen link vertex
        for (;;) {
            const bool in = (comp >> lane) & 1u;
            const uint32_t fw = __reduce_or_sync(0xffffffffu, in ? adj : 0u);        // forward edges
            const uint32_t bw = __ballot_sync(0xffffffffu, (adj & comp) != 0u);       // backward edges
            const uint32_t nc = (comp | fw | bw) & all;
            if (nc == comp) break;
            comp = nc;
        }
        // UpperLinkRep: the (value, id) maximum of the component
        const bool in = (comp >> lane) & 1u;
        const uint32_t kmax = __reduce_max_sync(0xffffffffu, in ? kA : 0u);
        const int32_t rv = __reduce_max_sync(0xffffffffu, (in && kA == kmax) ? uA : -1);
        if (lane == beta) my_rep = rv;
        ++beta;
        seen |= comp;
    }
    if (beta >= 2 && reps) {
        int rank = 0;   // ascending reps: rank among the component reps
        for (int j = 0; j < beta; ++j) rank += __shfl_sync(0xffffffffu, my_rep, j) < my_rep;
        if (lane < beta) reps[rank] = my_rep;
    }
    return beta;
}

__global__ void __launch_bounds__(32 * kCsrWarps) k_csr_link(
    const int64_t *__restrict__ rp, const int32_t *__restrict__ ci, const float *__restrict__ f, int64_t v0,
    int64_t v1, const int32_t *__restrict__ upl, const int32_t *__restrict__ nup, uint32_t *sad_bits,
    uint8_t *beta_out, int32_t *rep_buf, int32_t *slow_p) {
    __shared__ CsrLinkSmem sm_all[kCsrWarps];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    CsrLinkSmem &sm = sm_all[wib];
    const int64_t n = v1 - v0, words = (n + 31) / 32;
    const int pa = lane, pb = lane + 32;
    for (int64_t w = int64_t(blockIdx.x) * kCsrWarps + wib; w < words; w += int64_t(gridDim.x) * kCsrWarps) {
        const int jn = n - w * 32 < 32 ? int(n - w * 32) : 32;
        const int my_nu = lane < jn ? nup[v0 + w * 32 + lane] : 0;
        int my_beta = my_nu < 2 ? my_nu : 0;            // 0: maximum, 1: regular
        uint32_t todo = __ballot_sync(0xffffffffu, my_nu >= 2);
        while (todo) {
            const int j = __ffs(todo) - 1;
            todo &= todo - 1;
            const int32_t v = int32_t(v0 + w * 32 + j);
            const int nu = __shfl_sync(0xffffffffu, my_nu, j);
            const int64_t b0 = rp[v];
            const int32_t *U = upl + b0;
            int beta = 0;
            if (nu <= 32) {
                beta = csr_link32(sm, rp, f, upl, nup, U, nu, lane, rep_buf ? rep_buf + b0 : nullptr);
                __syncwarp();
            } else if (nu <= kCsrFast) {
                reinterpret_cast<int4 *>(sm.hkey)[lane] = make_int4(-1, -1, -1, -1);
                __syncwarp();
                const int32_t uA = pa < nu ? U[pa] : -1, uB = pb < nu ? U[pb] : -1;
                if (uA >= 0) {
                    uint32_t h = hslot(uA);
                    while (atomicCAS(&sm.hkey[h], -1, uA) != -1) h = (h + 1) & (kHash - 1);
                    sm.hpos[h] = pa;
                }
                if (uB >= 0) {
                    uint32_t h = hslot(uB);
                    while (atomicCAS(&sm.hkey[h], -1, uB) != -1) h = (h + 1) & (kHash - 1);
                    sm.hpos[h] = pb;
                }
                // the upper lists of a = U[pa] / U[pb]
                int64_t sA = 0, sB = 0;
                int lA = 0, lB = 0;
                if (uA >= 0) {
                    sA = rp[uA];
                    lA = nup[uA];
                }
                if (uB >= 0) {
                    sB = rp[uB];
                    lB = nup[uB];
                }
                __syncwarp();
                // forward link edges: b in U(a) and b in U(v)
                unsigned long long adjA = 0ull, adjB = 0ull;
                for (int k = 0; k < lA; ++k) {
                    const int32_t x = upl[sA + k];
                    uint32_t h = hslot(x);
                    for (;;) {
                        const int32_t key = sm.hkey[h];
                        if (key == x) {
                            adjA |= 1ull << sm.hpos[h];
                            break;
                        }
                        if (key == -1) break;
                        h = (h + 1) & (kHash - 1);
                    }
                }
                for (int k = 0; k < lB; ++k) {
                    const int32_t x = upl[sB + k];
                    uint32_t h = hslot(x);
                    for (;;) {
                        const int32_t key = sm.hkey[h];
                        if (key == x) {
                            adjB |= 1ull << sm.hpos[h];
                            break;
                        }
                        if (key == -1) break;
                        h = (h + 1) & (kHash - 1);
                    }
                }
                const float fA = uA >= 0 ? __ldg(f + uA) : 0.f, fB = uB >= 0 ? __ldg(f + uB) : 0.f;
                const uint32_t kA = uA >= 0 ? fkey(fA) : 0u, kB = uB >= 0 ? fkey(fB) : 0u;
                const unsigned long long all = nu == 64 ? ~0ull : ((1ull << nu) - 1ull);
                unsigned long long seen = 0ull;
                while (seen != all) {
                    unsigned long long comp = 1ull << (__ffsll((long long)(all & ~seen)) - 1);
                    for (;;) {
                        const bool inA = (comp >> pa) & 1ull, inB = (comp >> pb) & 1ull;
                        const unsigned long long c = (inA ? adjA : 0ull) | (inB ? adjB : 0ull);
                        const unsigned lo32 = __reduce_or_sync(0xffffffffu, unsigned(c));
                        const unsigned hi32 = __reduce_or_sync(0xffffffffu, unsigned(c >> 32));
                        // backward edges: lanes whose forward word meets the frontier
                        const unsigned bA = __ballot_sync(0xffffffffu, (adjA & comp) != 0ull);
                        const unsigned bBk = __ballot_sync(0xffffffffu, (adjB & comp) != 0ull);
                        const unsigned long long nc =
                            (comp | ((unsigned long long)(hi32 | bBk) << 32) | (lo32 | bA)) & all;
                        if (nc == comp) break;
                        comp = nc;
                    }
                    // UpperLinkRep: the (value, id) maximum of the component
                    const bool inA = (comp >> pa) & 1ull, inB = (comp >> pb) & 1ull;
                    const uint32_t kk = max(inA ? kA : 0u, inB ? kB : 0u);
                    const uint32_t kmax = __reduce_max_sync(0xffffffffu, kk);
                    const int32_t cand = max((inA && kA == kmax) ? uA : -1, (inB && kB == kmax) ? uB : -1);
                    const int32_t rv = __reduce_max_sync(0xffffffffu, cand);
                    if (lane == 0) sm.rep[beta] = rv;
                    ++beta;
                    seen |= comp;
                }
                __syncwarp();
                if (beta >= 2 && rep_buf) {
                    // ascending reps: rank of each among the component reps
                    for (int k = lane; k < beta; k += 32) {
                        const int32_t r = sm.rep[k];
                        int rank = 0;
                        for (int j2 = 0; j2 < beta; ++j2) rank += sm.rep[j2] < r;
                        rep_buf[b0 + rank] = r;
                    }
                }
                __syncwarp();
            } else {
                // no degree cap: lane 0 finishes serially over the merged full rows
                if (lane == 0)
                    beta = csr_slow_components(rp, ci, f, U, slow_p + b0, nu, rep_buf ? rep_buf + b0 : nullptr);
                beta = __shfl_sync(0xffffffffu, beta, 0);
            }
            if (lane == j) my_beta = beta;
        }
        const uint32_t sb = __ballot_sync(0xffffffffu, my_beta >= 2);
        if (lane < jn && beta_out) beta_out[w * 32 + lane] = uint8_t(my_beta > 255 ? 255 : my_beta);
        if (lane == 0) sad_bits[w] = sb;
    }
}

// k_csr_link_flat: the same S3 with the link-edge search flattened over the
// warp.  The hash-set walk above gives lane p the whole list U(a_p) (about 11
// entries on C5) while lanes p >= |U| idle and every probe loop diverges: 820
// warp instructions per vertex at 15.7 active lanes (ncu, round 2).  Here the
// |U(a_p)| entries of all positions p are numbered t = 0 .. T-1 (warp prefix
// sum of the lengths), lane l takes t = l, l + 32, ...: the owner p of t is a
// branch-free binary search over the prefix sums, b = U(a_p)[t - off_p] one
// load, and b's position in the ascending U(v) a second binary search (5-6
// fixed steps, no divergence); a hit sets bit q of adj[p] by a shared-memory
// atomicOr.  Components, UpperLinkReps and the outputs are those of
// k_csr_link.
constexpr int kFlatMax = 64;
constexpr int kFlatHash = 512;          // direct-mapped id -> position table (|U| <= 32)
constexpr int kFlatShift = 23;          // slot = (id * golden) >> kFlatShift
struct __align__(16) CsrFlatSmem {
    int32_t hkey[kFlatHash];        // U(v) member with this slot, -1 = empty
    uint32_t adj32[32];
    int32_t owner[32];              // rank among the nonempty positions -> position
    unsigned long long adj[kFlatMax];
    int64_t sa[kFlatMax];          // upl offset of U(a_p)
    int32_t su[kFlatMax];          // U(v), ascending ids
    int32_t off[kFlatMax];         // exclusive prefix sums of |U(a_p)|
    int32_t rep[kFlatMax];
};

// largest i < n with a[i] <= x, given a[0] <= x or returning 0 (a ascending, n <= 64)
__device__ __forceinline__ int bsearch_le(const int32_t *a, int n, int32_t x) {
    int lo = 0;
#pragma unroll
    for (int step = 32; step >= 1; step >>= 1) {
        const int m = lo + step;
        if (m < n && a[m] <= x) lo = m;
    }
    return lo;
}

__global__ void __launch_bounds__(32 * kCsrWarps) k_csr_link_flat(
    const int64_t *__restrict__ rp, const int32_t *__restrict__ ci, const float *__restrict__ f, int64_t v0,
    int64_t v1, const int32_t *__restrict__ upl, const int32_t *__restrict__ nup, uint32_t *sad_bits,
    uint8_t *beta_out, int32_t *rep_buf, int32_t *slow_p) {
    __shared__ CsrFlatSmem sm_all[kCsrWarps];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    CsrFlatSmem &sm = sm_all[wib];
    const int64_t n = v1 - v0, words = (n + 31) / 32;
    const uint32_t lt = (1u << lane) - 1u;
    for (int64_t w = int64_t(blockIdx.x) * kCsrWarps + wib; w < words; w += int64_t(gridDim.x) * kCsrWarps) {
        const int jn = n - w * 32 < 32 ? int(n - w * 32) : 32;
        const int my_nu = lane < jn ? nup[v0 + w * 32 + lane] : 0;
        int my_beta = my_nu < 2 ? my_nu : 0;            // 0: maximum, 1: regular
        const int64_t my_b0 = lane < jn ? rp[v0 + w * 32 + lane] : 0;
        uint32_t todo = __ballot_sync(0xffffffffu, my_nu >= 2);
        // software pipeline over the word's vertices: the next vertex's U(v)
        // entries are loaded when the current one starts, their rows / values
        // while its link edges are searched (three dependent gathers per vertex
        // otherwise serialise with its compute)
        int32_t nx_u = -1;
        int64_t nx_s = 0;
        int nx_l = 0;
        float nx_f = 0.f;
        auto fetch_u = [&](uint32_t td) {
            nx_u = -1;
            if (!td) return;
            const int jj = __ffs(td) - 1;
            const int nn = __shfl_sync(0xffffffffu, my_nu, jj);
            const int64_t bb = __shfl_sync(0xffffffffu, my_b0, jj);
            if (lane < nn) nx_u = upl[bb + lane];
        };
        auto fetch_rows = [&]() {
            if (nx_u >= 0) {
                nx_s = rp[nx_u];
                nx_l = nup[nx_u];
                nx_f = __ldg(f + nx_u);
            }
        };
        fetch_u(todo);
        fetch_rows();
        while (todo) {
            const int j = __ffs(todo) - 1;
            todo &= todo - 1;
            const int nu = __shfl_sync(0xffffffffu, my_nu, j);
            const int64_t b0 = __shfl_sync(0xffffffffu, my_b0, j);
            const int32_t *U = upl + b0;
            const int32_t cu = nx_u;
            const int64_t cs = nx_s;
            const int cl = nx_l;
            const float cf = nx_f;
            fetch_u(todo);
            int beta = 0;
            if (nu <= 32) {
                // |U| <= 32 (almost every vertex of a kNN graph): position p = lane.
                // U(v) goes into a direct-mapped table (slot = id hash, 8 bits);
                // when two members share a slot the vertex takes the binary
                // searches of the general path below instead.
                const bool mine = lane < nu;
                const int32_t uA = cu;
                const int lA = mine ? cl : 0;
                const int64_t sA = mine ? cs : 0;
                const uint32_t kA = mine ? fkey(cf) : 0u;
                const uint32_t slot = (uint32_t(uA) * 2654435761u) >> kFlatShift;
#pragma unroll
                for (int k = 0; k < kFlatHash / 128; ++k)
                    reinterpret_cast<int4 *>(sm.hkey)[lane + 32 * k] = make_int4(-1, -1, -1, -1);
                const uint32_t same = __match_any_sync(0xffffffffu, mine ? slot : uint32_t(kFlatHash) + lane);
                const bool clash = __any_sync(0xffffffffu, mine && __popc(same) > 1);
                int iA = lA;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, iA, o);
                    if (lane >= o) iA += y;
                }
                const int T = __shfl_sync(0xffffffffu, iA, 31);
                const int offA = iA - lA;
                const uint32_t ne = __ballot_sync(0xffffffffu, lA > 0);
                __syncwarp();
                if (mine) {
                    sm.su[lane] = uA;
                    sm.off[lane] = offA;
                    sm.sa[lane] = sA;
                    if (!clash) sm.hkey[slot] = lane;    // the member's position (its id is sm.su[pos])
                }
                if (lA > 0) sm.owner[__popc(ne & lt)] = lane;
                sm.adj32[lane] = 0u;
                __syncwarp();
                // windows of 32 entries: the owner of entry t0 + l is the last
                // nonempty position starting at or before it (starts are distinct)
                // up to four windows per batch: every gather of the batch is in
                // flight before the first lookup
                for (int t00 = 0; t00 < T; t00 += 128) {
                    int32_t bb[4];
                    int pp[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int t0 = t00 + 32 * k;
                        const bool st = lA > 0 && offA >= t0 && offA < t0 + 32;
                        const uint32_t S = __reduce_or_sync(0xffffffffu, st ? 1u << (offA - t0) : 0u);
                        const int base = __popc(__ballot_sync(0xffffffffu, lA > 0 && offA < t0));
                        const int t = t0 + lane;
                        pp[k] = -1;
                        bb[k] = -1;
                        if (t < T) {
                            const int p = sm.owner[base - 1 + __popc(S & (0xffffffffu >> (31 - lane)))];
                            pp[k] = p;
                            bb[k] = upl[sm.sa[p] + (t - sm.off[p])];
                        }
                    }
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        if (pp[k] < 0) continue;
                        const int32_t b = bb[k];
                        int q;
                        bool hit;
                        if (!clash) {
                            q = sm.hkey[(uint32_t(b) * 2654435761u) >> kFlatShift];
                            hit = q >= 0 && sm.su[q] == b;
                        } else {
                            q = bsearch_le(sm.su, nu, b);
                            hit = sm.su[q] == b;
                        }
                        if (hit) atomicOr(&sm.adj32[pp[k]], 1u << q);
                    }
                }
                fetch_rows();
                __syncwarp();
                const uint32_t adj = sm.adj32[lane];
                const uint32_t all = nu == 32 ? 0xffffffffu : ((1u << nu) - 1u);
                uint32_t seen = 0u;
                int32_t my_rep = -1;
                while (seen != all) {
                    uint32_t comp = (all & ~seen) & (0u - (all & ~seen));
                    for (;;) {
                        const bool in = (comp >> lane) & 1u;
                        const uint32_t fw = __reduce_or_sync(0xffffffffu, in ? adj : 0u);
                        const uint32_t bw = __ballot_sync(0xffffffffu, (adj & comp) != 0u);
                        const uint32_t nc = (comp | fw | bw) & all;
                        if (nc == comp) break;
                        comp = nc;
                    }
                    const bool in = (comp >> lane) & 1u;
                    const uint32_t kmax = __reduce_max_sync(0xffffffffu, in ? kA : 0u);
                    const int32_t rv = __reduce_max_sync(0xffffffffu, (in && kA == kmax) ? uA : -1);
                    if (lane == beta) my_rep = rv;
                    ++beta;
                    seen |= comp;
                }
                if (beta >= 2 && rep_buf) {
                    int rank = 0;
                    for (int k = 0; k < beta; ++k) rank += __shfl_sync(0xffffffffu, my_rep, k) < my_rep;
                    if (lane < beta) rep_buf[b0 + rank] = my_rep;
                }
                __syncwarp();
            } else if (nu <= kFlatMax) {
                // positions lane and lane + 32: a, its upper list, its key
                const int pb = lane + 32;
                const int32_t uA = lane < nu ? U[lane] : -1, uB = pb < nu ? U[pb] : -1;
                int lA = 0, lB = 0;
                int64_t sA = 0, sB = 0;
                if (uA >= 0) {
                    sA = rp[uA];
                    lA = nup[uA];
                }
                if (uB >= 0) {
                    sB = rp[uB];
                    lB = nup[uB];
                }
                const uint32_t kA = uA >= 0 ? fkey(__ldg(f + uA)) : 0u, kB = uB >= 0 ? fkey(__ldg(f + uB)) : 0u;
                // exclusive prefix sums of the lengths over positions 0 .. nu-1
                int iA = lA, iB = lB;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int yA = __shfl_up_sync(0xffffffffu, iA, o), yB = __shfl_up_sync(0xffffffffu, iB, o);
                    if (lane >= o) {
                        iA += yA;
                        iB += yB;
                    }
                }
                const int totA = __shfl_sync(0xffffffffu, iA, 31), totB = __shfl_sync(0xffffffffu, iB, 31);
                const int T = totA + totB;
                if (lane < nu) {
                    sm.su[lane] = uA;
                    sm.off[lane] = iA - lA;
                    sm.sa[lane] = sA;
                }
                if (pb < nu) {
                    sm.su[pb] = uB;
                    sm.off[pb] = totA + iB - lB;
                    sm.sa[pb] = sB;
                }
                sm.adj[lane] = 0ull;
                sm.adj[pb] = 0ull;
                __syncwarp();
                // link edges {a_p, b}: b in U(a_p) and b in U(v), one entry per lane
                for (int t = lane; t < T; t += 32) {
                    const int p = bsearch_le(sm.off, nu, t);
                    const int32_t b = upl[sm.sa[p] + (t - sm.off[p])];
                    const int q = bsearch_le(sm.su, nu, b);
                    if (sm.su[q] == b) atomicOr(&sm.adj[p], 1ull << q);
                }
                __syncwarp();
                if (nu <= 32) {
                    const uint32_t adj = uint32_t(sm.adj[lane]);
                    const uint32_t all = nu == 32 ? 0xffffffffu : ((1u << nu) - 1u);
                    uint32_t seen = 0u;
                    int32_t my_rep = -1;
                    while (seen != all) {
                        uint32_t comp = (all & ~seen) & (0u - (all & ~seen));
                        for (;;) {
                            const bool in = (comp >> lane) & 1u;
                            const uint32_t fw = __reduce_or_sync(0xffffffffu, in ? adj : 0u);
                            const uint32_t bw = __ballot_sync(0xffffffffu, (adj & comp) != 0u);
                            const uint32_t nc = (comp | fw | bw) & all;
                            if (nc == comp) break;
                            comp = nc;
                        }
                        const bool in = (comp >> lane) & 1u;
                        const uint32_t kmax = __reduce_max_sync(0xffffffffu, in ? kA : 0u);
                        const int32_t rv = __reduce_max_sync(0xffffffffu, (in && kA == kmax) ? uA : -1);
                        if (lane == beta) my_rep = rv;
                        ++beta;
                        seen |= comp;
                    }
                    if (beta >= 2 && rep_buf) {
                        int rank = 0;
                        for (int k = 0; k < beta; ++k) rank += __shfl_sync(0xffffffffu, my_rep, k) < my_rep;
                        if (lane < beta) rep_buf[b0 + rank] = my_rep;
                    }
                } else {
                    const unsigned long long adjA = sm.adj[lane], adjB = sm.adj[pb];
                    const unsigned long long all = nu == 64 ? ~0ull : ((1ull << nu) - 1ull);
                    unsigned long long seen = 0ull;
                    while (seen != all) {
                        unsigned long long comp = 1ull << (__ffsll((long long)(all & ~seen)) - 1);
                        for (;;) {
                            const bool inA = (comp >> lane) & 1ull, inB = (comp >> pb) & 1ull;
                            const unsigned long long c = (inA ? adjA : 0ull) | (inB ? adjB : 0ull);
                            const unsigned lo32 = __reduce_or_sync(0xffffffffu, unsigned(c));
                            const unsigned hi32 = __reduce_or_sync(0xffffffffu, unsigned(c >> 32));
                            const unsigned bA = __ballot_sync(0xffffffffu, (adjA & comp) != 0ull);
                            const unsigned bBk = __ballot_sync(0xffffffffu, (adjB & comp) != 0ull);
                            const unsigned long long nc =
                                (comp | ((unsigned long long)(hi32 | bBk) << 32) | (lo32 | bA)) & all;
                            if (nc == comp) break;
                            comp = nc;
                        }
                        const bool inA = (comp >> lane) & 1ull, inB = (comp >> pb) & 1ull;
                        const uint32_t kk = max(inA ? kA : 0u, inB ? kB : 0u);
                        const uint32_t kmax = __reduce_max_sync(0xffffffffu, kk);
                        const int32_t cand = max((inA && kA == kmax) ? uA : -1, (inB && kB == kmax) ? uB : -1);
                        const int32_t rv = __reduce_max_sync(0xffffffffu, cand);
                        if (lane == 0) sm.rep[beta] = rv;
                        ++beta;
                        seen |= comp;
                    }
                    __syncwarp();
                    if (beta >= 2 && rep_buf) {
                        for (int k = lane; k < beta; k += 32) {
                            const int32_t r = sm.rep[k];
                            int rank = 0;
                            for (int j2 = 0; j2 < beta; ++j2) rank += sm.rep[j2] < r;
                            rep_buf[b0 + rank] = r;
                        }
                    }
                }
                __syncwarp();
            } else {
                // no degree cap: lane 0 finishes serially over the merged full rows
                if (lane == 0)
                    beta = csr_slow_components(rp, ci, f, U, slow_p + b0, nu, rep_buf ? rep_buf + b0 : nullptr);
                beta = __shfl_sync(0xffffffffu, beta, 0);
            }
            if (nu > 32) fetch_rows();
            if (lane == j) my_beta = beta;
        }
        const uint32_t sb = __ballot_sync(0xffffffffu, my_beta >= 2);
        if (lane < jn && beta_out) beta_out[w * 32 + lane] = uint8_t(my_beta > 255 ? 255 : my_beta);
        if (lane == 0) sad_bits[w] = sb;
    }
}

// EG_CHECK_CSR: row_ptr[0] = 0, monotone, row_ptr[N] = nnz;
// 0 <= col_idx < N; every row strictly ascending (sorted, no duplicates); no
// self loops; symmetric (u in N(v) => v in N(u), by binary search).  Reading
// L14's induced-subgraph link needs all of it.  bad |= 1 (row_ptr), 2 (range),
// 4 (order / duplicate), 8 (self loop), 16 (asymmetric).
__global__ void k_check_csr(const int64_t *__restrict__ rp, const int32_t *__restrict__ ci, int64_t N, int64_t nnz,
                            int *bad) {
    const int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (v >= N) return;
    const int64_t r0 = rp[v], r1 = rp[v + 1];
    int b = 0;
    if ((v == 0 && r0 != 0) || (v == N - 1 && r1 != nnz) || r0 < 0 || r1 > nnz || r0 > r1) {
        atomicOr(bad, 1);
        return;
    }
    int64_t prev = -1;
    for (int64_t e = r0; e < r1; ++e) {
        const int64_t u = ci[e];
        if (u < 0 || u >= N) {
            b |= 2;
            continue;
        }
        if (u <= prev) b |= 4;
        if (u == v) b |= 8;
        prev = u;
        const int64_t s0 = rp[u], s1 = rp[u + 1];
        if (s0 < 0 || s1 > nnz || s0 > s1) {
            b |= 1;
            continue;
        }
        int64_t lo = s0, hi = s1;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (ci[mid] < v) lo = mid + 1;
            else hi = mid;
        }
        if (lo >= s1 || ci[lo] != v) b |= 16;
    }
    if (b) atomicOr(bad, b);
}

cudaError_t launch_check_csr(const int64_t *row_ptr, const int32_t *col_idx, int64_t n, int64_t nnz, int *bad,
                             cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    k_check_csr<<<unsigned((n + 255) / 256), 256, 0, st>>>(row_ptr, col_idx, n, nnz, bad);
    return cudaGetLastError();
}

__device__ __forceinline__ int32_t label_of_csr(const LabelView &lv, int64_t g) {
    return lv.own[g - lv.v0];       // CSR: labels are gathered for every vertex
}

// S4 from the representatives classify stored (no second link computation):
// m = label[rep] per component, sorted, unique with multiplicity (reading L7).
// The m's are sorted in place in the saddle's own slots of tmp_m (no cap on
// beta0+).
__global__ void __launch_bounds__(128) k_arcs_csr_reps(const int64_t *__restrict__ rp,
                                                       const int32_t *__restrict__ rep_buf,
                                                       const int32_t *__restrict__ saddles,
                                                       const int32_t *__restrict__ sbeta, int64_t n_sad,
                                                       const int64_t *__restrict__ slot_off, LabelView lv,
                                                       int32_t *tmp_m, int32_t *tmp_mult, int32_t *n_unique,
                                                       int64_t *raw_s, int64_t *raw_rep, int64_t *raw_m) {
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= n_sad) return;
    const int32_t v = saddles[j];
    const int b = sbeta[j];
    const int32_t *reps = rep_buf + rp[v];
    const int64_t off = slot_off[j];
    int32_t *ms = tmp_m + off;
    for (int c = 0; c < b; ++c) {
        const int32_t r = reps[c];
        const int32_t m = label_of_csr(lv, r);
        if (raw_s) {
            raw_s[off + c] = v;
            raw_rep[off + c] = r;
            raw_m[off + c] = m;
        }
        int k = c - 1;                 // insertion into the sorted prefix
        while (k >= 0 && ms[k] > m) {
            ms[k + 1] = ms[k];
            --k;
        }
        ms[k + 1] = m;
    }
    int u = 0;
    for (int a = 0; a < b;) {
        int e = a;
        const int32_t m = ms[a];
        while (e < b && ms[e] == m) ++e;
        ms[u] = m;                     // u <= a: compaction in place
        tmp_mult[off + u] = e - a;
        ++u;
        a = e;
    }
    n_unique[j] = u;
}


// Arc geometry on CSR: s, rep, then the highest upper
// neighbour at every vertex until a maximum.
__global__ void __launch_bounds__(128) k_arc_paths_csr(const int64_t *__restrict__ rp, const int32_t *__restrict__ ci,
                                                       const float *__restrict__ f, const int64_t *__restrict__ raw_s,
                                                       const int64_t *__restrict__ raw_rep, int64_t n_raw,
                                                       const int64_t *__restrict__ off, int64_t *len_or_out,
                                                       int32_t *nxt) {
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= n_raw) return;
    int64_t *out = off ? len_or_out + off[j] : nullptr;
    int64_t k = 0;
    if (out) out[k] = raw_s[j];
    ++k;
    int32_t v = int32_t(raw_rep[j]);
    for (;;) {
        if (out) out[k] = v;
        ++k;
        const float fv = __ldg(f + v);
        int32_t bv = v;
        float bf = fv;
        for (int64_t e = rp[v]; e < rp[v + 1]; ++e) {
            const int32_t u = ci[e];
            const float fu = __ldg(f + u);
            if (csr_higher(u, fu, v, fv) && (fu > bf || (fu == bf && u > bv))) {
                bf = fu;
                bv = u;
            }
        }
        if (nxt) nxt[v] = bv;               // the next step (v itself at a maximum), for k_arc_paths_follow
        if (bv == v) break;                 // a maximum
        v = bv;
    }
    if (!off) len_or_out[j] = k;
}

static inline unsigned blocks_for(int64_t n, int bs) { return unsigned((n + bs - 1) / bs); }

static inline unsigned csr_blocks(int64_t n) {
    const int64_t words = (n + 31) / 32;
    return unsigned(std::min<int64_t>((words + kCsrWarps - 1) / kCsrWarps, 148 * 64));
}

cudaError_t launch_csr_upper(const int64_t *row_ptr, const int32_t *col_idx, const float *f, int64_t v0, int64_t v1,
                             int32_t *ptr, uint32_t *max_bits, int32_t *upl, int32_t *nup, int *nan_flag,
                             cudaStream_t st) {
    if (v1 <= v0) return cudaSuccess;
    k_csr_upper<<<csr_blocks(v1 - v0), 32 * kCsrWarps, 0, st>>>(row_ptr, col_idx, f, v0, v1, ptr, max_bits, upl, nup,
                                                                 nan_flag);
    return cudaGetLastError();
}

cudaError_t launch_csr_link(const int64_t *row_ptr, const int32_t *col_idx, const float *f, int64_t v0, int64_t v1,
                            const int32_t *upl, const int32_t *nup, uint32_t *sad_bits, uint8_t *beta_out,
                            int32_t *rep_buf, int32_t *par, cudaStream_t st) {
    if (v1 <= v0) return cudaSuccess;
    const char *ev = std::getenv("EG_CSR_LINK");   // tuning knob: 1 = the hash-set walk (k_csr_link)
    if (ev && std::atoi(ev) == 1)
        k_csr_link<<<csr_blocks(v1 - v0), 32 * kCsrWarps, 0, st>>>(row_ptr, col_idx, f, v0, v1, upl, nup, sad_bits,
                                                                    beta_out, rep_buf, par);
    else
        k_csr_link_flat<<<csr_blocks(v1 - v0), 32 * kCsrWarps, 0, st>>>(row_ptr, col_idx, f, v0, v1, upl, nup,
                                                                         sad_bits, beta_out, rep_buf, par);
    return cudaGetLastError();
}

cudaError_t launch_arcs_csr_reps(const int64_t *row_ptr, const int32_t *rep_buf, const int32_t *saddles,
                                 const int32_t *sbeta, int64_t n_sad, const int64_t *slot_off, LabelView lv,
                                 int32_t *tmp_m, int32_t *tmp_mult, int32_t *n_unique, int64_t *raw_s,
                                 int64_t *raw_rep, int64_t *raw_m, cudaStream_t st) {
    if (n_sad <= 0) return cudaSuccess;
    k_arcs_csr_reps<<<blocks_for(n_sad, 128), 128, 0, st>>>(row_ptr, rep_buf, saddles, sbeta, n_sad, slot_off, lv,
                                                            tmp_m, tmp_mult, n_unique, raw_s, raw_rep, raw_m);
    return cudaGetLastError();
}

cudaError_t launch_arc_paths_csr(const int64_t *row_ptr, const int32_t *col_idx, const float *f, const int64_t *raw_s,
                                 const int64_t *raw_rep, int64_t n_raw, const int64_t *off, int64_t *len_or_out,
                                 cudaStream_t st, int32_t *nxt) {
    if (n_raw <= 0) return cudaSuccess;
    k_arc_paths_csr<<<blocks_for(n_raw, 128), 128, 0, st>>>(row_ptr, col_idx, f, raw_s, raw_rep, n_raw, off,
                                                            len_or_out, nxt);
    return cudaGetLastError();
}

// Second pass of the arc geometry: the first pass left every visited vertex's
// next step in nxt (a vertex of a maximum points to itself), so a path is
// re-walked by one dependent load per vertex instead of a recomputed argmax.
__global__ void __launch_bounds__(128) k_arc_paths_follow(const int64_t *__restrict__ raw_s,
                                                          const int64_t *__restrict__ raw_rep, int64_t n_raw,
                                                          const int64_t *__restrict__ off,
                                                          const int32_t *__restrict__ nxt, int64_t v0, int64_t *out) {
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= n_raw) return;
    int64_t *o = out + off[j];
    o[0] = raw_s[j];
    int64_t k = 1;
    int64_t v = raw_rep[j];
    for (;;) {
        o[k++] = v;
        const int64_t w = __ldg(nxt + (v - v0));
        if (w == v) break;
        v = w;
    }
}

cudaError_t launch_arc_paths_follow(const int64_t *raw_s, const int64_t *raw_rep, int64_t n_raw, const int64_t *off,
                                    const int32_t *nxt, int64_t v0, int64_t *out, cudaStream_t st) {
    if (n_raw <= 0) return cudaSuccess;
    k_arc_paths_follow<<<blocks_for(n_raw, 128), 128, 0, st>>>(raw_s, raw_rep, n_raw, off, nxt, v0, out);
    return cudaGetLastError();
}

}  // namespace eg
