// CSR neighbourhood-graph kernels (reading L14: the link of v is the subgraph
// induced on N(v)).  S1: gradient = highest upper neighbour; S3:
// beta0+ = components of the induced upper link by union-find over
// the link edges, which are found by merging the sorted lists N(a) and U(v);
// a saddle's component representatives are stored by classify (in its own
// row range of a row_ptr-indexed buffer), so S4 only gathers their labels.
// One warp per vertex (k_classify_csr); no degree cap.
#include <algorithm>

#include "eg_impl.h"

namespace eg {

__device__ __forceinline__ bool csr_higher(int32_t u, float fu, int32_t v, float fv) {
    return fu > fv || (fu == fv && u > v);     // simulated perturbation (L1)
}

// One warp per vertex (north_star (b): "warp-level shuffles and ballots for
// link-component labelling"), a warp owns the 32 vertices of one bitmap word.
//  S1  lanes take N(v) 32 at a time; U = ballot of the upper neighbours,
//      compacted in order (ascending ids) into shared memory; the gradient is
//      a shuffle argmax over (f, id) (ties by id, L1).
//  S3  |U| <= 1: maximum / regular, no link edges needed.  Otherwise the link
//      edges inside U (reading L14: the subgraph induced on N(v)) are found by
//      flattening the rows N(a), a in U, over the lanes: every lane loads one
//      x in N(a) (coalesced within a row), finds x in U by binary search, and
//      sets bit q of a's adjacency word in shared memory.  Components
//       by frontier expansion: each lane owns two link vertices, a
//      step is one __reduce_or_sync of the owned adjacency words of the
//      frontier; UpperLinkRep = shuffle argmax over the component.
//  |U| > 64 (no degree cap): lane 0 runs a union-find over the merged sorted
//      rows in ctx-owned global scratch (row_ptr-indexed), slow but exact.
constexpr int kCsrWarps = 4;
constexpr int kCsrFast = 64;                  // |U| handled by the warp path

struct CsrWarpSmem {
    int32_t u[kCsrFast];
    float fu[kCsrFast];
    int32_t pre[kCsrFast + 1];                // prefix sums of deg(U[p])
    int64_t rs[kCsrFast];                     // row start of U[p]
    unsigned long long adj[kCsrFast];
    int32_t rep[kCsrFast];
};

__device__ __forceinline__ void argmax_fi(float &bf, int32_t &bv) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const float of = __shfl_xor_sync(0xffffffffu, bf, o);
        const int32_t ov = __shfl_xor_sync(0xffffffffu, bv, o);
        if (ov >= 0 && (bv < 0 || of > bf || (of == bf && ov > bv))) {
            bf = of;
            bv = ov;
        }
    }
}

__device__ __forceinline__ int uf_find_g(int32_t *par, int x) {
    while (par[x] != x) {
        par[x] = par[par[x]];
        x = par[x];
    }
    return x;
}

// lane 0 only: union-find over U (already in gU, ascending, with values in
// gF not needed: f is read again) for |U| > kCsrFast.  Returns beta0+; the
// reps (ascending) go to reps_out when non-null.
__device__ int csr_slow_components(const int64_t *__restrict__ rp, const int32_t *__restrict__ ci,
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

__global__ void __launch_bounds__(32 * kCsrWarps) k_classify_csr(
    const int64_t *__restrict__ rp, const int32_t *__restrict__ ci, const float *__restrict__ f, int64_t v0,
    int64_t v1, int32_t *ptr, uint32_t *sad_bits, uint32_t *max_bits, uint8_t *beta_out, int *nan_flag,
    int32_t *rep_buf, int32_t *slow_u, int32_t *slow_p) {
    __shared__ CsrWarpSmem sm_all[kCsrWarps];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    CsrWarpSmem &sm = sm_all[wib];
    const uint32_t lt = (1u << lane) - 1u;
    const int64_t n = v1 - v0, words = (n + 31) / 32;
    for (int64_t w = int64_t(blockIdx.x) * kCsrWarps + wib; w < words; w += int64_t(gridDim.x) * kCsrWarps) {
        uint32_t sb = 0, mb = 0;
        int32_t my_ptr = 0;
        int my_beta = 0;
        const int jn = n - w * 32 < 32 ? int(n - w * 32) : 32;
        for (int j = 0; j < jn; ++j) {
            const int32_t v = int32_t(v0 + w * 32 + j);
            const int64_t b0 = rp[v], b1 = rp[v + 1];
            const float fv = __ldg(f + v);
            if (lane == 0 && fv != fv) atomicOr(nan_flag, 1);
            // ---- S1: upper set U (ascending) and the gradient
            int nu = 0;
            float bf = fv;
            int32_t bv = v;
            for (int64_t e0 = b0; e0 < b1; e0 += 32) {
                const int64_t e = e0 + lane;
                const int32_t u = e < b1 ? ci[e] : -1;
                const float fu = u >= 0 ? __ldg(f + u) : 0.f;
                const bool up = u >= 0 && csr_higher(u, fu, v, fv);
                const uint32_t bal = __ballot_sync(0xffffffffu, up);
                const int pos = nu + __popc(bal & lt);
                if (up) {
                    if (pos < kCsrFast) {
                        sm.u[pos] = u;
                        sm.fu[pos] = fu;
                    } else if (slow_u) {
                        slow_u[b0 + pos] = u;
                    }
                    if (fu > bf || (fu == bf && u > bv)) {
                        bf = fu;
                        bv = u;
                    }
                }
                nu += __popc(bal);
            }
            argmax_fi(bf, bv);
            int beta = 0;
            if (nu >= 2 && nu <= kCsrFast) {
                __syncwarp();
                // ---- S3: link edges inside U, flattened over the rows N(a)
                const int pa = lane, pb = lane + 32;
                int64_t ra = 0, rb = 0;
                int da = 0, db = 0;
                if (pa < nu) {
                    const int32_t a = sm.u[pa];
                    ra = rp[a];
                    da = int(rp[a + 1] - ra);
                }
                if (pb < nu) {
                    const int32_t a = sm.u[pb];
                    rb = rp[a];
                    db = int(rp[a + 1] - rb);
                }
                // inclusive scan of (da, db) over the lanes: positions pa and pb
                int sa = da, sbb = db;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int ya = __shfl_up_sync(0xffffffffu, sa, o);
                    const int yb = __shfl_up_sync(0xffffffffu, sbb, o);
                    if (lane >= o) {
                        sa += ya;
                        sbb += yb;
                    }
                }
                const int tot_a = __shfl_sync(0xffffffffu, sa, 31);
                if (pa < nu) {
                    sm.pre[pa + 1] = sa;
                    sm.rs[pa] = ra;
                }
                if (pb < nu) {
                    sm.pre[pb + 1] = tot_a + sbb;
                    sm.rs[pb] = rb;
                }
                if (lane == 0) sm.pre[0] = 0;
                sm.adj[pa] = 0ull;
                sm.adj[pb] = 0ull;
                __syncwarp();
                const int T = sm.pre[nu];
                for (int t0 = 0; t0 < T; t0 += 32) {
                    const int t = t0 + lane;
                    if (t < T) {
                        // p = the row of element t: last p with pre[p] <= t
                        int lo = 0, hi = nu - 1;
                        while (lo < hi) {
                            const int mid = (lo + hi + 1) >> 1;
                            if (sm.pre[mid] <= t) lo = mid;
                            else hi = mid - 1;
                        }
                        const int32_t x = ci[sm.rs[lo] + (t - sm.pre[lo])];
                        // x in U?  (U ascending)
                        int a = 0, b = nu - 1;
                        while (a < b) {
                            const int mid = (a + b) >> 1;
                            if (sm.u[mid] < x) a = mid + 1;
                            else b = mid;
                        }
                        if (sm.u[a] == x) {
                            unsigned int *wd = reinterpret_cast<unsigned int *>(&sm.adj[lo]) + (a >> 5);
                            atomicOr(wd, 1u << (a & 31));
                        }
                    }
                }
                __syncwarp();
                const unsigned long long adjA = sm.adj[pa], adjB = sm.adj[pb];
                const float fA = pa < nu ? sm.fu[pa] : 0.f, fB = pb < nu ? sm.fu[pb] : 0.f;
                const int32_t uA = pa < nu ? sm.u[pa] : -1, uB = pb < nu ? sm.u[pb] : -1;
                const unsigned long long all = nu == 64 ? ~0ull : ((1ull << nu) - 1ull);
                unsigned long long seen = 0ull;
                while (seen != all) {
                    unsigned long long comp = 1ull << (__ffsll((long long)(all & ~seen)) - 1);
                    for (;;) {
                        const unsigned long long c =
                            (((comp >> pa) & 1ull) ? adjA : 0ull) | ((pb < 64 && ((comp >> pb) & 1ull)) ? adjB : 0ull);
                        const unsigned lo32 = __reduce_or_sync(0xffffffffu, unsigned(c));
                        const unsigned hi32 = __reduce_or_sync(0xffffffffu, unsigned(c >> 32));
                        const unsigned long long nc = (comp | (((unsigned long long)hi32 << 32) | lo32)) & all;
                        if (nc == comp) break;
                        comp = nc;
                    }
                    // UpperLinkRep: the highest member
                    float rf = 0.f;
                    int32_t rv = -1;
                    if ((comp >> pa) & 1ull) {
                        rf = fA;
                        rv = uA;
                    }
                    if (((comp >> pb) & 1ull) && (rv < 0 || fB > rf || (fB == rf && uB > rv))) {
                        rf = fB;
                        rv = uB;
                    }
                    argmax_fi(rf, rv);
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
            } else if (nu > kCsrFast) {
                // no degree cap: the first kCsrFast entries of U are in shared
                // memory, the rest in slow_u; lane 0 finishes serially
                __syncwarp();
                for (int k = lane; k < kCsrFast; k += 32) slow_u[b0 + k] = sm.u[k];
                __syncwarp();
                __threadfence_block();
                if (lane == 0)
                    beta = csr_slow_components(rp, ci, f, slow_u + b0, slow_p + b0, nu, rep_buf ? rep_buf + b0 : nullptr);
                beta = __shfl_sync(0xffffffffu, beta, 0);
                __syncwarp();
            } else {
                beta = nu;   // 0: maximum, 1: regular
            }
            if (lane == j) {
                my_ptr = bv;
                my_beta = beta;
            }
            sb |= uint32_t(beta >= 2) << j;
            mb |= uint32_t(nu == 0) << j;
        }
        const int64_t i = w * 32 + lane;
        if (lane < jn) {
            ptr[i] = my_ptr;
            if (beta_out) beta_out[i] = uint8_t(my_beta > 255 ? 255 : my_beta);
        }
        if (lane == 0) {
            sad_bits[w] = sb;
            max_bits[w] = mb;
        }
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
                                                       const int64_t *__restrict__ off, int64_t *len_or_out) {
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
        if (bv == v) break;                 // a maximum
        v = bv;
    }
    if (!off) len_or_out[j] = k;
}

static inline unsigned blocks_for(int64_t n, int bs) { return unsigned((n + bs - 1) / bs); }

cudaError_t launch_classify_csr(const int64_t *row_ptr, const int32_t *col_idx, const float *f, int64_t v0,
                                int64_t v1, int32_t *ptr, uint32_t *sad_bits, uint32_t *max_bits,
                                uint8_t *beta_out, int *nan_flag, cudaStream_t st, int32_t *rep_buf,
                                int32_t *slow_u, int32_t *slow_p) {
    if (v1 <= v0) return cudaSuccess;
    const int64_t words = (v1 - v0 + 31) / 32;
    const int64_t blocks = std::min<int64_t>((words + kCsrWarps - 1) / kCsrWarps, 148 * 64);
    k_classify_csr<<<unsigned(blocks), 32 * kCsrWarps, 0, st>>>(row_ptr, col_idx, f, v0, v1, ptr, sad_bits,
                                                                 max_bits, beta_out, nan_flag, rep_buf, slow_u,
                                                                 slow_p);
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
                                 cudaStream_t st) {
    if (n_raw <= 0) return cudaSuccess;
    k_arc_paths_csr<<<blocks_for(n_raw, 128), 128, 0, st>>>(row_ptr, col_idx, f, raw_s, raw_rep, n_raw, off,
                                                            len_or_out);
    return cudaGetLastError();
}

}  // namespace eg
