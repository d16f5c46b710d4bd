// CSR neighbourhood-graph kernels (reading L14: the link of v is the subgraph
// induced on N(v)).  S1: gradient = highest upper neighbour; S3:
// beta0+ = components of the induced upper link by union-find over
// the link edges, which are found by merging the sorted lists N(a) and U(v);
// a saddle's component representatives are stored by classify (in its own
// row range of a row_ptr-indexed buffer), so S4 only gathers their labels.
// One thread per vertex.
#include "eg_impl.h"

namespace eg {

__device__ __forceinline__ bool csr_higher(const float *__restrict__ f, int32_t u, float fu, int32_t v, float fv) {
    return fu > fv || (fu == fv && u > v);     // simulated perturbation (L1)
}

__device__ __forceinline__ int uf_find(uint8_t *par, int x) {
    while (par[x] != x) {
        par[x] = par[par[x]];
        x = par[x];
    }
    return x;
}

// Upper set U (ascending ids, since N(v) is sorted), gradient, and
// union-find parents over U.  Returns |U| or -1 if deg > kCsrMaxDeg.
__device__ __forceinline__ int csr_upper_uf(const int64_t *__restrict__ rp, const int32_t *__restrict__ ci,
                                            const float *__restrict__ f, int32_t v, float fv, int32_t *U,
                                            uint8_t *par, int32_t *best) {
    const int64_t b0 = rp[v], b1 = rp[v + 1];
    if (b1 - b0 > kCsrMaxDeg) return -1;
    int nu = 0;
    int32_t bv = v;
    float bf = fv;
    for (int64_t e = b0; e < b1; ++e) {
        const int32_t u = ci[e];
        const float fu = __ldg(f + u);
        if (csr_higher(f, u, fu, v, fv)) {
            U[nu++] = u;
            if (fu >= bf) {   // ascending ids: >= keeps the highest index on ties
                bf = fu;
                bv = u;
            }
        }
    }
    *best = bv;
    for (int p = 0; p < nu; ++p) par[p] = uint8_t(p);
    // link edges inside U: for a = U[p], merge N(a) with U[p+1..]
    for (int p = 0; p < nu; ++p) {
        const int32_t a = U[p];
        int64_t e = rp[a];
        const int64_t e1 = rp[a + 1];
        int q = p + 1;
        while (e < e1 && q < nu) {
            const int32_t x = ci[e], y = U[q];
            if (x < y) ++e;
            else if (y < x) ++q;
            else {
                int ra = uf_find(par, p), rb = uf_find(par, q);
                if (ra != rb) par[rb > ra ? rb : ra] = uint8_t(rb > ra ? ra : rb);
                ++e;
                ++q;
            }
        }
    }
    return nu;
}


// UpperLinkRep: the highest member of every component (roots are the
// smallest position of their component), ascending by id.  Returns beta0+.
__device__ __forceinline__ int csr_reps(const float *__restrict__ f, const int32_t *U, uint8_t *par, int nu,
                                        int32_t *reps) {
    int b = 0;
    for (int p = 0; p < nu; ++p) {
        if (uf_find(par, p) != p) continue;
        int32_t r = -1;
        float rf = 0.f;
        for (int q = p; q < nu; ++q) {
            if (uf_find(par, q) != p) continue;
            const float fq = __ldg(f + U[q]);
            if (r < 0 || fq >= rf) {   // ascending ids
                r = U[q];
                rf = fq;
            }
        }
        reps[b++] = r;
    }
    for (int a = 1; a < b; ++a) {
        const int32_t x = reps[a];
        int c = a - 1;
        while (c >= 0 && reps[c] > x) {
            reps[c + 1] = reps[c];
            --c;
        }
        reps[c + 1] = x;
    }
    return b;
}

__global__ void __launch_bounds__(128) k_classify_csr(const int64_t *__restrict__ rp, const int32_t *__restrict__ ci,
                                                      const float *__restrict__ f, int64_t v0, int64_t v1,
                                                      int32_t *ptr, uint32_t *sad_bits, uint32_t *max_bits,
                                                      uint8_t *beta_out, int *nan_flag, int *deg_overflow,
                                                      int32_t *rep_buf) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool active = i < v1 - v0;
    bool is_sad = false, is_max = false;
    if (active) {
        const int32_t v = int32_t(v0 + i);
        const float fv = __ldg(f + v);
        if (fv != fv) atomicOr(nan_flag, 1);
        int32_t U[kCsrMaxDeg];
        uint8_t par[kCsrMaxDeg];
        int32_t best;
        int nu = csr_upper_uf(rp, ci, f, v, fv, U, par, &best);
        int beta = 0;
        if (nu < 0) {
            atomicOr(deg_overflow, 1);
        } else {
            for (int p = 0; p < nu; ++p) beta += (uf_find(par, p) == p);
            // a saddle keeps its component representatives (beta0+ <= deg(v)
            // of them) in its own row range of rep_buf, for the arcs
            if (beta >= 2 && rep_buf) {
                int32_t reps[kCsrMaxDeg];
                const int b = csr_reps(f, U, par, nu, reps);
                int32_t *out = rep_buf + rp[v];
                for (int k = 0; k < b; ++k) out[k] = reps[k];
            }
        }
        is_max = nu == 0;
        is_sad = beta >= 2;
        ptr[i] = best;
        if (beta_out) beta_out[i] = uint8_t(beta > 255 ? 255 : beta);
    }
    const uint32_t sb = __ballot_sync(0xffffffffu, is_sad);
    const uint32_t mb = __ballot_sync(0xffffffffu, is_max);
    if ((threadIdx.x & 31) == 0 && active) {
        sad_bits[i >> 5] = sb;
        max_bits[i >> 5] = mb;
    }
}

__device__ __forceinline__ int32_t label_of_csr(const LabelView &lv, int64_t g) {
    return lv.own[g - lv.v0];       // CSR: labels are gathered for every vertex
}

// S4 from the representatives classify stored (no second link computation):
// m = label[rep] per component, sorted, unique with multiplicity (reading L7).
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
    int32_t ms[kCsrMaxDeg];
    for (int c = 0; c < b; ++c) {
        const int32_t r = reps[c];
        ms[c] = label_of_csr(lv, r);
        if (raw_s) {
            raw_s[off + c] = v;
            raw_rep[off + c] = r;
            raw_m[off + c] = ms[c];
        }
    }
    for (int a = 1; a < b; ++a) {
        const int32_t x = ms[a];
        int c = a - 1;
        while (c >= 0 && ms[c] > x) {
            ms[c + 1] = ms[c];
            --c;
        }
        ms[c + 1] = x;
    }
    int u = 0;
    for (int a = 0; a < b;) {
        int e = a;
        while (e < b && ms[e] == ms[a]) ++e;
        tmp_m[off + u] = ms[a];
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
            if (csr_higher(f, u, fu, v, fv) && (fu > bf || (fu == bf && u > bv))) {
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
                                uint8_t *beta_out, int *nan_flag, int *deg_overflow, cudaStream_t st,
                                int32_t *rep_buf) {
    if (v1 <= v0) return cudaSuccess;
    k_classify_csr<<<blocks_for(v1 - v0, 128), 128, 0, st>>>(row_ptr, col_idx, f, v0, v1, ptr, sad_bits, max_bits,
                                                             beta_out, nan_flag, deg_overflow, rep_buf);
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
