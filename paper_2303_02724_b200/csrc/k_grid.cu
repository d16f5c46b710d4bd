// Generic n-D grid kernels (n = 1..6): S1 steepest-ascent pointer, S3 upper-
// link components, and the per-saddle part of S4.  One thread per vertex, the
// way the paper's classification kernel is organised ("launching a CUDA
// thread for each vertex"), but with the link's edge set replaced by constant
// bitmasks over the 2 (2^n - 1) link offsets: beta0+ is a bitset flood fill
// (every upper link vertex is visited once) instead of P:184's union-find.
// This path serves every n; n <= 3 grids normally take the tiled kernel in
// k_grid3d.cu instead.
#include <cstdio>

#include "eg_impl.h"

namespace eg {

template <int NW>
struct Bits {
    uint64_t w[NW];
    __device__ __forceinline__ void clear() {
#pragma unroll
        for (int i = 0; i < NW; ++i) w[i] = 0;
    }
    __device__ __forceinline__ bool any() const {
        uint64_t x = 0;
#pragma unroll
        for (int i = 0; i < NW; ++i) x |= w[i];
        return x != 0;
    }
    __device__ __forceinline__ void set(int k) { w[k >> 6] |= 1ull << (k & 63); }
    __device__ __forceinline__ int pop_lowest() {  // index of the lowest set bit, cleared; -1 if none
#pragma unroll
        for (int i = 0; i < NW; ++i)
            if (w[i]) {
                int b = __ffsll((long long)w[i]) - 1;
                w[i] &= w[i] - 1;
                return i * 64 + b;
            }
        return -1;
    }
};

template <int NDIM>
struct GridSmem {
    static constexpr int K = 2 * ((1 << NDIM) - 1);
    static constexpr int NW = (K + 63) / 64;
    int32_t delta[K];                       // N < 2^31: 32-bit linear offsets
    uint64_t nbr[K][NW];
    uint64_t neg[NDIM][NW], pos[NDIM][NW];  // offsets with d_a = -1 / +1
    int32_t dims[NDIM];
};

template <int NDIM>
__device__ __forceinline__ void load_tables(GridSmem<NDIM> &S, const LinkTable *__restrict__ tab) {
    constexpr int K = GridSmem<NDIM>::K, NW = GridSmem<NDIM>::NW;
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
        S.delta[k] = int32_t(tab->delta[k]);
#pragma unroll
        for (int w = 0; w < NW; ++w) S.nbr[k][w] = tab->nbr[k][w];
    }
    if (threadIdx.x < NDIM) {
        const int a = threadIdx.x;
        S.dims[a] = int32_t(tab->dims[a]);
#pragma unroll
        for (int w = 0; w < NW; ++w) S.neg[a][w] = S.pos[a][w] = 0;
        for (int k = 0; k < K; ++k) {
            if (tab->d[k][a] < 0) S.neg[a][k >> 6] |= 1ull << (k & 63);
            if (tab->d[k][a] > 0) S.pos[a][k >> 6] |= 1ull << (k & 63);
        }
    }
    __syncthreads();
}

// Upper mask and gradient of global vertex v.  Offsets are
// scanned in ascending global index, so `>=` keeps the highest index among
// equal values (simulated perturbation, reading L1).  Returns the mask; *best
// is the gradient (v for a maximum).
template <int NDIM>
__device__ __forceinline__ Bits<GridSmem<NDIM>::NW> upper_link(const GridSmem<NDIM> &S, const FieldView &F, int64_t v,
                                                               float fv, int64_t *best) {
    constexpr int K = GridSmem<NDIM>::K, NW = GridSmem<NDIM>::NW;
    // the truncated link (reading L3): drop the offsets that leave the domain,
    // one mask per face the vertex lies on
    uint64_t valid[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) valid[w] = ~0ull;
    uint32_t r = uint32_t(v);
#pragma unroll
    for (int a = 0; a < NDIM; ++a) {
        const uint32_t D = uint32_t(S.dims[a]);
        const uint32_t c = r % D;
        r /= D;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            if (c == 0) valid[w] &= ~S.neg[a][w];
            if (c + 1 == D) valid[w] &= ~S.pos[a][w];
        }
    }
    Bits<NW> m;
    m.clear();
    int64_t b = v;
    float bf = fv;
    // one slab (no halo planes): plain loads from the owned array
    const bool plain = F.lo == nullptr && F.hi == nullptr;
    const float *own = F.own - F.v0;
    // the table is sorted by offset: the first K/2 offsets lead to lower
    // indices (up iff f > fv), the rest to higher ones (up iff f >= fv)
#pragma unroll 2
    for (int k = 0; k < K / 2; ++k) {
        if (!((valid[k >> 6] >> (k & 63)) & 1ull)) continue;
        const int64_t u = v + S.delta[k];
        const float fu = plain ? __ldg(own + u) : F.at(u);
        if (fu > fv) {
            m.set(k);
            if (fu >= bf) {
                bf = fu;
                b = u;
            }
        }
    }
#pragma unroll 2
    for (int k = K / 2; k < K; ++k) {
        if (!((valid[k >> 6] >> (k & 63)) & 1ull)) continue;
        const int64_t u = v + S.delta[k];
        const float fu = plain ? __ldg(own + u) : F.at(u);
        if (fu >= fv) {
            m.set(k);
            if (fu >= bf) {
                bf = fu;
                b = u;
            }
        }
    }
    *best = b;
    return m;
}

// beta0+: components of the upper link by bitset flood fill over
// the constant link adjacency.  If reps != null, also the highest vertex of
// every component (UpperLinkRep), in component order.
template <int NDIM>
__device__ __forceinline__ int components(const GridSmem<NDIM> &S, Bits<GridSmem<NDIM>::NW> rem, const FieldView &F,
                                          int64_t v, int32_t *reps) {
    constexpr int NW = GridSmem<NDIM>::NW;
    int beta = 0;
    while (rem.any()) {
        Bits<NW> front;
        front.clear();
        int seed = rem.pop_lowest();
        front.set(seed);
        int64_t rep = -1;
        float rf = 0.f;
        int k;
        while ((k = front.pop_lowest()) >= 0) {
            if (reps) {
                int64_t u = v + S.delta[k];
                float fu = F.at(u);
                if (rep < 0 || fu > rf || (fu == rf && u > rep)) {
                    rep = u;
                    rf = fu;
                }
            }
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                uint64_t nb = S.nbr[k][w] & rem.w[w];
                rem.w[w] &= ~nb;
                front.w[w] |= nb;
            }
        }
        if (reps) reps[beta] = int32_t(rep);
        ++beta;
    }
    return beta;
}

template <int NDIM>
__global__ void __launch_bounds__(256) k_classify_grid(const LinkTable *__restrict__ tab, FieldView F, Slab s,
                                                       int32_t *ptr,
                                                       uint32_t *sad_bits, uint32_t *max_bits, uint8_t *beta_out,
                                                       int *nan_flag) {
    __shared__ GridSmem<NDIM> S;
    load_tables<NDIM>(S, tab);
    const int64_t nown = s.v1 - s.v0;
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool active = i < nown;
    bool is_sad = false, is_max = false;
    if (active) {
        const int64_t v = s.v0 + i;
        const float fv = F.at(v);
        if (fv != fv) atomicOr(nan_flag, 1);
        int64_t best;
        auto m = upper_link<NDIM>(S, F, v, fv, &best);
        is_max = !m.any();
        int beta = is_max ? 0 : components<NDIM>(S, m, F, v, nullptr);
        is_sad = beta >= 2;
        ptr[i] = int32_t(best);
        if (beta_out) beta_out[i] = uint8_t(beta > 255 ? 255 : beta);
    }
    const uint32_t sb = __ballot_sync(0xffffffffu, is_sad);
    const uint32_t mb = __ballot_sync(0xffffffffu, is_max);
    if ((threadIdx.x & 31) == 0 && i < nown) {
        sad_bits[i >> 5] = sb;
        max_bits[i >> 5] = mb;
    }
}

template <int NDIM>
__global__ void __launch_bounds__(256) k_saddle_beta_grid(const LinkTable *__restrict__ tab, FieldView F,
                                                          const int32_t *__restrict__ saddles, int64_t n_sad,
                                                          int32_t *beta) {
    __shared__ GridSmem<NDIM> S;
    load_tables<NDIM>(S, tab);
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= n_sad) return;
    const int64_t v = saddles[j];
    const float fv = F.at(v);
    int64_t best;
    auto m = upper_link<NDIM>(S, F, v, fv, &best);
    beta[j] = components<NDIM>(S, m, F, v, nullptr);
}


// Per saddle: for every component, m = label[rep]; sort the (<= K) m values
// and reduce to unique (m, multiplicity) (reading L7).  Writes into the
// saddle's slots [slot_off[j], slot_off[j] + beta) and the unique count.
__device__ __forceinline__ void reduce_arcs(int32_t *ms, int b, int64_t off, int32_t *tmp_m, int32_t *tmp_mult,
                                            int32_t *n_unique_j) {
    for (int a = 1; a < b; ++a) {  // insertion sort (b <= link size)
        int32_t x = ms[a];
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
    *n_unique_j = u;
}

__device__ __forceinline__ void sort_reps(int32_t *reps, int b) {
    for (int a = 1; a < b; ++a) {
        int32_t x = reps[a];
        int c = a - 1;
        while (c >= 0 && reps[c] > x) {
            reps[c + 1] = reps[c];
            --c;
        }
        reps[c + 1] = x;
    }
}

template <int NDIM>
__global__ void __launch_bounds__(128) k_arcs_grid(const LinkTable *__restrict__ tab, FieldView F,
                                                   const int32_t *__restrict__ saddles, int64_t n_sad,
                                                   const int64_t *__restrict__ slot_off, LabelView lv,
                                                   int32_t *tmp_m, int32_t *tmp_mult, int32_t *n_unique,
                                                   int64_t *raw_s, int64_t *raw_rep, int64_t *raw_m) {
    __shared__ GridSmem<NDIM> S;
    load_tables<NDIM>(S, tab);
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= n_sad) return;
    constexpr int K = GridSmem<NDIM>::K;
    int32_t reps[K];
    const int64_t v = saddles[j];
    const float fv = F.at(v);
    int64_t best;
    auto m = upper_link<NDIM>(S, F, v, fv, &best);
    int b = components<NDIM>(S, m, F, v, reps);
    sort_reps(reps, b);
    const int64_t off = slot_off[j];
    int32_t ms[K];
    for (int c = 0; c < b; ++c) {
        ms[c] = lv.at(reps[c]);
        if (raw_s) {
            raw_s[off + c] = v;
            raw_rep[off + c] = reps[c];
            raw_m[off + c] = ms[c];
        }
    }
    reduce_arcs(ms, b, off, tmp_m, tmp_mult, n_unique + j);
}

#define EG_DISPATCH_NDIM(ndim, CALL)           \
    switch (ndim) {                             \
        case 1: CALL(1); break;                 \
        case 2: CALL(2); break;                 \
        case 3: CALL(3); break;                 \
        case 4: CALL(4); break;                 \
        case 5: CALL(5); break;                 \
        case 6: CALL(6); break;                 \
        default: return cudaErrorInvalidValue;  \
    }

static inline unsigned blocks_for(int64_t n, int bs) { return unsigned((n + bs - 1) / bs); }

cudaError_t launch_classify_grid(const LinkTable *d_tab, int ndim, FieldView F, const Slab &s, int32_t *ptr,
                                 uint32_t *sad_bits, uint32_t *max_bits, uint8_t *beta_out, int *nan_flag,
                                 cudaStream_t st) {
    const int64_t n = s.v1 - s.v0;
    if (n <= 0) return cudaSuccess;
#define CALL(D) k_classify_grid<D><<<blocks_for(n, 256), 256, 0, st>>>(d_tab, F, s, ptr, sad_bits, max_bits, beta_out, nan_flag)
    EG_DISPATCH_NDIM(ndim, CALL)
#undef CALL
    return cudaGetLastError();
}

cudaError_t launch_saddle_beta_grid(const LinkTable *d_tab, int ndim, FieldView F, const int32_t *saddles,
                                    int64_t n_sad, int32_t *beta, cudaStream_t st) {
    if (n_sad <= 0) return cudaSuccess;
#define CALL(D) k_saddle_beta_grid<D><<<blocks_for(n_sad, 256), 256, 0, st>>>(d_tab, F, saddles, n_sad, beta)
    EG_DISPATCH_NDIM(ndim, CALL)
#undef CALL
    return cudaGetLastError();
}

cudaError_t launch_arcs_grid(const LinkTable *d_tab, int ndim, FieldView F, const int32_t *saddles, int64_t n_sad,
                             const int64_t *slot_off, LabelView lv,
                             int32_t *tmp_m, int32_t *tmp_mult, int32_t *n_unique, int64_t *raw_s, int64_t *raw_rep,
                             int64_t *raw_m, cudaStream_t st) {
    if (n_sad <= 0) return cudaSuccess;
#define CALL(D)                                                                                            \
    k_arcs_grid<D><<<blocks_for(n_sad, 128), 128, 0, st>>>(d_tab, F, saddles, n_sad, slot_off, lv, \
                                                           tmp_m, tmp_mult, n_unique, raw_s, raw_rep, raw_m)
    EG_DISPATCH_NDIM(ndim, CALL)
#undef CALL
    return cudaGetLastError();
}

}  // namespace eg
