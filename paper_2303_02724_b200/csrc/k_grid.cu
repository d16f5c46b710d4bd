// Generic n-D grid kernels (n = 1..8): S1 steepest-ascent pointer, S3 upper-
// link components, and the per-saddle part of S4.  One thread per vertex, the
// way the paper's classification kernel is organised ("launching a CUDA
// thread for each vertex"); n <= 3 grids normally take the tiled kernel in
// k_grid3d.cu instead.
//
// beta0+ without a union-find (P:184 uses one).  The link offsets of the
// Freudenthal triangulation are +d and -e for nonempty subsets d, e of the n
// axes (d, e read as n-bit masks), and two link vertices are adjacent iff the
// difference of their offsets is again an offset:
//     +d1 ~ +d2  iff  d1 is a proper subset of d2 or vice versa,
//     -e1 ~ -e2  likewise,
//     +d  ~ -e   iff  d and e are disjoint (e is a subset of ~d).
// So a set of link vertices is a pair of 2^n-bit words P, N (bit d of P =
// offset +d), and one flood-fill step over ALL adjacencies at once is a
// subset / superset closure of a 2^n-bit word -- n shift-and-or steps each:
//     P' = U+ & (up(P) | down(P | rev(N))),   N' = U- & (up(N) | down(N | rev(P)))
// where rev(x) maps bit d to bit ~d.  A component is the fixed point from one
// seed bit; beta0+ is the number of seeds needed to exhaust U+ and U-.  The
// adjacency rule is pinned against the oracle's explicit link graph by the
// n = 1..6 parity tests.
#include <algorithm>
#include <cstdio>
#include <type_traits>

#include "eg_impl.h"

namespace eg {

// A 2^n-bit word for n = 7, 8 (M = 128, 256): K 64-bit limbs, bit i in limb
// i / 64.  Only what the lattice closure needs: bit ops, single-bit set,
// lowest-bit / pop, and the subset shifts (see Lattice::up / down).
template <int K>
struct Bits {
    uint64_t w[K];
    __host__ __device__ constexpr Bits() : w{} {}
    __host__ __device__ constexpr explicit Bits(uint64_t lo) : w{} { w[0] = lo; }
    __host__ __device__ static constexpr Bits bit(int i) {
        Bits r;
        r.w[i >> 6] = 1ull << (i & 63);
        return r;
    }
    __host__ __device__ constexpr Bits operator|(const Bits &o) const {
        Bits r;
        for (int k = 0; k < K; ++k) r.w[k] = w[k] | o.w[k];
        return r;
    }
    __host__ __device__ constexpr Bits operator&(const Bits &o) const {
        Bits r;
        for (int k = 0; k < K; ++k) r.w[k] = w[k] & o.w[k];
        return r;
    }
    __host__ __device__ constexpr Bits operator~() const {
        Bits r;
        for (int k = 0; k < K; ++k) r.w[k] = ~w[k];
        return r;
    }
    __host__ __device__ constexpr Bits &operator|=(const Bits &o) {
        for (int k = 0; k < K; ++k) w[k] |= o.w[k];
        return *this;
    }
    __host__ __device__ constexpr Bits &operator&=(const Bits &o) {
        for (int k = 0; k < K; ++k) w[k] &= o.w[k];
        return *this;
    }
    __host__ __device__ constexpr bool operator==(const Bits &o) const {
        for (int k = 0; k < K; ++k)
            if (w[k] != o.w[k]) return false;
        return true;
    }
    __host__ __device__ constexpr bool operator!=(const Bits &o) const { return !(*this == o); }
    __host__ __device__ constexpr explicit operator bool() const {
        for (int k = 0; k < K; ++k)
            if (w[k]) return true;
        return false;
    }
    __host__ __device__ constexpr bool test(int i) const { return (w[i >> 6] >> (i & 63)) & 1ull; }
    // shift left / right by s bits, s a power of two (the subset shifts)
    __host__ __device__ constexpr Bits shl(int s) const {
        Bits r;
        if (s >= 64) {
            const int q = s >> 6;
            for (int k = K - 1; k >= q; --k) r.w[k] = w[k - q];
        } else {
            for (int k = K - 1; k >= 0; --k) r.w[k] = (w[k] << s) | (k ? (w[k - 1] >> (64 - s)) : 0ull);
        }
        return r;
    }
    __host__ __device__ constexpr Bits shr(int s) const {
        Bits r;
        if (s >= 64) {
            const int q = s >> 6;
            for (int k = 0; k + q < K; ++k) r.w[k] = w[k + q];
        } else {
            for (int k = 0; k < K; ++k) r.w[k] = (w[k] >> s) | (k + 1 < K ? (w[k + 1] << (64 - s)) : 0ull);
        }
        return r;
    }
};

template <int NDIM, bool kWide = (NDIM > 6)>
struct Lattice {
    static constexpr int M = 1 << NDIM;  // subsets of the n axes
    using W = std::conditional_t<(M <= 32), uint32_t, uint64_t>;
    static constexpr int WB = 8 * sizeof(W);
    __host__ __device__ static constexpr W full() { return M == WB ? ~W(0) : ((W(1) << M) - 1); }
    // bits of the subsets that do not contain axis a
    __host__ __device__ static constexpr W without(int a) {
        W x = 0;
        for (int i = 0; i < M; ++i)
            if (!((i >> a) & 1)) x |= W(1) << i;
        return x;
    }
    __device__ __forceinline__ static W up(W x) {  // all supersets of members
#pragma unroll
        for (int a = 0; a < NDIM; ++a) x |= (x & without(a)) << (1 << a);
        return x;
    }
    __device__ __forceinline__ static W down(W x) {  // all subsets of members
#pragma unroll
        for (int a = 0; a < NDIM; ++a) x |= (x >> (1 << a)) & without(a);
        return x;
    }
    __device__ __forceinline__ static W rev(W x) {  // bit d -> bit (M-1-d) = ~d
        if constexpr (WB == 32) return __brev(x) >> (32 - M);
        else return W(__brevll(x));
    }
    __device__ __forceinline__ static W lowest(W x) { return x & (~x + 1); }
    __device__ __forceinline__ static int pop(W &x) {
        int b;
        if constexpr (WB == 32) b = __ffs(x) - 1;
        else b = __ffsll(x) - 1;
        x &= x - 1;
        return b;
    }
    __device__ __forceinline__ static W bit(int i) { return W(1) << i; }
    __device__ __forceinline__ static bool test(W x, int i) { return (x >> i) & 1; }
};

// n = 7, 8: the same closure on multi-limb words
template <int NDIM>
struct Lattice<NDIM, true> {
    static constexpr int M = 1 << NDIM;
    using W = Bits<M / 64>;
    __host__ __device__ static constexpr W full() { return ~W(); }
    __host__ __device__ static constexpr W without(int a) {
        W x;
        for (int i = 0; i < M; ++i)
            if (!((i >> a) & 1)) x |= W::bit(i);
        return x;
    }
    __device__ __forceinline__ static W up(W x) {
#pragma unroll
        for (int a = 0; a < NDIM; ++a) x |= (x & without(a)).shl(1 << a);
        return x;
    }
    __device__ __forceinline__ static W down(W x) {
#pragma unroll
        for (int a = 0; a < NDIM; ++a) x |= x.shr(1 << a) & without(a);
        return x;
    }
    __device__ __forceinline__ static W rev(W x) {   // bit d -> bit M-1-d
        W r;
#pragma unroll
        for (int k = 0; k < M / 64; ++k) r.w[M / 64 - 1 - k] = __brevll(x.w[k]);
        return r;
    }
    __device__ __forceinline__ static W lowest(W x) {
        W r;
#pragma unroll
        for (int k = 0; k < M / 64; ++k)
            if (x.w[k]) {
                r.w[k] = x.w[k] & (~x.w[k] + 1);
                break;
            }
        return r;
    }
    __device__ __forceinline__ static int pop(W &x) {
#pragma unroll
        for (int k = 0; k < M / 64; ++k)
            if (x.w[k]) {
                const int b = __ffsll(x.w[k]) - 1;
                x.w[k] &= x.w[k] - 1;
                return 64 * k + b;
            }
        return -1;
    }
    __device__ __forceinline__ static W bit(int i) { return W::bit(i); }
    __device__ __forceinline__ static bool test(const W &x, int i) { return x.test(i); }
};

// Per-grid constants, passed by value: every access with an unrolled (compile-
// time) index becomes a constant-bank operand.
template <int NDIM>
struct GridConst {
    int32_t dpos[1 << NDIM];  // linear offset of +d (N < 2^31)
    int32_t dneg[1 << NDIM];  // -dpos
    uint32_t dims[NDIM];
    uint32_t mag[NDIM];       // r / dims[a] = umulhi(r, mag[a]) >> sh[a] for r < 2^31
    int32_t sh[NDIM];
    int32_t dposP[1 << NDIM]; // offset of +d in the NaN-padded copy (every axis + 2)
    int32_t dnegP[1 << NDIM]; // -dposP (no negation per load)
    int32_t pstride[NDIM];    // strides of the padded copy
};

template <int NDIM>
static GridConst<NDIM> make_grid_const(const LinkTable &t) {
    GridConst<NDIM> S{};
    for (int d = 0; d < (1 << NDIM); ++d) {
        int64_t x = 0;
        for (int a = 0; a < NDIM; ++a)
            if ((d >> a) & 1) x += t.stride[a];
        S.dpos[d] = int32_t(x);
        S.dneg[d] = -int32_t(x);
    }
    {
        int64_t ps = 1;
        for (int a = 0; a < NDIM; ++a) {
            S.pstride[a] = int32_t(ps);
            ps *= t.dims[a] + 2;
        }
        for (int d = 0; d < (1 << NDIM); ++d) {
            int64_t x = 0;
            for (int a = 0; a < NDIM; ++a)
                if ((d >> a) & 1) x += S.pstride[a];
            S.dposP[d] = int32_t(x);
            S.dnegP[d] = -int32_t(x);
        }
    }
    for (int a = 0; a < NDIM; ++a) {
        // round-up reciprocal: with l = ceil(log2 D) and m = ceil(2^(31+l) / D),
        // floor(r m / 2^(31+l)) = floor(r / D) for every r < 2^31, since
        // m D - 2^(31+l) < D <= 2^l.  D = 1 is flagged by sh = -1.
        const uint32_t D = uint32_t(t.dims[a]);
        S.dims[a] = D;
        if (D <= 1) {
            S.mag[a] = 0u;
            S.sh[a] = -1;
        } else {
            int l = 0;
            while ((uint64_t(1) << l) < D) ++l;
            S.mag[a] = uint32_t(((uint64_t(1) << (31 + l)) + D - 1u) / D);
            S.sh[a] = l - 1;
        }
    }
    return S;
}

__device__ __forceinline__ float nan_f() { return __int_as_float(0x7fffffff); }

// The upper link of v as (U+, U-) and its gradient.  The
// link is truncated at the domain boundary (reading L3): +d is dropped when v
// sits on the upper face of an axis in d, -e on the lower face; a dropped
// offset reads as NaN, which compares false both ways.  The gradient is the
// highest link vertex in simulated-perturbation order (reading L1) -- if any
// link vertex is above v, the highest one is -- so it is tracked over the
// whole link: the offsets are scanned in ascending global index (-e for
// e = M-1 .. 1, then +d for d = 1 .. M-1; the linear offset of a mask is
// monotone in the mask over the axes of extent >= 2), and `>=` keeps the
// highest index among equal values.  *best = v for a maximum.
//
// kPlain: the field is one array holding the whole domain (one slab, no halo
// planes); a vertex whose whole link box lies inside it loads without
// clamping the dropped offsets.
template <int NDIM, bool kPlain, bool kPad = false>
__device__ __forceinline__ void upper_link(const GridConst<NDIM> &S, const FieldView &F, int64_t v, float fv,
                                           typename Lattice<NDIM>::W &Up, typename Lattice<NDIM>::W &Un,
                                           int64_t *best, const float *pad = nullptr, float *fv_out = nullptr) {
    using L = Lattice<NDIM>;
    using W = typename L::W;
    constexpr int M = L::M;
    W vp = L::full() & ~L::bit(0), vn = vp;
    uint32_t r = uint32_t(v);
    int32_t pidx = 0;          // kPad: v's cell in the padded copy
#pragma unroll
    for (int a = 0; a < NDIM; ++a) {
        const uint32_t D = S.dims[a];
        const uint32_t q = S.sh[a] < 0 ? r : (__umulhi(r, S.mag[a]) >> S.sh[a]);
        const uint32_t c = r - q * D;
        r = q;
        if constexpr (kPad) {
            pidx += int32_t(c + 1) * S.pstride[a];
        } else {
            if (c == 0) vn &= L::without(a);
            if (c + 1 == D) vp &= L::without(a);
        }
    }
    W up{}, un{};
    float bf = -INFINITY;
    int bk = 0;  // -e or +d of the highest link vertex so far
    // kSafe: every offset's address is inside the array, so the loads are
    // unconditional and a dropped offset is replaced by NaN afterwards
    auto scan = [&](auto load, auto safe) {
        constexpr bool kSafe = decltype(safe)::value;
#pragma unroll
        for (int e = M - 1; e >= 1; --e) {  // lower indices: above v iff f > fv
            const bool ok = L::test(vn, e);
            float fu;
            if constexpr (kSafe) {
                fu = load(S.dneg[e]);
                if (!ok) fu = nan_f();
            } else {
                fu = ok ? load(S.dneg[e]) : nan_f();
            }
            if (fu > fv) un |= L::bit(e);
            if (fu >= bf) {
                bf = fu;
                bk = -e;
            }
        }
#pragma unroll
        for (int d = 1; d < M; ++d) {  // higher indices: above v iff f >= fv
            const bool ok = L::test(vp, d);
            float fu;
            if constexpr (kSafe) {
                fu = load(S.dpos[d]);
                if (!ok) fu = nan_f();
            } else {
                fu = ok ? load(S.dpos[d]) : nan_f();
            }
            if (fu >= fv) up |= L::bit(d);
            if (fu >= bf) {
                bf = fu;
                bk = d;
            }
        }
    };
    if constexpr (kPad) {
        // the NaN border of the padded copy stands in for the truncated link
        // (reading L3): every offset loads, no per-offset domain test
        const float *p = pad + pidx;
        asm("" : "+l"(p));
        // f(v) from the padded copy too (its load issues with the neighbours')
        fv = __ldg(p);
        if (fv_out) *fv_out = fv;
        // running maximum by integer selects (FSEL issues at half rate on sm_100)
        auto keep = [&](float fu, int k) {
            asm("{\n\t.reg .pred q;\n\tsetp.ge.f32 q, %2, %3;\n\tselp.b32 %0, %2, %3, q;\n\tselp.b32 %1, %4, %5, q;\n\t}"
                : "=f"(bf), "=r"(bk)
                : "f"(fu), "f"(bf), "r"(k), "r"(bk));
        };
#pragma unroll
        for (int e = M - 1; e >= 1; --e) {
            const float fu = __ldg(p + S.dnegP[e]);
            if (fu > fv) un |= L::bit(e);
            keep(fu, -e);
        }
#pragma unroll
        for (int d = 1; d < M; ++d) {
            const float fu = __ldg(p + S.dposP[d]);
            if (fu >= fv) up |= L::bit(d);
            keep(fu, d);
        }
    } else if constexpr (kPlain) {
        // an opaque base keeps each address one wide multiply-add off it
        const float *p = F.own + (v - F.v0);
        asm("" : "+l"(p));
        const int64_t reach = S.dpos[M - 1];
        if (v - reach >= F.v0 && v + reach < F.v1)
            scan([&](int32_t off) { return __ldg(p + off); }, std::true_type{});
        else
            scan([&](int32_t off) { return __ldg(p + off); }, std::false_type{});
    } else {
        scan([&](int32_t off) { return F.at(v + off); }, std::false_type{});
    }
    Up = up;
    Un = un;
    *best = bool(up | un) ? v + (bk < 0 ? -S.dpos[-bk] : S.dpos[bk]) : v;
}

// beta0+  by lattice closure, see the file comment.  If reps !=
// null, also the highest vertex of every component (UpperLinkRep), in
// component order.
template <int NDIM>
__device__ __forceinline__ int components(const GridConst<NDIM> &S, typename Lattice<NDIM>::W Up,
                                          typename Lattice<NDIM>::W Un, const FieldView &F, int64_t v,
                                          int32_t *reps) {
    using L = Lattice<NDIM>;
    using W = typename L::W;
    W P = Up, N = Un;  // not yet assigned to a component
    int beta = 0;
    while (bool(P | N)) {
        // seed: the member with the most axes (the highest bit; +1 / -1 when
        // present, adjacent to every other member of its sign), so the closure
        // reaches the rest in fewer steps; the components do not depend on it
        W cp, cn;
        if constexpr (std::is_integral<W>::value) {
            auto top = [](W x) -> W {
                if constexpr (sizeof(W) == 4) return W(1) << (31 - __clz(x));
                else return W(1) << (63 - __clzll((long long)x));
            };
            cp = bool(P) ? top(P) : W{};
            cn = bool(P) ? W{} : top(N);
        } else {
            cp = bool(P) ? L::lowest(P) : W{};
            cn = bool(P) ? W{} : L::lowest(N);
        }
        for (;;) {
            const W np = Up & (L::up(cp) | L::down(cp | L::rev(cn)));
            const W nn = Un & (L::up(cn) | L::down(cn | L::rev(cp)));
            if (np == cp && nn == cn) break;
            cp = np;
            cn = nn;
            if (cp == P && cn == N) break;   // every unassigned upper vertex reached: nothing can grow
        }
        P &= ~cp;
        N &= ~cn;
        if (reps) {
            int64_t rep = -1;
            float rf = 0.f;
            while (bool(cn)) {
                const int64_t u = v - S.dpos[L::pop(cn)];
                const float fu = F.at(u);
                if (rep < 0 || fu > rf || (fu == rf && u > rep)) {
                    rep = u;
                    rf = fu;
                }
            }
            while (bool(cp)) {
                const int64_t u = v + S.dpos[L::pop(cp)];
                const float fu = F.at(u);
                if (rep < 0 || fu > rf || (fu == rf && u > rep)) {
                    rep = u;
                    rf = fu;
                }
            }
            reps[beta] = int32_t(rep);
        }
        ++beta;
    }
    return beta;
}

template <int NDIM, bool kPlain, bool kPad = false>
__global__ void __launch_bounds__(256) k_classify_grid(const __grid_constant__ GridConst<NDIM> S, FieldView F, Slab s,
                                                       int32_t *ptr, uint32_t *sad_bits, uint32_t *max_bits,
                                                       uint8_t *beta_out, int *nan_flag, const float *pad = nullptr) {
    const int64_t nown = s.v1 - s.v0;
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool active = i < nown;
    bool is_sad = false, is_max = false;
    if (active) {
        const int64_t v = s.v0 + i;
        float fv = kPad ? 0.f : F.at(v);
        int64_t best;
        typename Lattice<NDIM>::W up, un;
        upper_link<NDIM, kPlain, kPad>(S, F, v, fv, up, un, &best, pad, &fv);
        if (fv != fv) atomicOr(nan_flag, 1);
        is_max = !bool(up | un);
        const int beta = is_max ? 0 : components<NDIM>(S, up, un, F, v, nullptr);
        is_sad = beta >= 2;
        ptr[i] = int32_t(best);
        if (beta_out) beta_out[i] = uint8_t(beta > 255 ? 255 : beta);
    }
    const uint32_t sb = __ballot_sync(0xffffffffu, is_sad);
    const uint32_t mb = __ballot_sync(0xffffffffu, is_max);
    if ((threadIdx.x & 31) == 0 && active) {
        sad_bits[i >> 5] = sb;
        max_bits[i >> 5] = mb;
    }
}

template <int NDIM>
__global__ void __launch_bounds__(256) k_saddle_beta_grid(const __grid_constant__ GridConst<NDIM> S, FieldView F,
                                                          const int32_t *__restrict__ saddles, int64_t n_sad,
                                                          int32_t *beta) {
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= n_sad) return;
    const int64_t v = saddles[j];
    const float fv = F.at(v);
    int64_t best;
    typename Lattice<NDIM>::W up, un;
    upper_link<NDIM, false>(S, F, v, fv, up, un, &best);
    beta[j] = components<NDIM>(S, up, un, F, v, nullptr);
}

// Per saddle: for every component, m = label[rep]; sort the (<= K) m values
// and reduce to unique (m, multiplicity) (reading L7).  Writes into the
// saddle's slots [slot_off[j], slot_off[j] + beta) and the unique count.
__device__ __forceinline__ void reduce_arcs(int32_t *ms, int b, int64_t off, int32_t *tmp_m, int32_t *tmp_mult,
                                            int32_t *n_unique_j) {
    for (int a = 1; a < b; ++a) {  // insertion sort (b <= link size)
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
    *n_unique_j = u;
}

__device__ __forceinline__ void sort_reps(int32_t *reps, int b) {
    for (int a = 1; a < b; ++a) {
        const int32_t x = reps[a];
        int c = a - 1;
        while (c >= 0 && reps[c] > x) {
            reps[c + 1] = reps[c];
            --c;
        }
        reps[c + 1] = x;
    }
}

template <int NDIM>
__global__ void __launch_bounds__(128) k_arcs_grid(const __grid_constant__ GridConst<NDIM> S, FieldView F,
                                                   const int32_t *__restrict__ saddles, int64_t n_sad,
                                                   const int64_t *__restrict__ slot_off, LabelView lv,
                                                   int32_t *tmp_m, int32_t *tmp_mult, int32_t *n_unique,
                                                   int64_t *raw_s, int64_t *raw_rep, int64_t *raw_m,
                                                   int32_t *beta_out) {
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= n_sad) return;
    constexpr int K = 2 * ((1 << NDIM) - 1);
    int32_t reps[K];
    const int64_t v = saddles[j];
    const float fv = F.at(v);
    int64_t best;
    typename Lattice<NDIM>::W up, un;
    upper_link<NDIM, false>(S, F, v, fv, up, un, &best);
    const int b = components<NDIM>(S, up, un, F, v, reps);
    sort_reps(reps, b);
    if (beta_out) beta_out[j] = b;
    const int64_t off = slot_off ? slot_off[j] : j * K;
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


// ----------------------------------------------- arc geometry
// The integral line of a raw arc (s, rep, m): s, rep, then gradient steps
// (the steepest-ascent pointer recomputed from f at every vertex) until
// the maximum -- Alg. 2's path for that upper-link component.
// Pass 1 counts the vertices of every path, pass 2 writes them at the
// scanned offsets.
template <int NDIM>
__global__ void __launch_bounds__(128) k_arc_paths_grid(const __grid_constant__ GridConst<NDIM> S, FieldView F,
                                                        const int64_t *__restrict__ raw_s,
                                                        const int64_t *__restrict__ raw_rep, int64_t n_raw,
                                                        const int64_t *__restrict__ off, int64_t *len_or_out,
                                                        int32_t *nxt) {
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= n_raw) return;
    int64_t *out = off ? len_or_out + off[j] : nullptr;
    int64_t k = 0;
    if (out) out[k] = raw_s[j];
    ++k;
    int64_t v = raw_rep[j];
    for (;;) {
        if (out) out[k] = v;
        ++k;
        int64_t best;
        typename Lattice<NDIM>::W up, un;
        upper_link<NDIM, false>(S, F, v, F.at(v), up, un, &best);
        const bool top = !bool(up | un);    // a maximum
        if (nxt) nxt[v - F.v0] = int32_t(top ? v : best);   // the next step, for k_arc_paths_follow
        if (top) break;
        v = best;
    }
    if (!off) len_or_out[j] = k;
}

#define EG_DISPATCH_NDIM(ndim, CALL)           \
    switch (ndim) {                             \
        case 1: CALL(1); break;                 \
        case 2: CALL(2); break;                 \
        case 3: CALL(3); break;                 \
        case 4: CALL(4); break;                 \
        case 5: CALL(5); break;                 \
        case 6: CALL(6); break;                 \
        case 7: CALL(7); break;                 \
        case 8: CALL(8); break;                 \
        default: return cudaErrorInvalidValue;  \
    }

static inline unsigned blocks_for(int64_t n, int bs) { return unsigned((n + bs - 1) / bs); }

// the field into the interior of a copy padded by one NaN cell on every side
// of every axis (the border was filled with NaN bytes first)
template <int NDIM>
__global__ void __launch_bounds__(256) k_pad_grid(const __grid_constant__ GridConst<NDIM> S, const float *__restrict__ f,
                                                  int64_t n, float *pad) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        uint32_t r = uint32_t(i);
        int32_t pidx = 0;
#pragma unroll
        for (int a = 0; a < NDIM; ++a) {
            const uint32_t q = S.sh[a] < 0 ? r : (__umulhi(r, S.mag[a]) >> S.sh[a]);
            pidx += int32_t(r - q * S.dims[a] + 1) * S.pstride[a];
            r = q;
        }
        pad[pidx] = __ldg(f + i);
    }
}

int64_t padded_cells(const LinkTable &tab, int ndim) {
    int64_t c = 1;
    for (int a = 0; a < ndim; ++a) c *= tab.dims[a] + 2;
    return c;
}

cudaError_t launch_classify_grid(const LinkTable &tab, int ndim, FieldView F, const Slab &s, int32_t *ptr,
                                 uint32_t *sad_bits, uint32_t *max_bits, uint8_t *beta_out, int *nan_flag,
                                 cudaStream_t st, float *pad) {
    const int64_t n = s.v1 - s.v0;
    if (n <= 0) return cudaSuccess;
    const bool plain = F.lo == nullptr && F.hi == nullptr;
    if (pad && plain && s.v0 == 0) {
        // one slab: classify on a NaN-padded copy (no per-offset domain tests)
        cudaError_t e = cudaMemsetAsync(pad, 0xff, sizeof(float) * size_t(padded_cells(tab, ndim)), st);
        if (e != cudaSuccess) return e;
#define CALL(D)                                                                                           \
    {                                                                                                     \
        const GridConst<D> G = make_grid_const<D>(tab);                                                   \
        k_pad_grid<D><<<unsigned(std::min<int64_t>(blocks_for(n, 256), 148 * 16)), 256, 0, st>>>(G, F.own, n, pad); \
        k_classify_grid<D, true, true><<<blocks_for(n, 256), 256, 0, st>>>(G, F, s, ptr, sad_bits, max_bits,   \
                                                                           beta_out, nan_flag, pad);      \
    }
        EG_DISPATCH_NDIM(ndim, CALL)
#undef CALL
        return cudaGetLastError();
    }
#define CALL(D)                                                                                           \
    if (plain)                                                                                            \
        k_classify_grid<D, true><<<blocks_for(n, 256), 256, 0, st>>>(             \
            make_grid_const<D>(tab), F, s, ptr, sad_bits, max_bits, beta_out, nan_flag);                                    \
    else                                                                                                  \
        k_classify_grid<D, false><<<blocks_for(n, 256), 256, 0, st>>>(           \
            make_grid_const<D>(tab), F, s, ptr, sad_bits, max_bits, beta_out, nan_flag)
    EG_DISPATCH_NDIM(ndim, CALL)
#undef CALL
    return cudaGetLastError();
}

cudaError_t launch_saddle_beta_grid(const LinkTable &tab, int ndim, FieldView F, const int32_t *saddles,
                                    int64_t n_sad, int32_t *beta, cudaStream_t st) {
    if (n_sad <= 0) return cudaSuccess;
#define CALL(D) k_saddle_beta_grid<D><<<blocks_for(n_sad, 256), 256, 0, st>>>(make_grid_const<D>(tab), F, saddles, n_sad, beta)
    EG_DISPATCH_NDIM(ndim, CALL)
#undef CALL
    return cudaGetLastError();
}

cudaError_t launch_arcs_grid(const LinkTable &tab, int ndim, FieldView F, const int32_t *saddles, int64_t n_sad,
                             const int64_t *slot_off, LabelView lv, int32_t *tmp_m, int32_t *tmp_mult,
                             int32_t *n_unique, int64_t *raw_s, int64_t *raw_rep, int64_t *raw_m, cudaStream_t st,
                             int32_t *beta_out) {
    if (n_sad <= 0) return cudaSuccess;
#define CALL(D)                                                                                              \
    k_arcs_grid<D><<<blocks_for(n_sad, 128), 128, 0, st>>>(make_grid_const<D>(tab), F, saddles, n_sad, slot_off, lv, tmp_m, \
                                                           tmp_mult, n_unique, raw_s, raw_rep, raw_m, beta_out)
    EG_DISPATCH_NDIM(ndim, CALL)
#undef CALL
    return cudaGetLastError();
}

cudaError_t launch_arc_paths_grid(const LinkTable &tab, int ndim, FieldView F, const int64_t *raw_s,
                                  const int64_t *raw_rep, int64_t n_raw, const int64_t *off, int64_t *len_or_out,
                                  cudaStream_t st, int32_t *nxt) {
    if (n_raw <= 0) return cudaSuccess;
#define CALL(D)                                                                                              \
    k_arc_paths_grid<D><<<blocks_for(n_raw, 128), 128, 0, st>>>(make_grid_const<D>(tab), F, raw_s, raw_rep, n_raw, off, \
                                                                len_or_out, nxt)
    EG_DISPATCH_NDIM(ndim, CALL)
#undef CALL
    return cudaGetLastError();
}

}  // namespace eg
