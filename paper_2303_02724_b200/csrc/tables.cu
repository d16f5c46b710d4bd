// Host-side construction of the implicit Freudenthal link.
//
// The edge set of the tessellated grid is never stored ("can be stored
// implicitly"): every vertex uses the same list of offset vectors, and the
// link edges are the pairs of offsets that Alg. 1 accepts.  Built once per
// (ndim, dims) on the host, uploaded to the device.
#include <algorithm>
#include <cstring>
#include <numeric>

#include "eg_impl.h"

namespace eg {

static bool alg1_offsets_adjacent(const int8_t *a, const int8_t *b, int n) {
    // Alg. 1 on two vertices v+a, v+b: the coordinate differences must all lie
    // in {0, 1} or all in {0, -1}, and not all be zero (reading L6).
    bool pos = false, neg = false, other = false, nz = false;
    for (int i = 0; i < n; ++i) {
        int d = int(a[i]) - int(b[i]);
        if (d == 1) pos = true;
        else if (d == -1) neg = true;
        else if (d != 0) other = true;
        if (d != 0) nz = true;
    }
    return nz && !other && !(pos && neg);
}

LinkTable make_link_table(int ndim, const int64_t *dims) {
    LinkTable t;
    std::memset(&t, 0, sizeof(t));
    t.ndim = ndim;
    int64_t s = 1;
    for (int i = 0; i < ndim; ++i) {
        t.dims[i] = dims[i];
        t.stride[i] = s;
        s *= dims[i];
    }
    // offsets: +1 on a non-empty axis subset, or -1 on it (2 (2^n - 1))
    std::vector<std::vector<int8_t>> offs;
    for (uint32_t m = 1; m < (1u << ndim); ++m) {
        for (int sign : {+1, -1}) {
            std::vector<int8_t> d(8, 0);
            for (int i = 0; i < ndim; ++i)
                if (m & (1u << i)) d[i] = int8_t(sign);
            offs.push_back(d);
        }
    }
    auto delta = [&](const std::vector<int8_t> &d) {
        int64_t x = 0;
        for (int i = 0; i < ndim; ++i) x += int64_t(d[i]) * t.stride[i];
        return x;
    };
    // ascending linear offset; ties (possible only when some dim < 3, and then
    // at most one of the tied offsets is in-domain for any vertex) broken by
    // lexicographic order from the slowest axis
    std::stable_sort(offs.begin(), offs.end(), [&](const auto &a, const auto &b) {
        int64_t da = delta(a), db = delta(b);
        if (da != db) return da < db;
        for (int i = ndim - 1; i >= 0; --i)
            if (a[i] != b[i]) return a[i] < b[i];
        return false;
    });
    t.K = int32_t(offs.size());
    for (int k = 0; k < t.K; ++k) {
        std::memcpy(t.d[k], offs[k].data(), 8);
        t.delta[k] = delta(offs[k]);
    }
    if (t.K <= 128)   // explicit neighbour masks (the 3-D LUT builder); the kernels use the lattice closure
        for (int a = 0; a < t.K; ++a)
            for (int b = 0; b < t.K; ++b)
                if (a != b && alg1_offsets_adjacent(t.d[a], t.d[b], ndim)) t.nbr[a][b >> 6] |= 1ull << (b & 63);
    return t;
}

std::vector<uint8_t> make_beta_lut3(const LinkTable &t) {
    // beta0+ of every subset of the 14-vertex 3-D link: components of the
    // induced subgraph, by repeated neighbourhood expansion.
    std::vector<uint8_t> lut(1u << 14, 0);
    for (uint32_t m = 0; m < (1u << 14); ++m) {
        uint32_t rem = m;
        int beta = 0;
        while (rem) {
            uint32_t front = rem & (~rem + 1);
            rem &= ~front;
            while (front) {
                int k = __builtin_ctz(front);
                front &= front - 1;
                uint32_t nb = uint32_t(t.nbr[k][0]) & rem;
                rem &= ~nb;
                front |= nb;
            }
            ++beta;
        }
        lut[m] = uint8_t(beta);
    }
    return lut;
}

}  // namespace eg
