// Cross-slab label resolution (multi-GPU slabs and virtual partitions).
//
// The paper's hybrid mode pauses a gradient path when it reaches a block
// boundary and keeps a partial path (saddle, first, last) until the adjacent
// block is processed.  Here every slab (one GPU, or one virtual
// partition) first resolves paths locally; a path that leaves the slab ends
// in an "exit pointer" to a vertex of a halo plane (label = kUnresolved | x).
// The slabs then exchange the labels of their two boundary planes with their
// neighbours and jump over those values (bval / hval) until no boundary value
// is unresolved; a final pass rewrites every unresolved owned label.  Paths
// cross a slab boundary only through its two planes, so the exchange is a
// fixed 2 planes per neighbour per round.
#include <cstdlib>
#include <type_traits>

#include "eg_impl.h"

namespace eg {

static inline unsigned blocks_for(int64_t n, int bs) { return unsigned((n + bs - 1) / bs); }

__global__ void k_flag_remote(int32_t *label, int64_t n, int64_t v0) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t w = label[i];
    if (w < v0 || w >= v0 + n) label[i] = int32_t(uint32_t(w) | kUnresolved);
}

cudaError_t launch_flag_remote(int32_t *label, int64_t n, int64_t v0, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    k_flag_remote<<<blocks_for(n, 256), 256, 0, st>>>(label, n, v0);
    return cudaGetLastError();
}

// value of owned vertex g: its label followed through owned vertices until it
// is final or points to the first vertex of its path outside the slab (a
// vertex of a halo plane: a path changes the slowest coordinate by <= 1 per step)
__device__ __forceinline__ int32_t local_value(const int32_t *label, int64_t g, int64_t v0, int64_t v1) {
    int32_t w = label[g - v0];
    while (w < 0) {
        const int64_t x = w & 0x7fffffff;
        if (x < v0 || x >= v1) break;
        w = __ldcg(label + (x - v0));
    }
    return w;
}

__global__ void k_bval_init(const int32_t *label, Slab s, int32_t *bval) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= 2 * s.plane) return;
    const int64_t g = i < s.plane ? s.v0 + i : s.v1 - s.plane + (i - s.plane);
    bval[i] = local_value(label, g, s.v0, s.v1);
}

cudaError_t launch_bval_init(const int32_t *label, const Slab &s, int32_t *bval, cudaStream_t st) {
    k_bval_init<<<blocks_for(2 * s.plane, 256), 256, 0, st>>>(label, s, bval);
    return cudaGetLastError();
}

__global__ void k_bval_update(int32_t *bval, const int32_t *__restrict__ hlo, const int32_t *__restrict__ hhi, Slab s,
                              unsigned long long *unresolved, const unsigned long long *prev) {
    if (prev && *prev == 0) return;             // converged in an earlier round of this batch
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    bool still = false;
    if (i < 2 * s.plane) {
        int32_t w = bval[i];
        if (w < 0) {
            const int64_t x = w & 0x7fffffff;          // a vertex of a halo plane
            int32_t nv = w;
            if (x >= s.v0 - s.plane && x < s.v0 && hlo) nv = hlo[x - (s.v0 - s.plane)];
            else if (x >= s.v1 && x < s.v1 + s.plane && hhi) nv = hhi[x - s.v1];
            if (nv >= 0) {
                w = nv;
            } else {
                const int64_t x2 = nv & 0x7fffffff;    // the neighbour's path continues at x2
                if (x2 >= s.v0 && x2 < s.v0 + s.plane) w = bval[x2 - s.v0];
                else if (x2 >= s.v1 - s.plane && x2 < s.v1) w = bval[s.plane + (x2 - (s.v1 - s.plane))];
                // else: x2 lies beyond the neighbour; wait for it to resolve x
            }
            bval[i] = w;
            still = w < 0;
        }
    }
    if (__any_sync(0xffffffffu, still)) {
        const unsigned c = __popc(__ballot_sync(0xffffffffu, still));
        if ((threadIdx.x & 31) == 0) atomicAdd(unresolved, (unsigned long long)c);
    }
}

cudaError_t launch_bval_update(int32_t *bval, const int32_t *hval_lo, const int32_t *hval_hi, const Slab &s,
                               unsigned long long *unresolved, cudaStream_t st, const unsigned long long *prev) {
    k_bval_update<<<blocks_for(2 * s.plane, 256), 256, 0, st>>>(bval, hval_lo, hval_hi, s, unresolved, prev);
    return cudaGetLastError();
}

// Final pass.  A warp owns kW words of owned vertices (32 kW vertices); the
// loads of all of them are issued before any is used (memory-level
// parallelism for the dependent gather), and only changed labels are stored.
// (kW = 6 words per warp at full occupancy measured best for the one-slab
// chase: C3 3.13 ms vs 3.27 at kW = 4 or 8, 3.75 at 12; the smooth F1-1024
// field prefers 8, 4.59 vs 5.18 ms; 128-thread blocks retire a block held by
// one long chain sooner: C3 3.09 vs 3.12 ms at 256 or 64)
// kStats (EG_STATS): hist[k] += vertices whose chase followed k exit
// pointers (k >= 15 in hist[15]), hist[16] = max over vertices.
constexpr int kW = 6;
template <bool kStats>
__global__ void __launch_bounds__(128, 16) k_finalize(int32_t *label, const uint32_t *__restrict__ bits, int64_t v0,
                                                  int64_t v1, unsigned long long *hist) {
    const int64_t n = v1 - v0;
    const int64_t words = (n + 31) / 32;
    const int64_t w0 = (int64_t(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5)) * kW;
    if (w0 >= words) return;
    const int lane = threadIdx.x & 31;
    bool need[kW];
    int32_t e[kW];
#pragma unroll
    for (int k = 0; k < kW; ++k) {
        const int64_t i = (w0 + k) * 32 + lane;
        if (bits) {
            const uint32_t b = (w0 + k < words) ? __ldg(bits + w0 + k) : 0u;
            need[k] = (b >> lane) & 1u;
        } else {
            need[k] = i < n;
        }
    }
#pragma unroll
    for (int k = 0; k < kW; ++k) e[k] = need[k] ? label[(w0 + k) * 32 + lane] : 0;
#pragma unroll
    for (int k = 0; k < kW; ++k) need[k] = need[k] && e[k] < 0;
    {
        // every exit target lies in [v0, v1) (one slab; several slabs: the
        // array then spans the halo planes, whose values are final).  Its label
        // is final when the exit list was resolved first (k_resolve_exits);
        // otherwise the chain is chased here, through L1-cached loads (race-benign: every value
        // ever stored is a later vertex of the same ascending path or the
        // final label, and a root's label is final before this pass, so a
        // stale value only lengthens a walk).  Measured on C3 / F1-512 /
        // F1-1024: volatile loads + memoising the final label in the first
        // target 3281 / - / 8085 us; L1 + memo 3094 / 726 / 6021; L1 without
        // memo 3130 / 353 / 5180 (kept: the memo stores keep hitting lines
        // the other SMs' L1s still hold stale, so every reader re-walks and
        // re-stores); whole-chain compression 5x slower.
#pragma unroll
        for (int k = 0; k < kW; ++k)
            if (need[k]) e[k] = label[(e[k] & 0x7fffffff) - v0];
        int hops[kW];
#pragma unroll
        for (int k = 0; k < kW; ++k) {
            hops[k] = need[k] ? 1 : 0;
            if (need[k] && e[k] < 0) {
                int32_t w = e[k];
                do {
                    w = __ldca(label + ((w & 0x7fffffff) - v0));
                    if (kStats) ++hops[k];
                } while (w < 0);
                e[k] = w;
            }
        }
        if (kStats) {
            int mx = 0;
#pragma unroll
            for (int k = 0; k < kW; ++k) {
                if (need[k]) atomicAdd(hist + min(hops[k], 15), 1ull);
                mx = max(mx, hops[k]);
            }
            mx = __reduce_max_sync(0xffffffffu, unsigned(mx));
            if (lane == 0 && mx) atomicMax(hist + 16, (unsigned long long)mx);
        }
#pragma unroll
        for (int k = 0; k < kW; ++k)
            if (need[k]) label[(w0 + k) * 32 + lane] = e[k];
    }
}

// The one-slab label pass split by tile faces (3-D grid, one slab, tiles of
// 16 planes x 16 rows starting at the slab's first plane / row 0).  Every exit
// target is a halo cell of the tile the path leaves, i.e. a vertex of the
// outer layer of a neighbouring tile: on a z face (local plane z with
// z % 16 == 15 or == 0 next to a tile boundary), on a y face (row y likewise)
// or on an x face.  Pass 0 finishes the z-face plane pairs (12.5 % of the
// vertices), pass 1 (optional) the y-face row pairs of the other planes, pass
// 2 everything else: a chain of pass 2 that leaves its tile through a z face
// ends one load later, at a label pass 0 already finished.  The chase is the
// one of k_finalize (race-benign the same way).  The per-vertex face tests are
// shifts and compares only: with the tile size a runtime value the `%` made
// pass 2 issue-bound (2.29 G vs 1.66 G warp instructions, +0.5 ms on C3).
constexpr int kFaceT = 16;         // tile planes (TZ) = tile rows (TY) of k_tile
struct FaceSplit {
    int32_t nx, ny, planes, ysplit;    // ysplit = 0: no pass 1, pass 2 takes the y-face rows too
    uint64_t m_nx, m_2nx;              // ceil(2^64 / d) for d = nx, 2 nx (0 when d == 1)
};

__device__ __forceinline__ uint32_t fdiv(uint32_t k, uint64_t m) { return m ? uint32_t(__umul64hi(k, m)) : k; }

__device__ __forceinline__ bool face_pair(int32_t z, int32_t n) {   // z in a pair (16 j - 1, 16 j), 0 < 16 j < n
    const int32_t r = z & (kFaceT - 1);
    return (r == kFaceT - 1 && z + 1 < n) || (r == 0 && z > 0);
}

template <bool kStats, int kW>
__global__ void __launch_bounds__(128, 16) k_finalize_faces(int32_t *label, int64_t v0, FaceSplit F, int pass,
                                                            unsigned long long *hist) {
    const int64_t plane = int64_t(F.nx) * F.ny;
    const int32_t z = blockIdx.y;   // pass 0: pair index; else the local plane
    int64_t base, count;
    if (pass == 0) {
        base = (int64_t(z + 1) * kFaceT - 1) * plane;
        count = 2 * plane;
    } else {
        if (face_pair(z, F.planes)) return;
        base = int64_t(z) * plane;
        count = pass == 1 ? int64_t((F.ny - 1) / kFaceT) * 2 * F.nx : plane;
    }
    const int64_t w0 = (int64_t(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5)) * kW;
    if (w0 * 32 >= count) return;
    const int lane = threadIdx.x & 31;
    bool need[kW];
    int32_t e[kW];
    int64_t at[kW];
#pragma unroll
    for (int k = 0; k < kW; ++k) {
        const uint32_t q = uint32_t((w0 + k) * 32 + lane);
        need[k] = q < count;
        if (pass == 1) {     // q -> run (one y-face row pair), offset within it
            const uint32_t run = fdiv(q, F.m_2nx);
            at[k] = base + (int64_t(run + 1) * kFaceT - 1) * F.nx + (q - run * 2 * uint32_t(F.nx));
        } else {
            at[k] = base + q;
            if (pass == 2 && F.ysplit && need[k]) need[k] = !face_pair(int32_t(fdiv(q, F.m_nx)), F.ny);
        }
    }
#pragma unroll
    for (int k = 0; k < kW; ++k) e[k] = need[k] ? label[at[k]] : 0;
#pragma unroll
    for (int k = 0; k < kW; ++k) need[k] = need[k] && e[k] < 0;
#pragma unroll
    for (int k = 0; k < kW; ++k)
        if (need[k]) e[k] = label[(e[k] & 0x7fffffff) - v0];
    int hops[kW];
#pragma unroll
    for (int k = 0; k < kW; ++k) {
        hops[k] = need[k] ? 1 : 0;
        if (need[k] && e[k] < 0) {
            int32_t w = e[k];
            do {
                w = __ldca(label + ((w & 0x7fffffff) - v0));
                if (kStats) ++hops[k];
            } while (w < 0);
            e[k] = w;
        }
    }
    if (kStats) {
        int mx = 0;
#pragma unroll
        for (int k = 0; k < kW; ++k) {
            if (need[k]) atomicAdd(hist + min(hops[k], 15), 1ull);
            mx = max(mx, hops[k]);
        }
        mx = __reduce_max_sync(0xffffffffu, unsigned(mx));
        if (lane == 0 && mx) atomicMax(hist + 16, (unsigned long long)mx);
    }
#pragma unroll
    for (int k = 0; k < kW; ++k)
        if (need[k]) label[at[k]] = e[k];
}

static uint64_t div_magic(int64_t d) {
    if (d <= 1) return 0;
    const unsigned __int128 one = static_cast<unsigned __int128>(1) << 64;
    return uint64_t((one + uint64_t(d) - 1) / uint64_t(d));
}

cudaError_t launch_finalize_faces(int32_t *label, int64_t v0, int64_t nx, int64_t ny, int64_t planes, int tz, int ty,
                                  int ysplit, int passes, cudaStream_t st, unsigned long long *hist) {
    if (nx * ny * planes <= 0) return cudaSuccess;
    if (tz != kFaceT || ty != kFaceT) return cudaErrorInvalidValue;
    const FaceSplit F{int32_t(nx), int32_t(ny), int32_t(planes), ysplit, div_magic(nx), div_magic(2 * nx)};
    const int64_t plane = nx * ny;
    const int64_t zpairs = (planes - 1) / tz, ypair_words = ((ny - 1) / ty) * 2 * nx / 32 + 1;
    const char *kv = std::getenv("EG_FIN_KW");       // tuning knob: words per warp (4, 6, 8, 12)
    const int kw = kv ? std::atoi(kv) : 6;
    for (int pass = 0; pass < 3; ++pass) {
        const int64_t gy = pass == 0 ? zpairs : planes;
        const int64_t words = pass == 0 ? (2 * plane + 31) / 32 : pass == 1 ? ypair_words : (plane + 31) / 32;
        if (!((passes >> pass) & 1) || gy <= 0 || (pass == 1 && (ny <= ty || !ysplit))) continue;
        auto go = [&](auto kwc) {
            constexpr int K = decltype(kwc)::value;
            const dim3 grid(unsigned((words + 4 * K - 1) / (4 * K)), unsigned(gy));
            if (hist)
                k_finalize_faces<true, K><<<grid, 128, 0, st>>>(label, v0, F, pass, hist);
            else
                k_finalize_faces<false, K><<<grid, 128, 0, st>>>(label, v0, F, pass, nullptr);
        };
        if (kw == 4) go(std::integral_constant<int, 4>{});
        else if (kw == 8) go(std::integral_constant<int, 8>{});
        else if (kw == 12) go(std::integral_constant<int, 12>{});
        else go(std::integral_constant<int, 6>{});
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

// The one-slab label pass in z-chunks, for the end-to-end pipeline of
// eg_compute_host (k_grid3d.cu, tiled3d_local): chunk k of the owned words
// is finalised as soon as the tile kernel has labelled chunk k + 1, so its
// labels can travel to the host while later chunks of the field are still
// arriving.  A chain is followed only through vertices the tile kernel has
// labelled (local index < lim); one that reaches beyond keeps its progress
// (kFlag | the vertex it stopped at) and its index is appended to `list` for
// k_finalize_list, which runs once every chunk is labelled.
template <bool kStats>
__global__ void __launch_bounds__(128, 16) k_finalize_chunk(int32_t *label, int64_t w_begin, int64_t w_end, int64_t n,
                                                        int64_t v0, int64_t lim, int32_t *list,
                                                        unsigned long long *list_n, int64_t list_cap,
                                                        unsigned long long *hist) {
    const int64_t w0 = w_begin + (int64_t(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5)) * kW;
    if (w0 >= w_end) return;
    const int lane = threadIdx.x & 31;
    bool need[kW];
    int32_t e[kW];
#pragma unroll
    for (int k = 0; k < kW; ++k) {
        const int64_t i = (w0 + k) * 32 + lane;
        need[k] = w0 + k < w_end && i < n;
    }
#pragma unroll
    for (int k = 0; k < kW; ++k) e[k] = need[k] ? label[(w0 + k) * 32 + lane] : 0;
#pragma unroll
    for (int k = 0; k < kW; ++k) need[k] = need[k] && e[k] < 0;
    int hops[kW];
    bool unres[kW];
    // the first hop of every word's chains first (independent loads in flight)
#pragma unroll
    for (int k = 0; k < kW; ++k) {
        hops[k] = 0;
        unres[k] = false;
        if (need[k]) {
            const int64_t x = int64_t(e[k] & 0x7fffffff) - v0;
            if (x >= lim) unres[k] = true;              // not labelled by the tile kernel yet
            else {
                e[k] = label[x];
                hops[k] = 1;
            }
        }
    }
#pragma unroll
    for (int k = 0; k < kW; ++k) {
        if (need[k] && !unres[k] && e[k] < 0) {
            int32_t w = e[k];
            do {
                const int64_t x = int64_t(w & 0x7fffffff) - v0;
                if (x >= lim) {
                    unres[k] = true;
                    break;
                }
                w = __ldca(label + x);        // race-benign as in k_finalize
                if (kStats) ++hops[k];
            } while (w < 0);
            e[k] = w;
        }
    }
#pragma unroll
    for (int k = 0; k < kW; ++k)
        if (need[k]) label[(w0 + k) * 32 + lane] = e[k];
#pragma unroll
    for (int k = 0; k < kW; ++k) {
        const uint32_t b = __ballot_sync(0xffffffffu, unres[k]);
        if (b) {
            unsigned long long base = 0;
            if (lane == 0) base = atomicAdd(list_n, (unsigned long long)__popc(b));
            base = __shfl_sync(0xffffffffu, base, 0);
            const unsigned long long j = base + __popc(b & ((1u << lane) - 1u));
            if (unres[k] && j < (unsigned long long)list_cap) list[j] = int32_t((w0 + k) * 32 + lane);
        }
    }
    if (kStats) {
        int mx = 0;
#pragma unroll
        for (int k = 0; k < kW; ++k) {
            if (need[k] && !unres[k]) atomicAdd(hist + min(hops[k], 15), 1ull);
            mx = max(mx, hops[k]);
        }
        mx = __reduce_max_sync(0xffffffffu, unsigned(mx));
        if (lane == 0 && mx) atomicMax(hist + 16, (unsigned long long)mx);
    }
}

// the vertices a chunk could not finish (every vertex is labelled by now); if
// the list overflowed, every owned label is checked instead (exact, slower)
template <bool kStats>
__global__ void __launch_bounds__(128) k_finalize_list(int32_t *label, const int32_t *__restrict__ list,
                                                       const unsigned long long *list_n, int64_t list_cap, int64_t v0,
                                                       int64_t n_all, unsigned long long *hist) {
    const int64_t nl = int64_t(*list_n);
    const bool all = nl > list_cap;
    const int64_t n = all ? n_all : nl;
    for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = all ? j : list[j];
        int32_t w = label[i];
        int h = 0;
        while (w < 0) {
            w = __ldca(label + (int64_t(w & 0x7fffffff) - v0));
            ++h;
        }
        if (h) label[i] = w;
        if (kStats && h) atomicAdd(hist + min(h, 15), 1ull);   // hops after the chunk stopped
    }
}

__global__ void k_gather_labels(const int32_t *__restrict__ label, const int32_t *__restrict__ list, int64_t n,
                                int32_t *out) {
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j < n) out[j] = label[list[j]];
}

cudaError_t launch_finalize_chunk(int32_t *label, int64_t w_begin, int64_t w_end, int64_t n, int64_t v0, int64_t lim,
                                  int32_t *list, unsigned long long *list_n, int64_t list_cap, cudaStream_t st,
                                  unsigned long long *hist) {
    if (w_end <= w_begin) return cudaSuccess;
    const unsigned blocks = blocks_for(w_end - w_begin, 4 * kW);
    if (hist)
        k_finalize_chunk<true><<<blocks, 128, 0, st>>>(label, w_begin, w_end, n, v0, lim, list, list_n, list_cap,
                                                        hist);
    else
        k_finalize_chunk<false><<<blocks, 128, 0, st>>>(label, w_begin, w_end, n, v0, lim, list, list_n, list_cap,
                                                         nullptr);
    return cudaGetLastError();
}

cudaError_t launch_finalize_list(int32_t *label, const int32_t *list, const unsigned long long *list_n,
                                 int64_t list_cap, int64_t v0, int64_t n_all, cudaStream_t st,
                                 unsigned long long *hist) {
    if (n_all <= 0) return cudaSuccess;
    const unsigned blocks = 148 * 16;
    if (hist)
        k_finalize_list<true><<<blocks, 128, 0, st>>>(label, list, list_n, list_cap, v0, n_all, hist);
    else
        k_finalize_list<false><<<blocks, 128, 0, st>>>(label, list, list_n, list_cap, v0, n_all, nullptr);
    return cudaGetLastError();
}

cudaError_t launch_gather_labels(const int32_t *label, const int32_t *list, int64_t n, int32_t *out,
                                 cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    k_gather_labels<<<blocks_for(n, 256), 256, 0, st>>>(label, list, n, out);
    return cudaGetLastError();
}

cudaError_t launch_finalize(int32_t *label, const uint32_t *bits, int64_t v0, int64_t v1, cudaStream_t st,
                            unsigned long long *hist) {
    const int64_t words = (v1 - v0 + 31) / 32;
    if (words <= 0) return cudaSuccess;
    if (hist)
        k_finalize<true><<<blocks_for(words, 4 * kW), 128, 0, st>>>(label, bits, v0, v1, hist);
    else
        k_finalize<false><<<blocks_for(words, 4 * kW), 128, 0, st>>>(label, bits, v0, v1, nullptr);
    return cudaGetLastError();
}

}  // namespace eg
