// Shared device passes: pointer jumping (S2), stable bitmap compaction of
// maxima / saddles (S3 node lists), scans and arc emission (S4).
#include <algorithm>

#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include "eg_impl.h"

namespace eg {

static inline unsigned blocks_for(int64_t n, int bs) { return unsigned((n + bs - 1) / bs); }

// ----------------------------------------------------------- S2 jumping
// Each round follows every vertex's pointer chain for up to kHops links and
// stores where it got to (P:205-208's path following, bounded).  Concurrent
// rounds are benign: a vertex's own entry is the only one it writes, and
// every value ever stored is a vertex further along the same ascending path,
// so a stale or a fresh read both lead to the path's end; entries already
// finished by other threads shortcut the walk.  Targets outside
// [v0, v0 + n) are terminal (remote vertices).  changed[round] is set when
// some chain was cut at kHops; a round after one that cut nothing exits at
// once (the chains are all terminal: max or remote).  Bounding the walk keeps
// a long monotone path from serialising one thread (the next round restarts
// from the stored ancestor, so the rounds still halve-or-better every chain).
constexpr int kHops = 32;

__global__ void __launch_bounds__(256) k_jump(int32_t *ptr, int64_t n, int64_t v0, int *changed, int round) {
    // converged earlier?  changed[round - 1] was written by the previous launch,
    // so a cached read is coherent (a volatile read from every thread would
    // queue ~N/32 requests on one L2 line)
    if (round > 0 && __ldg(&changed[round - 1]) == 0) return;
    bool cut = false;
    // grid-stride over a resident grid: a round that has nothing to do costs
    // one launch, not N/256 block launches
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int32_t p0 = ptr[i];
        int32_t p = p0;
        bool c = true;
#pragma unroll 1
        for (int h = 0; h < kHops; ++h) {
            const int64_t pi = int64_t(p) - v0;
            if (pi < 0 || pi >= n) {
                c = false;
                break;
            }
            const int32_t pp = __ldcg(ptr + pi);
            if (pp == p) {
                c = false;
                break;
            }
            p = pp;
        }
        if (p != p0) ptr[i] = p;
        cut |= c;
    }
    // one flag store per block at most (a single global flag hammered by
    // every warp serialises in L2)
    if (__syncthreads_or(cut) && threadIdx.x == 0 && *(volatile int *)&changed[round] == 0) changed[round] = 1;
}

cudaError_t launch_jump_round(int32_t *ptr, int64_t n, int64_t v0, int *changed, int round, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    // 8 blocks of 256 = 2048 threads: a full SM at this kernel's register count
    k_jump<<<unsigned(std::min<int64_t>(blocks_for(n, 256), int64_t(sms) * 8)), 256, 0, st>>>(ptr, n, v0, changed,
                                                                                               round);
    return cudaGetLastError();
}

// ------------------------------------------------------ bitmap compaction
// Stable: ids come out ascending.  Block b owns words [256 b, 256 b + 256).
constexpr int kCompactBS = 256;

__global__ void __launch_bounds__(kCompactBS) k_count_bits(const uint32_t *__restrict__ bits, int64_t words,
                                                           int32_t *chunk_cnt) {
    using BR = cub::BlockReduce<int, kCompactBS>;
    __shared__ typename BR::TempStorage tmp;
    const int64_t w = int64_t(blockIdx.x) * kCompactBS + threadIdx.x;
    int c = w < words ? __popc(bits[w]) : 0;
    int tot = BR(tmp).Sum(c);
    if (threadIdx.x == 0) chunk_cnt[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kCompactBS) k_emit_bits(const uint32_t *__restrict__ bits, int64_t words, int64_t n,
                                                          int64_t v0, const int64_t *__restrict__ chunk_off,
                                                          int32_t *out32, int64_t *out64) {
    using BS = cub::BlockScan<int, kCompactBS>;
    __shared__ typename BS::TempStorage tmp;
    const int64_t w = int64_t(blockIdx.x) * kCompactBS + threadIdx.x;
    uint32_t x = w < words ? bits[w] : 0u;
    if (w == words - 1 && (n & 31)) x &= (1u << (n & 31)) - 1u;   // tail
    int pre;
    BS(tmp).ExclusiveSum(__popc(x), pre);
    int64_t o = chunk_off[blockIdx.x] + pre;
    while (x) {
        const int b = __ffs(x) - 1;
        x &= x - 1;
        const int64_t id = v0 + w * 32 + b;
        if (out32) out32[o] = int32_t(id);
        if (out64) out64[o] = id;
        ++o;
    }
}

struct PadI32 {
    const int32_t *in;
    int64_t n;
    __host__ __device__ int64_t operator()(int64_t i) const { return i < n ? int64_t(in[i]) : 0; }
};

using PadIt = thrust::transform_iterator<PadI32, thrust::counting_iterator<int64_t>, int64_t>;

size_t scan_scratch_bytes(int64_t n) {
    size_t bytes = 0;
    PadIt it(thrust::counting_iterator<int64_t>(0), PadI32{nullptr, n});
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, it, (int64_t *)nullptr, n + 1);
    return bytes;
}

cudaError_t launch_scan_i32(const int32_t *in, int64_t *out, int64_t n, void *scratch, size_t scratch_bytes,
                            cudaStream_t st) {
    PadIt it(thrust::counting_iterator<int64_t>(0), PadI32{in, n});
    return cub::DeviceScan::ExclusiveSum(scratch, scratch_bytes, it, out, n + 1, st);
}

struct PadI64 {
    const int64_t *in;
    int64_t n;
    __host__ __device__ int64_t operator()(int64_t i) const { return i < n ? in[i] : 0; }
};
using PadIt64 = thrust::transform_iterator<PadI64, thrust::counting_iterator<int64_t>, int64_t>;

size_t scan64_scratch_bytes(int64_t n) {
    size_t bytes = 0;
    PadIt64 it(thrust::counting_iterator<int64_t>(0), PadI64{nullptr, n});
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, it, (int64_t *)nullptr, n + 1);
    return bytes;
}

cudaError_t launch_scan_i64(const int64_t *in, int64_t *out, int64_t n, void *scratch, size_t scratch_bytes,
                            cudaStream_t st) {
    PadIt64 it(thrust::counting_iterator<int64_t>(0), PadI64{in, n});
    return cub::DeviceScan::ExclusiveSum(scratch, scratch_bytes, it, out, n + 1, st);
}

size_t compact_scratch_bytes(int64_t n) {
    const int64_t words = (n + 31) / 32;
    const int64_t chunks = (words + kCompactBS - 1) / kCompactBS;
    size_t b = scan_scratch_bytes(chunks);
    // layout: [chunk_cnt int32 x chunks][chunk_off int64 x (chunks + 1)][cub scratch]
    return size_t(chunks) * 4 + 16 + size_t(chunks + 1) * 8 + 16 + b + 256;
}

cudaError_t launch_compact_bits(const uint32_t *bits, int64_t n, int64_t v0, void *scratch, int32_t *out32,
                                int64_t *out64, int64_t *d_count, cudaStream_t st) {
    const int64_t words = (n + 31) / 32;
    const int64_t chunks = (words + kCompactBS - 1) / kCompactBS;
    if (n <= 0) return cudaMemsetAsync(d_count, 0, sizeof(int64_t), st);
    char *p = static_cast<char *>(scratch);
    int32_t *cnt = reinterpret_cast<int32_t *>(p);
    p += (size_t(chunks) * 4 + 15) / 16 * 16 + 16;
    int64_t *off = reinterpret_cast<int64_t *>(p);
    p += (size_t(chunks + 1) * 8 + 15) / 16 * 16 + 16;
    const size_t sb = scan_scratch_bytes(chunks);
    k_count_bits<<<unsigned(chunks), kCompactBS, 0, st>>>(bits, words, cnt);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    // the tail word may carry junk bits above n only if the producer set them;
    // producers only set bits of active lanes, so counts are exact.
    e = launch_scan_i32(cnt, off, chunks, p, sb, st);
    if (e != cudaSuccess) return e;
    k_emit_bits<<<unsigned(chunks), kCompactBS, 0, st>>>(bits, words, n, v0, off, out32, out64);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return cudaMemcpyAsync(d_count, off + chunks, sizeof(int64_t), cudaMemcpyDeviceToDevice, st);
}

// emission using the chunk offsets a previous launch_count_bits left in `scratch`
cudaError_t launch_emit_counted(const uint32_t *bits, int64_t n, int64_t v0, const void *scratch, int32_t *out32,
                                int64_t *out64, cudaStream_t st) {
    const int64_t words = (n + 31) / 32;
    const int64_t chunks = (words + kCompactBS - 1) / kCompactBS;
    if (n <= 0) return cudaSuccess;
    const char *p = static_cast<const char *>(scratch);
    p += (size_t(chunks) * 4 + 15) / 16 * 16 + 16;
    const int64_t *off = reinterpret_cast<const int64_t *>(p);
    k_emit_bits<<<unsigned(chunks), kCompactBS, 0, st>>>(bits, words, n, v0, off, out32, out64);
    return cudaGetLastError();
}

cudaError_t launch_count_bits(const uint32_t *bits, int64_t n, void *scratch, int64_t *d_count, cudaStream_t st) {
    const int64_t words = (n + 31) / 32;
    const int64_t chunks = (words + kCompactBS - 1) / kCompactBS;
    if (n <= 0) return cudaMemsetAsync(d_count, 0, sizeof(int64_t), st);
    char *p = static_cast<char *>(scratch);
    int32_t *cnt = reinterpret_cast<int32_t *>(p);
    p += (size_t(chunks) * 4 + 15) / 16 * 16 + 16;
    int64_t *off = reinterpret_cast<int64_t *>(p);
    p += (size_t(chunks + 1) * 8 + 15) / 16 * 16 + 16;
    const size_t sb = scan_scratch_bytes(chunks);
    k_count_bits<<<unsigned(chunks), kCompactBS, 0, st>>>(bits, words, cnt);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    e = launch_scan_i32(cnt, off, chunks, p, sb, st);
    if (e != cudaSuccess) return e;
    return cudaMemcpyAsync(d_count, off + chunks, sizeof(int64_t), cudaMemcpyDeviceToDevice, st);
}

// ------------------------------------------------------------ arc emission
__global__ void k_emit_arcs(const int32_t *__restrict__ saddles, int64_t n_sad, const int64_t *__restrict__ slot_off,
                            int slot_stride, const int64_t *__restrict__ arc_off, const int32_t *__restrict__ tmp_m,
                            const int32_t *__restrict__ tmp_mult, const int32_t *__restrict__ n_unique,
                            int64_t *arc_s, int64_t *arc_m, int32_t *arc_mult) {
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= n_sad) return;
    const int64_t so = slot_off ? slot_off[j] : j * slot_stride, ao = arc_off[j];
    const int u = n_unique[j];
    const int64_t s = saddles[j];
    for (int k = 0; k < u; ++k) {
        arc_s[ao + k] = s;
        arc_m[ao + k] = tmp_m[so + k];
        arc_mult[ao + k] = tmp_mult[so + k];
    }
}

cudaError_t launch_emit_arcs(const int32_t *saddles, int64_t n_sad, const int64_t *slot_off, const int64_t *arc_off,
                             const int32_t *tmp_m, const int32_t *tmp_mult, const int32_t *n_unique,
                             int64_t *arc_s, int64_t *arc_m, int32_t *arc_mult, cudaStream_t st, int slot_stride) {
    if (n_sad <= 0) return cudaSuccess;
    k_emit_arcs<<<blocks_for(n_sad, 256), 256, 0, st>>>(saddles, n_sad, slot_off, slot_stride, arc_off, tmp_m,
                                                        tmp_mult, n_unique, arc_s, arc_m, arc_mult);
    return cudaGetLastError();
}

__global__ void k_narrow(const int64_t *__restrict__ in, int32_t *out, int64_t n) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) out[i] = int32_t(in[i]);
}

cudaError_t launch_narrow(const int64_t *in, int32_t *out, int64_t n, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    k_narrow<<<blocks_for(n, 256), 256, 0, st>>>(in, out, n);
    return cudaGetLastError();
}

__global__ void k_gather_beta(const uint8_t *__restrict__ beta8, int64_t v0, const int32_t *__restrict__ saddles,
                              int64_t n, int32_t *out) {
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j < n) out[j] = beta8[saddles[j] - v0];
}

cudaError_t launch_gather_beta(const uint8_t *beta8, int64_t v0, const int32_t *saddles, int64_t n, int32_t *out,
                               cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    k_gather_beta<<<blocks_for(n, 256), 256, 0, st>>>(beta8, v0, saddles, n, out);
    return cudaGetLastError();
}

__global__ void k_i32_to_i64(const int32_t *__restrict__ in, int64_t *out, int64_t n) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) out[i] = in[i];
}

cudaError_t launch_i32_to_i64(const int32_t *in, int64_t *out, int64_t n, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    k_i32_to_i64<<<blocks_for(n, 256), 256, 0, st>>>(in, out, n);
    return cudaGetLastError();
}


// ------------------------------------------------ arc bundling
// Saddles whose arcs reach exactly two distinct maxima {m1 < m2} are keyed by
// the pair (others by an "absent" key); after a radix sort by key the first
// thread of every pair's run keeps the highest saddle (value, then index) and
// drops the rest; kept saddles and their arcs are compacted by scans.
__global__ void k_bundle_keys(const int32_t *__restrict__ n_unique, const int64_t *__restrict__ arc_off,
                              const int64_t *__restrict__ arc_m, int64_t ns, uint64_t *keys, int32_t *idx,
                              int32_t *keep) {
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= ns) return;
    uint64_t k = ~0ull;
    if (n_unique[j] == 2) {
        const int64_t o = arc_off[j];
        k = (uint64_t(arc_m[o]) << 32) | uint64_t(arc_m[o + 1]);
    }
    keys[j] = k;
    idx[j] = int32_t(j);
    keep[j] = 1;
}

// order key of a saddle's value (order-preserving, -0 == +0: reading L2)
__global__ void k_bundle_vkeys(const int32_t *__restrict__ saddles, const float *__restrict__ f, int64_t f_base,
                               int64_t ns, uint32_t *vkey) {
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= ns) return;
    const float x = __ldg(f + (saddles[j] - f_base));
    const uint32_t b = x == 0.0f ? 0u : __float_as_uint(x);
    vkey[j] = b ^ ((b & 0x80000000u) ? 0xffffffffu : 0x80000000u);
}

__global__ void k_bundle_gather_keys(const uint64_t *__restrict__ keys, const int32_t *__restrict__ idx, int64_t ns,
                                     uint64_t *out) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < ns) out[i] = keys[idx[i]];
}

// After the stable sorts (value key, then pair key) every pair's run lists its
// saddles in ascending (value, index) order: the last one is the highest
// (SoS) and survives; the others of a run of two or more are dropped.  O(1)
// per saddle (a serial scan of every run by its first thread took 9 ms on C5,
// whose 187 maxima give runs of thousands of saddles).
__global__ void k_bundle_pick(const uint64_t *__restrict__ keys, const int32_t *__restrict__ idx, int64_t ns,
                              int32_t *keep) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= ns) return;
    const uint64_t k = keys[i];
    if (k == ~0ull) return;
    const bool last = i + 1 == ns || keys[i + 1] != k;
    if (!last) keep[idx[i]] = 0;
}

// kept counts: saddles (keep) and arcs (keep * n_unique), for the scans
__global__ void k_bundle_counts(const int32_t *__restrict__ keep, const int32_t *__restrict__ n_unique, int64_t ns,
                                int32_t *arc_cnt) {
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j < ns) arc_cnt[j] = keep[j] ? n_unique[j] : 0;
}

__global__ void k_bundle_emit(const int32_t *__restrict__ keep, const int64_t *__restrict__ s_pos,
                              const int64_t *__restrict__ a_pos, const int64_t *__restrict__ arc_off, int64_t ns,
                              const int64_t *__restrict__ sad64, const int32_t *__restrict__ sad32,
                              const int32_t *__restrict__ sbeta, const int32_t *__restrict__ n_unique,
                              const int64_t *__restrict__ arc_s, const int64_t *__restrict__ arc_m,
                              const int32_t *__restrict__ arc_mult, int64_t *o_sad64, int32_t *o_sad32,
                              int32_t *o_sbeta, int32_t *o_nu, int64_t *o_arc_s, int64_t *o_arc_m, int32_t *o_arc_mult) {
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= ns || !keep[j]) return;
    const int64_t p = s_pos[j];
    o_sad64[p] = sad64[j];
    o_sad32[p] = sad32[j];
    o_sbeta[p] = sbeta[j];
    o_nu[p] = n_unique[j];
    const int64_t a = a_pos[j], o = arc_off[j];
    for (int k = 0; k < n_unique[j]; ++k) {
        o_arc_s[a + k] = arc_s[o + k];
        o_arc_m[a + k] = arc_m[o + k];
        o_arc_mult[a + k] = arc_mult[o + k];
    }
}

size_t bundle_sort_bytes(int64_t ns) {
    size_t b = 0, b32 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, b, (const uint64_t *)nullptr, (uint64_t *)nullptr,
                                    (const int32_t *)nullptr, (int32_t *)nullptr, int(std::max<int64_t>(ns, 1)));
    cub::DeviceRadixSort::SortPairs(nullptr, b32, (const uint32_t *)nullptr, (uint32_t *)nullptr,
                                    (const int32_t *)nullptr, (int32_t *)nullptr, int(std::max<int64_t>(ns, 1)));
    return std::max(b, b32);
}

cudaError_t launch_bundle(const BundleArgs &B, cudaStream_t st) {
    const int64_t ns = B.ns;
    if (ns <= 0) return cudaSuccess;
    const unsigned nb = blocks_for(ns, 256);
    k_bundle_keys<<<nb, 256, 0, st>>>(B.n_unique, B.arc_off, B.arc_m, ns, B.keys, B.idx, B.keep);
    // saddle order (value, then index: idx starts ascending and the sorts are
    // stable), then the pair key: keys2 holds the two value-key arrays first
    uint32_t *vkey = reinterpret_cast<uint32_t *>(B.keys2), *vkey2 = vkey + ns;
    k_bundle_vkeys<<<nb, 256, 0, st>>>(B.sad32, B.f, B.f_base, ns, vkey);
    size_t bytes = B.sort_bytes;
    cudaError_t e = cub::DeviceRadixSort::SortPairs(B.sort_tmp, bytes, vkey, vkey2, B.idx, B.idx2, int(ns), 0, 32, st);
    if (e != cudaSuccess) return e;
    k_bundle_gather_keys<<<nb, 256, 0, st>>>(B.keys, B.idx2, ns, B.keys2);
    bytes = B.sort_bytes;
    e = cub::DeviceRadixSort::SortPairs(B.sort_tmp, bytes, B.keys2, B.keys, B.idx2, B.idx, int(ns), 0, 64, st);
    if (e != cudaSuccess) return e;
    k_bundle_pick<<<nb, 256, 0, st>>>(B.keys, B.idx, ns, B.keep);
    k_bundle_counts<<<nb, 256, 0, st>>>(B.keep, B.n_unique, ns, B.arc_cnt);
    if ((e = launch_scan_i32(B.keep, B.s_pos, ns, B.scan_tmp, B.scan_bytes, st)) != cudaSuccess) return e;
    if ((e = launch_scan_i32(B.arc_cnt, B.a_pos, ns, B.scan_tmp, B.scan_bytes, st)) != cudaSuccess) return e;
    k_bundle_emit<<<nb, 256, 0, st>>>(B.keep, B.s_pos, B.a_pos, B.arc_off, ns, B.sad64, B.sad32, B.sbeta, B.n_unique,
                                      B.arc_s, B.arc_m, B.arc_mult, B.o_sad64, B.o_sad32, B.o_sbeta, B.o_nu,
                                      B.o_arc_s, B.o_arc_m, B.o_arc_mult);
    return cudaGetLastError();
}

// ------------------------------------------- exact conversions to float32 (L21)
template <class T>
__device__ __forceinline__ float to_f32(T x) { return float(x); }
template <>
__device__ __forceinline__ float to_f32<__half>(__half x) { return __half2float(x); }
template <>
__device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }

template <class T>
__global__ void k_to_f32(const T *__restrict__ in, float *__restrict__ out, int64_t n) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        out[i] = to_f32(in[i]);
}

cudaError_t launch_to_f32(const void *in, int dtype, float *out, int64_t n, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    const unsigned nb = unsigned(std::min<int64_t>((n + 255) / 256, 148 * 16));
    switch (dtype) {
        case EG_DTYPE_F16: k_to_f32<__half><<<nb, 256, 0, st>>>(static_cast<const __half *>(in), out, n); break;
        case EG_DTYPE_BF16:
            k_to_f32<__nv_bfloat16><<<nb, 256, 0, st>>>(static_cast<const __nv_bfloat16 *>(in), out, n);
            break;
        case EG_DTYPE_U8: k_to_f32<uint8_t><<<nb, 256, 0, st>>>(static_cast<const uint8_t *>(in), out, n); break;
        case EG_DTYPE_I8: k_to_f32<int8_t><<<nb, 256, 0, st>>>(static_cast<const int8_t *>(in), out, n); break;
        case EG_DTYPE_U16: k_to_f32<uint16_t><<<nb, 256, 0, st>>>(static_cast<const uint16_t *>(in), out, n); break;
        case EG_DTYPE_I16: k_to_f32<int16_t><<<nb, 256, 0, st>>>(static_cast<const int16_t *>(in), out, n); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

// ------------------ exact float32 image of a wider type, when there is one
// float64 / (u)int32 / (u)int64 fields whose every value is exactly a float32
// (f32 data stored as f64, integers below 2^24, ...): the cast is then an
// order isomorphism of the values, so the graph on it is the type's own
// graph (reading L22) without the rank sort.  *inexact |= 1 if any value is
// not exactly representable (NaN included: the rank path rejects it).
__device__ __forceinline__ bool exact_back(double x, float f) { return double(f) == x; }
__device__ __forceinline__ bool exact_back(int32_t x, float f) {
    return f >= -2147483648.0f && f < 2147483648.0f && int32_t(f) == x;
}
__device__ __forceinline__ bool exact_back(uint32_t x, float f) { return f < 4294967296.0f && uint32_t(f) == x; }
__device__ __forceinline__ bool exact_back(int64_t x, float f) {
    return f >= -9.2233720e18f && f < 9.2233720e18f && int64_t(f) == x;
}
__device__ __forceinline__ bool exact_back(uint64_t x, float f) { return f < 1.8446744e19f && uint64_t(f) == x; }

template <typename T>
__global__ void k_exact_f32(const T *__restrict__ in, float *__restrict__ out, int64_t n, int *inexact) {
    bool bad = false;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const T x = in[i];
        const float f = float(x);
        out[i] = f;
        bad = bad || !exact_back(x, f);
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(inexact, 1);
}

cudaError_t launch_exact_f32(const void *in, int dtype, float *out, int64_t n, int *inexact, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    const unsigned nb = unsigned(std::min<int64_t>((n + 255) / 256, 148 * 16));
    switch (dtype) {
        case EG_DTYPE_F64: k_exact_f32<double><<<nb, 256, 0, st>>>(static_cast<const double *>(in), out, n, inexact); break;
        case EG_DTYPE_I32: k_exact_f32<int32_t><<<nb, 256, 0, st>>>(static_cast<const int32_t *>(in), out, n, inexact); break;
        case EG_DTYPE_U32: k_exact_f32<uint32_t><<<nb, 256, 0, st>>>(static_cast<const uint32_t *>(in), out, n, inexact); break;
        case EG_DTYPE_I64: k_exact_f32<int64_t><<<nb, 256, 0, st>>>(static_cast<const int64_t *>(in), out, n, inexact); break;
        case EG_DTYPE_U64: k_exact_f32<uint64_t><<<nb, 256, 0, st>>>(static_cast<const uint64_t *>(in), out, n, inexact); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

// ----------------------------- SoS-rank image of a wider type (reading L22)
// The method only ever compares values under the SoS order (a
// total order with ties broken by the vertex index), so a field and the
// permutation that ranks its vertices in that order have the same extremum
// graph.  A stable radix sort of order-preserving unsigned keys (the index
// order survives among equal keys) gives the rank p of every vertex; its
// float image is the normal float with bit pattern p + 2^23, a strictly
// increasing map on [0, 2^31 - 2^24 - 2^23), so every comparison downstream
// is exact and free of ties.  NaN inputs become NaN (the path flags them).
// reverse: rank N-1-p instead -- the reversed total order of reading L11,
// whose maximum graph is the minimum graph of the input.
// (IEEE: -0 == +0, so both map to the key of +0 and tie by index.)
template <class T>
struct OrderKey;
template <>
struct OrderKey<float> {
    using K = uint32_t;
    __device__ static K key(float x) {
        const uint32_t b = uint32_t(__float_as_int(x == 0.0f ? 0.0f : x));
        return (b >> 31) ? ~b : (b | 0x80000000u);
    }
    __device__ static bool nan(float x) { return x != x; }
};
template <>
struct OrderKey<double> {
    using K = uint64_t;
    __device__ static K key(double x) {
        const uint64_t b = uint64_t(__double_as_longlong(x == 0.0 ? 0.0 : x));
        return (b >> 63) ? ~b : (b | (uint64_t(1) << 63));
    }
    __device__ static bool nan(double x) { return x != x; }
};
template <>
struct OrderKey<int32_t> {
    using K = uint32_t;
    __device__ static K key(int32_t x) { return uint32_t(x) ^ 0x80000000u; }
    __device__ static bool nan(int32_t) { return false; }
};
template <>
struct OrderKey<uint32_t> {
    using K = uint32_t;
    __device__ static K key(uint32_t x) { return x; }
    __device__ static bool nan(uint32_t) { return false; }
};
template <>
struct OrderKey<int64_t> {
    using K = uint64_t;
    __device__ static K key(int64_t x) { return uint64_t(x) ^ (uint64_t(1) << 63); }
    __device__ static bool nan(int64_t) { return false; }
};
template <>
struct OrderKey<uint64_t> {
    using K = uint64_t;
    __device__ static K key(uint64_t x) { return x; }
    __device__ static bool nan(uint64_t) { return false; }
};

template <class T>
__global__ void k_rank_keys(const T *__restrict__ in, typename OrderKey<T>::K *__restrict__ key,
                            int32_t *__restrict__ idx, int64_t n) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        key[i] = OrderKey<T>::key(in[i]);
        idx[i] = int32_t(i);
    }
}

template <class T>
__global__ void k_rank_scatter(const T *__restrict__ in, const int32_t *__restrict__ idx, float *__restrict__ out,
                               int64_t n, bool reverse) {
    for (int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < n; p += int64_t(gridDim.x) * blockDim.x) {
        const int32_t v = idx[p];
        const int32_t r = int32_t(reverse ? n - 1 - p : p);
        out[v] = OrderKey<T>::nan(in[v]) ? __int_as_float(0x7fc00000) : __int_as_float(r + (1 << 23));
    }
}

template <class T>
static cudaError_t rank_typed(const T *in, float *out, int64_t n, void *scratch, size_t *bytes, bool reverse,
                              cudaStream_t st) {
    using K = typename OrderKey<T>::K;
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    const size_t kb = al(sizeof(K) * size_t(n)), ib = al(sizeof(int32_t) * size_t(n));
    size_t sort_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, (const K *)nullptr, (K *)nullptr, (const int32_t *)nullptr,
                                    (int32_t *)nullptr, int(n));
    const size_t need = 2 * kb + 2 * ib + al(sort_bytes);
    if (!scratch) {
        *bytes = need;
        return cudaSuccess;
    }
    if (*bytes < need) return cudaErrorInvalidValue;
    char *p = static_cast<char *>(scratch);
    K *k0 = reinterpret_cast<K *>(p), *k1 = reinterpret_cast<K *>(p + kb);
    int32_t *i0 = reinterpret_cast<int32_t *>(p + 2 * kb), *i1 = reinterpret_cast<int32_t *>(p + 2 * kb + ib);
    void *tmp = p + 2 * kb + 2 * ib;
    const unsigned nb = unsigned(std::min<int64_t>((n + 255) / 256, 148 * 16));
    k_rank_keys<T><<<nb, 256, 0, st>>>(in, k0, i0, n);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    size_t tb = sort_bytes;
    e = cub::DeviceRadixSort::SortPairs(tmp, tb, k0, k1, i0, i1, int(n), 0, int(sizeof(K) * 8), st);
    if (e != cudaSuccess) return e;
    k_rank_scatter<T><<<nb, 256, 0, st>>>(in, i1, out, n, reverse);
    return cudaGetLastError();
}

cudaError_t launch_rank_f32(const void *in, int dtype, float *out, int64_t n, void *scratch, size_t *bytes,
                            bool reverse, cudaStream_t st) {
    if (n <= 0 || n > kRankMaxN) return cudaErrorInvalidValue;
    switch (dtype) {
        case EG_DTYPE_F32: return rank_typed(static_cast<const float *>(in), out, n, scratch, bytes, reverse, st);
        case EG_DTYPE_F64: return rank_typed(static_cast<const double *>(in), out, n, scratch, bytes, reverse, st);
        case EG_DTYPE_I32: return rank_typed(static_cast<const int32_t *>(in), out, n, scratch, bytes, reverse, st);
        case EG_DTYPE_U32: return rank_typed(static_cast<const uint32_t *>(in), out, n, scratch, bytes, reverse, st);
        case EG_DTYPE_I64: return rank_typed(static_cast<const int64_t *>(in), out, n, scratch, bytes, reverse, st);
        case EG_DTYPE_U64: return rank_typed(static_cast<const uint64_t *>(in), out, n, scratch, bytes, reverse, st);
        default: return cudaErrorInvalidValue;
    }
}

// ------------------------------------------------- minimum graph (reading L11)
// The minimum graph of f is the maximum graph of g[i] = -f[N-1-i]: the point
// reflection x -> dims-1-x maps the Freudenthal grid onto itself and reverses
// the linear index, so "lower under the reversed SoS order of f" becomes
// "lower under the SoS order of g".  Outputs map back by i -> N-1-i, which
// reverses every sorted list.
__global__ void k_reflect_negate(const float *__restrict__ f, float *__restrict__ g, int64_t n) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        g[i] = -__ldg(f + (n - 1 - i));
}

// a[0..n) := reverse(a), each entry x mapped to N - 1 - x when map_ids
template <class T>
__global__ void k_reverse(T *a, int64_t n, int64_t N, bool map_ids) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < (n + 1) / 2;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t j = n - 1 - i;
        T x = a[i], y = a[j];
        if (map_ids) {
            x = T(N - 1 - int64_t(x));
            y = T(N - 1 - int64_t(y));
        }
        a[i] = y;
        a[j] = x;
    }
}

cudaError_t launch_reflect_negate(const float *f, float *g, int64_t n, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    k_reflect_negate<<<148 * 8, 256, 0, st>>>(f, g, n);
    return cudaGetLastError();
}

cudaError_t launch_reverse_i64(int64_t *a, int64_t n, int64_t N, bool map_ids, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    k_reverse<int64_t><<<unsigned(std::min<int64_t>((n + 511) / 512, 148 * 8)), 256, 0, st>>>(a, n, N, map_ids);
    return cudaGetLastError();
}

cudaError_t launch_reverse_i32(int32_t *a, int64_t n, int64_t N, bool map_ids, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    k_reverse<int32_t><<<unsigned(std::min<int64_t>((n + 511) / 512, 148 * 8)), 256, 0, st>>>(a, n, N, map_ids);
    return cudaGetLastError();
}

__global__ void k_nan_scan(const float *__restrict__ f, int64_t n, int *flag) {
    bool bad = false;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        bad |= (f[i] != f[i]);
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

cudaError_t launch_nan_scan(const float *f, int64_t n, int *flag, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    k_nan_scan<<<148 * 8, 256, 0, st>>>(f, n, flag);
    return cudaGetLastError();
}

}  // namespace eg
