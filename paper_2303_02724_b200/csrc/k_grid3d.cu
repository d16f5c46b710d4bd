// Tiled path for n <= 3 grids (2-D and 1-D grids are 3-D grids with unit
// axes: the Freudenthal link of a 2-D vertex is exactly the dz = 0 part of the
// 3-D link, Fig. 2).
//
// Pass T  (k_tile): one CTA per 32 x 16 x 16 tile (2 CTAs per SM).  The tile
//         plus a one-vertex halo ("ghost vertices") is brought into
//         shared memory by one TMA bulk-tensor copy (out-of-domain cells are
//         filled with NaN by the TMA unit); every thread walks one z-column and
//         computes, per vertex,
//           S1  the gradient = SoS argmax of the closed star,
//               separably: closed star = box(v) u box(v - 1), box(w) = w + {0,1}^3,
//               so the argmax is 2x2 in-plane maxima combined across z;
//           S3  the 14-bit upper mask -> a 2-bit class code (saddle: beta0+ >= 2, maximum: empty mask) from a 4 KB LUT
//               (Table 1; maximum iff the mask is empty).
//         The gradients are stored as 16-bit byte offsets into a pointer box
//         (also kept in registers for the thread's own column) and compressed
//         in shared memory (S2 inside the tile): every vertex ends at an
//         in-tile maximum (its final label) or at the first halo vertex on its
//         path (an exit: the path leaves the tile, the paper's partial path
//         P:296).  label[v] = global id of that root, with bit 31 set for
//         exits.  The box of the tile one resident-CTA count ahead is
//         prefetched into L2; the pointer-box template, LUT and plane table
//         arrive by bulk copies.
// Default (one slab, no exit list): the label pass (k_finalize_faces,
//         k_slab.cu) chases every exit -- first the z-face plane pairs of the
//         tile layers, then the rest, whose z-face exits end one load later.
// EG_ELIST=1: the distinct exit targets of every tile are appended to a list
//         E; k_resolve_exits follows label[] from each to its maximum, and
//         the label pass then needs one load per exiting vertex.
// All in-place updates are race-benign: every value ever stored on a chain is
// a later vertex of the same ascending path.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <algorithm>

#include "eg_tiled.h"

namespace eg {

constexpr int TX = 32, TY = kTileY, TZ = kTileZ;
constexpr int XO = 4;                                // box x of the tile's first column: boxes start at x0 - 4 (16-byte aligned)
constexpr int BX = TX + 2 * XO;                      // 40
constexpr int BY = TY + 2, BZ = TZ + 2;
constexpr int PL = BX * BY;                          // 720 cells per plane of the field box
constexpr int BOX = PL * BZ;                         // 12960 field-box cells = one TMA box
constexpr int PS = 1024;                             // pointer-box plane stride: cell r = bz * PS + by * BX + bx
constexpr int PBOX = BZ * PS;                        // 18432 cells; pointers are byte offsets 2 r < 65536 (16 bits)
// plane bz of the pointer box starts at byte bz * (2 PS + SKEW): the skew turns
// the plane stride from a multiple of 128 B (cells of three planes at one
// (x, y) in one bank: 2-way conflicts in the pointer gathers) into one that
// shifts the banks by 8 per plane; bz = offset >> 11 still holds, since
// 17 * SKEW + 2 * (PL - 1) < 2 PS
#ifndef EG_PB_SKEW
#define EG_PB_SKEW 32
#endif
constexpr int SKEW = EG_PB_SKEW;
constexpr int PSB = 2 * PS + SKEW;                   // plane stride in bytes
static_assert((BY * BX * 18 > 0) && 17 * SKEW + 2 * (18 * 40 - 1) < 2 * 1024, "skewed planes keep plane = offset >> 11");
constexpr int kThreads = TX * TY;                    // one z-column per thread
constexpr int kWarps = kThreads / 32;
constexpr int kLutWords = (1 << 14) / 16;            // 2 bits per 14-bit upper mask: beta0+ >= 2, beta0+ == 0
constexpr uint32_t kFlag = 0x80000000u;              // label bit 31: exit (not yet final)
constexpr int kMaxChunks = 32;                       // z-chunks of the eg_compute_host pipeline
#ifndef EG_S1_UNROLL
#define EG_S1_UNROLL 16
#endif
#ifndef EG_OUT_UNROLL
#define EG_OUT_UNROLL 16
#endif
constexpr int kS1Unroll = EG_S1_UNROLL, kOutUnroll = EG_OUT_UNROLL;   // z-loop unrolling (tuned on C3)
// the halo shell of a box (the cells a path can exit to): both z faces, and
// the y rows / x columns of the inner planes, over box x in [XO - 1, XO + TX]
constexpr int kShellW = TX + 2;
constexpr int kShell = 2 * BY * kShellW + (BZ - 2) * (2 * kShellW + 2 * (BY - 2));   // 2824
// shared memory: field box | pointer box | LUT | mbarrier + reduction | plane table
constexpr size_t kOffP = size_t(BOX) * 4;
constexpr size_t kOffL = kOffP + size_t(PBOX) * 2;
constexpr size_t kOffM = kOffL + size_t(kLutWords) * 4;
constexpr size_t kOffT = kOffM + 256;
constexpr size_t kTileSmem = kOffT + size_t(PL) * 4;   // ~92 KB -> 2 CTAs per SM
static_assert(2 * PBOX <= BOX * 4, "exit marks (1 byte per pointer-box byte offset) fit the dead field box");
static_assert(TZ == 16, "saddle / maximum column masks pack into one 32-bit word");

struct Tiled3D {
    uint32_t *d_lut = nullptr;
    unsigned char *d_tmpl = nullptr;                 // pointer-box image (shell cells self-pointing) + LUT, smem layout
    uint16_t *d_shell = nullptr;                     // pointer-box index of every shell cell
    bool ready = false;
    int64_t bdims[3] = {0, 0, 0};
    int64_t bz[2] = {-1, -1};                        // slab planes of the cached list
    int rounds = 2;
    int32_t *d_btiles = nullptr;                     // boundary tile list for the cached dims
    int32_t *d_ptab = nullptr;                       // plane table for nx = ptab_nx
    int64_t ptab_nx = -1;
    int64_t n_btiles = 0;
    int32_t *d_elist = nullptr;                      // exit targets E
    int64_t ecap = 0;
    unsigned long long *d_ecount = nullptr;          // [0] |E|, [1] maxima, [2] saddles, [3] unfinished labels
    int32_t *d_max = nullptr, *d_sad = nullptr;      // unordered maxima / saddles of the last call
    int64_t list_cap = 0;
    int64_t n_max = 0, n_sad = 0, v0 = 0, v1 = 0;
    void *d_sort_tmp = nullptr;                      // cub radix-sort scratch
    size_t sort_tmp_bytes = 0;
    int32_t *d_alt = nullptr;                        // sorted maxima (int32)
    int64_t alt_cap = 0;
    void *encode = nullptr;                          // cuTensorMapEncodeTiled
    int n_sm = 148;
    // eg_compute_host pipeline: events per chunk (H2D, tile, label), the
    // list of vertices a label chunk could not finish
    cudaEvent_t ev_io[3 * kMaxChunks + 2] = {};
    int32_t *d_fin_list = nullptr;
    int64_t fin_cap = 0;
};

void tiled3d_fin_list(const Tiled3D *t, const int32_t **list, const unsigned long long **count, int64_t *cap) {
    *list = t->d_fin_list;
    *count = t->d_ecount + 3;
    *cap = t->fin_cap;
}

Tiled3D *tiled3d_create() { return new Tiled3D(); }

void tiled3d_destroy(Tiled3D *t) {
    if (!t) return;
    if (t->d_lut) cudaFree(t->d_lut);
    if (t->d_tmpl) cudaFree(t->d_tmpl);
    if (t->d_shell) cudaFree(t->d_shell);
    if (t->d_btiles) cudaFree(t->d_btiles);
    if (t->d_ptab) cudaFree(t->d_ptab);
    if (t->d_elist) cudaFree(t->d_elist);
    if (t->d_ecount) cudaFree(t->d_ecount);
    if (t->d_max) cudaFree(t->d_max);
    if (t->d_sad) cudaFree(t->d_sad);
    if (t->d_sort_tmp) cudaFree(t->d_sort_tmp);
    if (t->d_alt) cudaFree(t->d_alt);
    if (t->d_fin_list) cudaFree(t->d_fin_list);
    for (auto &e : t->ev_io)
        if (e) cudaEventDestroy(e);
    delete t;
}

struct Dims3 {
    int32_t nx, ny, nz;
};

struct TileArgs {
    const float *f;                 // owned planes [z_lo, z_hi) of the slab
    const float *f_lo, *f_hi;       // halo planes z_lo - 1 and z_hi (neighbour slabs) or null
    int32_t z_lo, z_hi;
    int64_t v0;                     // global id of the first owned vertex
    int32_t *label;                 // owned labels (index v - v0)
    int32_t *max_list, *sad_list;   // maxima / saddles (global ids, unordered)
    int64_t list_cap;
    int *nan_flag;
    int32_t *elist;
    unsigned long long *ecount;     // [0] exit targets, [1] maxima, [2] saddles
    int64_t ecap;
    const uint32_t *lut;
    const unsigned char *tmpl;      // TMA launches: pointer-box template + LUT, bulk-copied at the tile start
    const int32_t *ptab;            // per box-plane cell: by * nx + bx, bit 31 = in-plane shell
    const uint16_t *shell;          // kShell pointer-box byte offsets
    const int32_t *btiles;          // boundary variant: packed tile ids
    int32_t tiles_x, tiles_y;       // interior variant: sub-box extents
    uint64_t mx, my;                // ceil(2^32 / tiles_x), ceil(2^32 / tiles_y): t / tiles = (t m) >> 32
    int32_t n_tiles;                // interior variant: tiles of the sub-box
    int3 origin;                    // interior variant: first interior tile
    int32_t rounds;                 // pointer-doubling rounds before the chase
    int32_t no_elist;               // one slab: no exit-target list (the finalize pass chases)
    int32_t tma;                    // field box by TMA (else plain row loads)
    int32_t prefetch;               // TMA launches: prefetch the box of tile blockIdx + prefetch into L2 (0: off)
    unsigned long long *exit_count; // EG_STATS: += vertices whose root is an exit (else null)
};

// ------------------------------------------------------------ TMA helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra LAB_WAIT;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

// A box may start outside the tensor (the TMA unit fills those cells with NaN)
// as long as its x start is 16-byte aligned (measured with tools/tma_probe:
// x = -4 loads, x = -1 faults).
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, uint64_t *bar, int x, int y, int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}

// L2 prefetch of a box (no shared-memory destination, no completion)
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap *map, int x, int y, int z) {
    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global [%0, {%1, %2, %3}];"
                 ::"l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z)
                 : "memory");
}

// one bulk copy global -> shared (16-byte aligned, size a multiple of 16),
// completing on the mbarrier like the tensor copy
__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// ------------------------------------------------------------ the tile kernel

struct VK {           // a value with its pointer-box offset from the centre vertex
    float v;
    int d;
};

// b wins ties: b is the later (higher-index) operand.  Both selects are
// integer SELs (full rate; FSEL issues at half rate on sm_100, measured with
// tools/pipe_probe).
__device__ __forceinline__ VK vmax(VK a, VK b) {
    VK r;
    asm("{\n\t.reg .pred p;\n\tsetp.ge.f32 p, %2, %3;\n\tselp.b32 %0, %2, %3, p;\n\tselp.b32 %1, %4, %5, p;\n\t}"
        : "=f"(r.v), "=r"(r.d)
        : "f"(b.v), "f"(a.v), "r"(b.d), "r"(a.d));
    return r;
}
// b is the earlier (lower-index) operand: it wins only if strictly greater
// (so ties keep the later a, and a NaN b never wins)
__device__ __forceinline__ VK vearlier(VK a, VK b) {
    VK r;
    asm("{\n\t.reg .pred p;\n\tsetp.gt.f32 p, %2, %3;\n\tselp.b32 %0, %2, %3, p;\n\tselp.b32 %1, %4, %5, p;\n\t}"
        : "=f"(r.v), "=r"(r.d)
        : "f"(b.v), "f"(a.v), "r"(b.d), "r"(a.d));
    return r;
}

// IEEE compares (no ftz: distinct denormals stay distinct, reading L2; a NaN
// compares false): m |= kBit if a > b (a >= b), one FSETP + one predicated add
template <uint32_t kBit>
__device__ __forceinline__ void or_if_gt(uint32_t &m, float a, float b) {
    asm("{\n\t.reg .pred p;\n\tsetp.gt.f32 p, %1, %2;\n\t@p or.b32 %0, %0, %3;\n\t}" : "+r"(m) : "f"(a), "f"(b), "n"(kBit));
}
template <uint32_t kBit>
__device__ __forceinline__ void or_if_ge(uint32_t &m, float a, float b) {
    asm("{\n\t.reg .pred p;\n\tsetp.ge.f32 p, %1, %2;\n\t@p or.b32 %0, %0, %3;\n\t}" : "+r"(m) : "f"(a), "f"(b), "n"(kBit));
}

// plain loads of box plane bz from `src` (a whole plane of the grid, row-major
// nx x ny) or NaN where the cell is outside the domain / src is null
__device__ __forceinline__ void load_plane(float *fbox, int bz, const float *src, int x0, int y0, const Dims3 &D,
                                           int tid) {
    for (int i = tid; i < PL; i += kThreads) {
        const int by = i / BX, bx = i - by * BX;
        const int gx = x0 + bx - XO, gy = y0 + by - 1;
        fbox[bz * PL + i] = (src && gx >= 0 && gx < D.nx && gy >= 0 && gy < D.ny)
                                ? __ldg(src + (int64_t(gy) * D.nx + gx))
                                : __int_as_float(0x7fffffff);
    }
}

// kPersist (interior tiles, TMA, one slab): one CTA per SM slot walks the
// tiles blockIdx.x, blockIdx.x + gridDim.x, ...; the LUT, the plane table and
// the self-pointing halo shell of the pointer box are staged once per CTA
// (the shell is never written afterwards), and the next tile's field box is
// requested by TMA as soon as S1 has consumed the current one, so the copy
// runs behind S2 and the label stores.
// kNoE: the launch has no exit list (A.no_elist known at compile time: the
// exit-mark stores and their flag test leave the output loop)
template <bool kInterior, bool kPersist, bool kStats = false, bool kNoE = false>
__global__ void __launch_bounds__(kThreads, 2)
    k_tile(const __grid_constant__ CUtensorMap tmap, TileArgs A, Dims3 D) {
    const bool no_elist = kNoE || A.no_elist;
    extern __shared__ __align__(128) unsigned char smem[];
    float *fbox = reinterpret_cast<float *>(smem);
    unsigned char *pb = smem + kOffP;
    // the pointer box holds byte offsets: a chase step is one load at base + value
    auto P = [pb](int b) -> uint16_t & { return *reinterpret_cast<uint16_t *>(pb + b); };
    const uint32_t pbase = smem_u32(pb);
    auto ld16 = [](uint32_t a) -> uint32_t {
        uint32_t v;
        asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
        return v;
    };
    uint32_t *lut = reinterpret_cast<uint32_t *>(smem + kOffL);
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + kOffM);
    uint32_t *red = reinterpret_cast<uint32_t *>(smem + kOffM + 16);                 // [kWarps] warp offsets
    unsigned long long *ebase = reinterpret_cast<unsigned long long *>(smem + kOffM + 16 + 4 * 32);
    int32_t *ptab = reinterpret_cast<int32_t *>(smem + kOffT);

    const int tid = threadIdx.x;
    const int tx = tid & 31, ty = tid >> 5;
    // tile t -> (bx, by, bz) of its origin (box coordinates in tiles)
    auto coords = [&](int t, int &bxo, int &byo, int &bzo) {
        if (kInterior) {
            const uint32_t q = uint32_t((uint64_t(t) * A.mx) >> 32);      // t / tiles_x (t * tiles_x < 2^32)
            bxo = t - int(q) * A.tiles_x + A.origin.x;
            const uint32_t q2 = uint32_t((uint64_t(q) * A.my) >> 32);     // q / tiles_y
            byo = int(q) - int(q2) * A.tiles_y + A.origin.y;
            bzo = int(q2) + A.origin.z;
        } else {
            const int packed = A.btiles[t];     // (bz << 20) | (by << 10) | bx
            bxo = packed & 1023;
            byo = (packed >> 10) & 1023;
            bzo = packed >> 20;
        }
    };
    // thread 0: request tile t's field box; with `tables` also the pointer-box
    // template (shell cells point to themselves, P:296 partial-path ends), the
    // LUT and the plane table -- three bulk copies instead of per-thread loops
    constexpr uint32_t kTmplBytes = uint32_t(kOffM - kOffP), kPtabBytes = uint32_t(PL * 4);
    static_assert(kTmplBytes % 16 == 0 && kPtabBytes % 16 == 0 && kOffP % 16 == 0 && kOffT % 16 == 0, "bulk copy");
    auto issue_tma = [&](int t, bool tables) {
        int bx, by, bz;
        coords(t, bx, by, bz);
        mbar_expect_tx(bar, uint32_t(BOX * 4) + (tables ? kTmplBytes + kPtabBytes : 0u));
        tma_load_3d(fbox, &tmap, bar, bx * TX - XO, by * TY - 1, A.z_lo + bz * TZ - 1 - A.z_lo);
        if (tables) {
            bulk_load(pb, A.tmpl, kTmplBytes, bar);
            bulk_load(ptab, A.ptab, kPtabBytes, bar);
        }
    };
    if (A.tma) {
        if (tid == 0) {
            mbar_init(bar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        if (tid == 0) {
            issue_tma(blockIdx.x, true);
            // the CTA that takes this slot about one tile-time later finds its box in L2
            const int tp = int(blockIdx.x) + A.prefetch;
            if (!kPersist && A.prefetch > 0 && tp < (kInterior ? A.n_tiles : int(gridDim.x))) {
                int bx, by, bz;
                coords(tp, bx, by, bz);
                tma_prefetch_3d(&tmap, bx * TX - XO, by * TY - 1, bz * TZ - 1);
            }
        }
    } else {
        // shell cells of the pointer box are terminal (point to themselves)
        for (int s = tid; s < kShell; s += kThreads) {
            const int i = __ldg(A.shell + s);
            P(i) = uint16_t(i);
        }
        for (int i = tid; i < kLutWords; i += kThreads) lut[i] = __ldg(A.lut + i);
        for (int i = tid; i < PL; i += kThreads) ptab[i] = __ldg(A.ptab + i);
    }
    const int t_end = kPersist ? A.n_tiles : int(blockIdx.x) + 1;
#pragma unroll 1
    for (int t = blockIdx.x, it = 0; t < t_end; t += gridDim.x, ++it) {
    int bxo, byo, bzo;
    coords(t, bxo, byo, bzo);
    const int x0 = bxo * TX, y0 = byo * TY, z0 = A.z_lo + bzo * TZ;

    // ---- stage the tile + halo: one TMA bulk-tensor copy over the owned
    // planes (cells outside them arrive as NaN), then the halo planes that
    // belong to a neighbour slab; or plain row loads.
    if (!A.tma) {
        // one warp per box row: the row's source (owned planes, a halo plane
        // of a neighbour slab, or nothing) is decided once per row
        constexpr int kRows = BY * BZ, kU = 4;
        for (int row0 = ty; row0 < kRows; row0 += kWarps * kU) {
            float v[kU][2];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int row = row0 + u * kWarps;
                const int by = row % BY, bz = row / BY;
                const int gy = y0 + by - 1, gz = z0 + bz - 1;
                const float *src = nullptr;
                if (row < kRows && gy >= 0 && gy < D.ny && gz >= 0 && gz < D.nz) {
                    const int64_t o = int64_t(gy) * D.nx;
                    if (gz >= A.z_lo && gz < A.z_hi) src = A.f + (int64_t(gz - A.z_lo) * D.ny * D.nx + o);
                    else if (gz == A.z_lo - 1) src = A.f_lo ? A.f_lo + o : nullptr;
                    else if (gz == A.z_hi) src = A.f_hi ? A.f_hi + o : nullptr;
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int b = tx + 32 * h;
                    const int gx = x0 + b - XO;
                    v[u][h] = (src && b < BX && gx >= 0 && gx < D.nx) ? __ldg(src + gx) : __int_as_float(0x7fffffff);
                }
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int row = row0 + u * kWarps;
                if (row >= kRows) break;
                fbox[row * BX + tx] = v[u][0];
                if (tx + 32 < BX) fbox[row * BX + tx + 32] = v[u][1];
            }
        }
    }
    if (A.tma) {
        mbar_wait(bar, uint32_t(it & 1));
        if (!kInterior) {
            // halo planes held by the neighbour slabs (the tensor map covers the owned planes only)
            if (z0 == A.z_lo && A.f_lo) load_plane(fbox, 0, A.f_lo, x0, y0, D, tid);
            const int hz = A.z_hi - z0 + 1;
            if (hz <= BZ - 1 && A.f_hi) load_plane(fbox, hz, A.f_hi, x0, y0, D, tid);
        }
    }
    __syncthreads();

    const int gx = x0 + tx, gy = y0 + ty;
    const bool col_ok = kInterior || (gx < D.nx && gy < D.ny);
    const int cf = (ty + 1) * BX + tx + XO;          // this column's in-plane cell (both boxes)
    const int cfb = 2 * cf;                          // ... as a pointer-box byte offset

    // 2-D star of box plane bz at this column: c, (1,0), (0,1), (1,1), (-1,0), (0,-1), (-1,-1)
    auto star = [&](int bz, float *s) {
        const float *p = fbox + cf + bz * PL;
        s[0] = p[0];
        s[1] = p[1];
        s[2] = p[BX];
        s[3] = p[BX + 1];
        s[4] = p[-1];
        s[5] = p[-BX];
        s[6] = p[-BX - 1];
    };
    // in-plane 2x2 maxima, offsets in pointer-box bytes, as scans that start
    // at the column's own cell: B+ forward in index order (a later cell wins
    // ties), B- backward (an earlier cell must be strictly greater).  Cells
    // outside the domain hold NaN (TMA fill): a NaN never wins, and every
    // compare with it is false, so the truncated link (reading L3) falls out
    // of the same code for every tile.
    auto bplus = [&](const float *s, int dz) -> VK {    // (0,0) (1,0) (0,1) (1,1)
        VK m{s[0], dz * PSB};
        m = vmax(m, VK{s[1], 2 * 1 + dz * PSB});
        m = vmax(m, VK{s[2], 2 * BX + dz * PSB});
        m = vmax(m, VK{s[3], 2 * (BX + 1) + dz * PSB});
        return m;
    };
    auto bminus = [&](const float *s, int dz) -> VK {   // (0,0) (-1,0) (0,-1) (-1,-1), backwards
        VK m{s[0], dz * PSB};
        m = vearlier(m, VK{s[4], 2 * (-1) + dz * PSB});
        m = vearlier(m, VK{s[5], 2 * (-BX) + dz * PSB});
        m = vearlier(m, VK{s[6], 2 * (-BX - 1) + dz * PSB});
        return m;
    };

    float pm[7], p0[7], pp[7];
    // the column's own pointer-box cells are written only by this thread, so
    // their values are also kept in registers (the z loops are fully unrolled):
    // the doubling rounds and the chase start skip the own-cell loads
    uint32_t own[TZ];
    star(0, pm);
    star(1, p0);
    VK bm_prev = bminus(pm, -1);       // B-(z-1) for z = 0
    VK bp_cur = bplus(p0, 0);          // B+(z)   for z = 0
    uint32_t cls = 0;                  // 2-bit class codes of the column's 16 vertices
#pragma unroll kS1Unroll
    for (int z = 0; z < TZ; ++z) {
        star(z + 2, pp);
        const bool ok = col_ok && (kInterior || z0 + z < A.z_hi);
        const float fv = p0[0];
        // S1: argmax over box(v) u box(v - 1); the upper box wins ties
        const VK bp_next = bplus(pp, 1);
        const VK bm_cur = bminus(p0, 0);
        const VK U = vmax(bp_cur, bp_next);        // B+(z+1) is later (NaN beyond the domain)
        const VK L = vearlier(bm_cur, bm_prev);     // B-(z-1) is earlier (NaN below the domain)
        int d = vmax(L, U).d;
        bp_cur = VK{bp_next.v, bp_next.d - PSB};
        bm_prev = VK{bm_cur.v, bm_cur.d - PSB};
        // S3: upper mask, bit k = k-th link vertex in ascending index order:
        // lower group (index < v: up iff f > fv), then the upper group (>=).
        uint32_t mask = 0u;
        or_if_ge<1u << 13>(mask, pp[3], fv);
        or_if_ge<1u << 12>(mask, pp[2], fv);
        or_if_ge<1u << 11>(mask, pp[1], fv);
        or_if_ge<1u << 10>(mask, pp[0], fv);
        or_if_ge<1u << 9>(mask, p0[3], fv);
        or_if_ge<1u << 8>(mask, p0[2], fv);
        or_if_ge<1u << 7>(mask, p0[1], fv);
        or_if_gt<1u << 6>(mask, p0[4], fv);
        or_if_gt<1u << 5>(mask, p0[5], fv);
        or_if_gt<1u << 4>(mask, p0[6], fv);
        or_if_gt<1u << 3>(mask, pm[0], fv);
        or_if_gt<1u << 2>(mask, pm[4], fv);
        or_if_gt<1u << 1>(mask, pm[5], fv);
        or_if_gt<1u << 0>(mask, pm[6], fv);
        // an empty upper link points to itself; this also makes a NaN vertex
        // (every compare false) terminal, so no pointer cycle can form
        d = mask ? d : 0;
        const int c = cfb + (z + 1) * PSB;
        own[z] = uint32_t(kInterior || ok ? c + d : c);
        P(c) = uint16_t(own[z]);
        // 2-bit class code from the LUT: bit 0 saddle (beta0+ >= 2), bit 1
        // maximum (empty mask); interleaved, vertex z at bits 2z, 2z + 1
        const uint32_t code = (lut[mask >> 4] >> ((mask & 15) << 1)) & 3u;
        cls |= ((kInterior || ok) ? code : 0u) << (2 * z);
#pragma unroll
        for (int k = 0; k < 7; ++k) {
            pm[k] = p0[k];
            p0[k] = pp[k];
        }
    }
    // deinterleave: even bits -> saddles, odd bits -> maxima
    auto compact = [](uint32_t x) {        // bits 0, 2, 4, ... -> 0, 1, 2, ...
        x &= 0x55555555u;
        x = (x | (x >> 1)) & 0x33333333u;
        x = (x | (x >> 2)) & 0x0f0f0f0fu;
        x = (x | (x >> 4)) & 0x00ff00ffu;
        return (x | (x >> 8)) & 0x0000ffffu;
    };
    const uint32_t sad_mask = compact(cls), max_mask = compact(cls >> 1);
    // NaN (reading L2): a NaN vertex compares false with everything, so its
    // upper mask is empty -- only the (rare) maxima need the test
    for (uint32_t m = max_mask; m; m &= m - 1) {
        const float v = fbox[cf + (__ffs(m)) * PL];   // box plane z + 1
        if (v != v) atomicOr(A.nan_flag, 1);
    }
    __syncthreads();
    if (kPersist && tid == 0 && t + int(gridDim.x) < t_end) {
        // the field box is dead (no exit marks on the one-slab path): the
        // next tile's copy overlaps the rest of this one
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue_tma(t + int(gridDim.x), false);
    }

    // ---- S2 inside the tile.  The field box is dead: it now holds one
    // exit-mark byte per pointer-box cell.  Two rounds of pointer doubling
    // (independent loads, no divergence) quarter every chain; then every
    // vertex follows the rest of its chain to the local root and stores the
    // root in its own cell only.  Any other thread reads that cell as either
    // the old pointer or the root -- both lie on the same ascending path --
    // so nothing needs settling, and chains that run into a finished cell end
    // one hop later.
    uint8_t *used = reinterpret_cast<uint8_t *>(fbox);
    if (!no_elist)   // exit marks are only read back when the tile appends to E
        for (int i = tid; i < 2 * PBOX / 16; i += kThreads) reinterpret_cast<uint4 *>(used)[i] = make_uint4(0, 0, 0, 0);
#pragma unroll 1
    for (int round = 0; round < A.rounds; ++round) {
#pragma unroll
        for (int z = 0; z < TZ; ++z) {
            const int c = cfb + (z + 1) * PSB;
            own[z] = ld16(pbase + own[z]);   // benign-race: a reader sees the old or the new pointer, both on the path
            P(c) = uint16_t(own[z]);
        }
        __syncthreads();
    }
    if (A.rounds == 0) __syncthreads();

    // ---- outputs: label (bit 31 = exit) and the exit mark of its root
    const int32_t nxy = D.ny * D.nx;
    // 32-bit index arithmetic (N < 2^31): the global id of box cell (0,0,0),
    // and this column's owned index at z = 0
    const int32_t g_box0 = ((z0 - 1) * D.ny + (y0 - 1)) * D.nx + (x0 - XO);
    const int32_t i_col = (z0 * D.ny + gy) * D.nx + gx - int32_t(A.v0);
    int n_exit = 0;
#pragma unroll kOutUnroll
    for (int zz = 0; zz < TZ; ++zz) {
        const int z = TZ - 1 - zz;   // top down: measured 1.5 % faster than bottom up on C3
        const bool ok = col_ok && (kInterior || z0 + z < A.z_hi);
        const int c = cfb + (z + 1) * PSB;
        // chase to the root (a cell that points to itself), two hops per
        // loop turn so that no register copies are needed
        uint32_t r = own[z];
        for (;;) {
            const uint32_t q = ld16(pbase + r);   // benign-race
            if (q == r) break;
            r = ld16(pbase + q);   // benign-race
            if (r == q) break;
        }
        P(c) = uint16_t(r);   // benign-race: the root is a later vertex of every path through c
        const int bz = r >> 11;
        const int32_t t = *reinterpret_cast<const int32_t *>(reinterpret_cast<const char *>(ptab) + (((r & (2 * PS - 1)) - bz * SKEW) << 1));
        // exit: the root is in the halo shell of the box, or (last tile of a
        // slab) in a plane the slab does not own
        bool exit = t < 0 || unsigned(bz - 1) >= unsigned(TZ);
        if (!kInterior) exit = exit || z0 - 1 + bz >= A.z_hi;
        const int32_t root = g_box0 + bz * nxy + (t & 0x7fffffff);
        if (kInterior || ok) {
            A.label[i_col + z * nxy] = exit ? int32_t(uint32_t(root) | kFlag) : root;
            if (exit && !no_elist) used[r] = 1;
            if (kStats) n_exit += exit;
        }
    }
    if (kStats) {
        const unsigned sum = __reduce_add_sync(0xffffffffu, unsigned(n_exit));
        if (tx == 0 && sum) atomicAdd(A.exit_count, (unsigned long long)sum);
    }

    // ---- maxima and saddles of this column, appended (unordered) to the
    // slab's lists: warp prefix sums, one atomic per list per warp that has any
    {
        const uint32_t mine = uint32_t(__popc(max_mask)) | (uint32_t(__popc(sad_mask)) << 16);
        if (__any_sync(0xffffffffu, mine != 0u)) {
            uint32_t incl = mine;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (tx >= o) incl += y;
            }
            const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
            unsigned long long bm = 0, bs = 0;
            if (tx == 0) {
                if (tot & 0xffffu) bm = atomicAdd(A.ecount + 1, (unsigned long long)(tot & 0xffffu));
                if (tot >> 16) bs = atomicAdd(A.ecount + 2, (unsigned long long)(tot >> 16));
            }
            const uint32_t excl = incl - mine;
            unsigned long long jm = __shfl_sync(0xffffffffu, bm, 0) + (excl & 0xffffu);
            unsigned long long js = __shfl_sync(0xffffffffu, bs, 0) + (excl >> 16);
            const int32_t g0 = i_col + int32_t(A.v0);     // global id of this column's z = 0 vertex
            for (uint32_t m = max_mask; m; m &= m - 1, ++jm)
                if (jm < (unsigned long long)A.list_cap) A.max_list[jm] = g0 + (__ffs(m) - 1) * nxy;
            for (uint32_t m = sad_mask; m; m &= m - 1, ++js)
                if (js < (unsigned long long)A.list_cap) A.sad_list[js] = g0 + (__ffs(m) - 1) * nxy;
        }
    }
    if (no_elist) {
        if (kPersist) __syncthreads();   // the next tile's S1 rewrites the pointer box
        continue;
    }
    __syncthreads();

    // ---- append the tile's exit targets (marked shell cells) to E: per-warp
    // ballot counts, one global atomic per tile, then the ids in warp order
    int cnt = 0;
    for (int s0 = ty * 32; s0 < kShell; s0 += kThreads) {
        const int s = s0 + tx;
        const bool m = s < kShell && used[__ldg(A.shell + s)];
        cnt += __popc(__ballot_sync(0xffffffffu, m));
    }
    if (tx == 0) red[ty] = uint32_t(cnt);
    __syncthreads();
    if (ty == 0) {
        const uint32_t mine = tx < kWarps ? red[tx] : 0u;
        uint32_t incl = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (tx >= o) incl += y;
        }
        if (tx < kWarps) red[tx] = incl - mine;
        if (tx == 31) *ebase = incl ? atomicAdd(A.ecount, (unsigned long long)incl) : 0ull;
    }
    __syncthreads();
    unsigned long long slot = *ebase + red[ty];
    const uint32_t lt = (1u << tx) - 1u;
    for (int s0 = ty * 32; s0 < kShell; s0 += kThreads) {
        const int s = s0 + tx;
        const int i = s < kShell ? __ldg(A.shell + s) : 0;
        const bool m = s < kShell && used[i];
        const uint32_t b = __ballot_sync(0xffffffffu, m);
        if (m) {
            const unsigned long long j = slot + __popc(b & lt);
            if (j < (unsigned long long)A.ecap) A.elist[j] = g_box0 + (i >> 11) * nxy + (ptab[((i & (2 * PS - 1)) - (i >> 11) * SKEW) >> 1] & 0x7fffffff);
        }
        slot += __popc(b);
    }
    }   // tiles
}

// Pass E: resolve every owned exit target through the exit graph (bit 31 =
// not final), one dependent load per tile hop (L1-cached: a stale value is an
// earlier vertex of the same path, so it only lengthens the walk).  A path that leaves the slab
// stops at its first remote vertex (resolved later by the boundary exchange).
__global__ void __launch_bounds__(256) k_resolve_exits(int32_t *label, const int32_t *__restrict__ elist,
                                                       const unsigned long long *ecount, int64_t ecap, int64_t v0,
                                                       int64_t v1) {
    const int64_t n = int64_t(min(*ecount, (unsigned long long)ecap));
    for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += int64_t(gridDim.x) * blockDim.x) {
        const int64_t e = elist[j];
        if (e < v0 || e >= v1) continue;                 // a halo vertex: another slab's
        int32_t w = __ldca(label + (e - v0));
        if (w >= 0) continue;
        for (;;) {
            const int64_t x = w & 0x7fffffff;
            if (x < v0 || x >= v1) break;                 // remote: stays unresolved
            const int32_t nw = __ldca(label + (x - v0));
            w = nw;
            if (w >= 0) break;
        }
        label[e - v0] = w;
    }
}

// Pass E' (fallback when E overflowed): every exiting vertex chases its own
// path as far as the slab allows.
__global__ void __launch_bounds__(256) k_exit_chase(int32_t *label, int64_t v0, int64_t v1) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= v1 - v0) return;
    int32_t w = label[i];
    if (w >= 0) return;
    while (w < 0) {
        const int64_t x = w & 0x7fffffff;
        if (x < v0 || x >= v1) break;
        w = __ldca(label + (x - v0));
    }
    label[i] = w;
}

__global__ void k_widen(const int32_t *__restrict__ in, int64_t *out, int64_t n) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) out[i] = in[i];
}

// --------------------------------------------------------------- host side

static eg_status fail(std::string *err, cudaError_t e, const char *what) {
    if (err) *err = std::string(what) + ": " + cudaGetErrorString(e);
    return e == cudaErrorMemoryAllocation ? EG_ERR_OOM : EG_ERR_CUDA;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static cudaError_t grow_lists(Tiled3D *t, int64_t cap) {
    if (t->d_max) cudaFree(t->d_max);
    if (t->d_sad) cudaFree(t->d_sad);
    t->d_max = t->d_sad = nullptr;
    t->list_cap = 0;
    cudaError_t e = cudaMalloc(&t->d_max, size_t(cap) * 4);
    if (e == cudaSuccess) e = cudaMalloc(&t->d_sad, size_t(cap) * 4);
    if (e == cudaSuccess) t->list_cap = cap;
    return e;
}

template <class T>
static cudaError_t upload(T **d, const std::vector<T> &h) {
    cudaError_t e = cudaMalloc(d, h.size() * sizeof(T));
    if (e != cudaSuccess) return e;
    return cudaMemcpy(*d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice);
}

// eg_compute_host pipeline (see ChunkIO): H2D chunk k on io->h2d; tile chunk k
// on st after H2D chunk k + 1 (its top halo plane); label chunk k - 1 on
// io->fst after tile chunk k, following chains only through labelled vertices
// (those ending beyond go to the fix-up list); its labels to the host on
// io->d2h.  After the last chunk the fix-up list is finished on the device;
// the caller patches those labels on the host.
static eg_status pipeline_chunks(Tiled3D *t, const TileArgs &A, const CUtensorMap &tmap, const Dims3 &D, int3 hi,
                                 int3 lo, int32_t *labels, const Slab &s, int64_t nown, int64_t nxy, cudaStream_t st,
                                 ChunkIO *io, eg_stats *stats, std::string *err) {
    cudaError_t e;
    const int layers = hi.z - lo.z + 1;
    const int K = std::max(1, std::min({io->K, kMaxChunks, layers}));
    const int64_t cap = std::max<int64_t>(nown / 16, 4096);
    if (t->fin_cap < cap) {
        if (t->d_fin_list) cudaFree(t->d_fin_list);
        t->d_fin_list = nullptr;
        t->fin_cap = 0;
        if ((e = cudaMalloc(&t->d_fin_list, cap * 4)) != cudaSuccess) return fail(err, e, "cudaMalloc fix-up list");
        t->fin_cap = cap;
    }
    auto first_layer = [&](int k) { return lo.z + int(int64_t(layers) * k / K); };
    auto vend = [&](int k) -> int64_t {       // local index where chunk k ends
        return k < 0 ? 0 : std::min<int64_t>(int64_t(first_layer(k + 1) - lo.z) * TZ * nxy, nown);
    };
    cudaEvent_t *evH = t->ev_io, *evT = t->ev_io + kMaxChunks, *evL = t->ev_io + 2 * kMaxChunks;
    cudaEvent_t *evS = t->ev_io + 3 * kMaxChunks;
    if ((e = cudaEventRecord(evS[0], st)) != cudaSuccess || (e = cudaStreamWaitEvent(io->h2d, evS[0], 0)) != cudaSuccess)
        return fail(err, e, "pipeline start");
    // H2D chunk k also carries the first plane of chunk k + 1 (tile chunk k's
    // top halo), so tile chunk k waits for H2D chunk k only
    const int64_t plane = nxy;
    for (int k = 0; k < K; ++k) {
        const int64_t a = k == 0 ? 0 : vend(k - 1) + plane, b = std::min(vend(k) + plane, nown);
        if ((e = cudaMemcpyAsync(io->d_field + a, io->h_field + a, sizeof(float) * size_t(b - a),
                                 cudaMemcpyHostToDevice, io->h2d)) != cudaSuccess ||
            (e = cudaEventRecord(evH[k], io->h2d)) != cudaSuccess)
            return fail(err, e, "H2D chunk");
    }
    auto label_chunk = [&](int k, int64_t lim) -> eg_status {
        if ((e = launch_finalize_chunk(labels, vend(k - 1) / 32, (vend(k) + 31) / 32, nown, s.v0, lim,
                                       t->d_fin_list, t->d_ecount + 3, t->fin_cap, io->fst)) != cudaSuccess)
            return fail(err, e, "k_finalize_chunk");
        stats->kernel_launches += 1;
        return EG_OK;
    };
    auto labels_out = [&](int k) -> eg_status {
        if (!io->h_labels) return EG_OK;
        const int64_t a = vend(k - 1), b = vend(k);
        if ((e = cudaStreamWaitEvent(io->d2h, evL[k], 0)) != cudaSuccess ||
            (e = cudaMemcpyAsync(io->h_labels + a, labels + a, sizeof(int32_t) * size_t(b - a),
                                 cudaMemcpyDeviceToHost, io->d2h)) != cudaSuccess)
            return fail(err, e, "D2H labels chunk");
        return EG_OK;
    };
    for (int k = 0; k < K; ++k) {
        TileArgs Ak = A;
        const int l0 = first_layer(k), l1 = first_layer(k + 1);
        Ak.origin.z = l0;
        Ak.n_tiles = int32_t(int64_t(A.tiles_x) * A.tiles_y * (l1 - l0));
        if ((e = cudaStreamWaitEvent(st, evH[k], 0)) != cudaSuccess) return fail(err, e, "H2D wait");
        k_tile<true, false, false, true><<<unsigned(Ak.n_tiles), kThreads, kTileSmem, st>>>(tmap, Ak, D);
        stats->kernel_launches += 1;
        if ((e = cudaGetLastError()) != cudaSuccess) return fail(err, e, "k_tile<interior> chunk");
        if ((e = cudaEventRecord(evT[k], st)) != cudaSuccess) return fail(err, e, "tile chunk event");
        if (k >= 1) {
            // chunk k - 1: its chains may run through every chunk <= k
            if ((e = cudaStreamWaitEvent(io->fst, evT[k], 0)) != cudaSuccess) return fail(err, e, "tile wait");
            const eg_status ls = label_chunk(k - 1, k == K - 1 ? nown : vend(k));
            if (ls != EG_OK) return ls;
            if ((e = cudaEventRecord(evL[k - 1], io->fst)) != cudaSuccess) return fail(err, e, "label event");
            const eg_status os = labels_out(k - 1);
            if (os != EG_OK) return os;
        }
    }
    if (K == 1 && (e = cudaStreamWaitEvent(io->fst, evT[0], 0)) != cudaSuccess) return fail(err, e, "tile wait");
    const eg_status ls = label_chunk(K - 1, nown);
    if (ls != EG_OK) return ls;
    if ((e = launch_finalize_list(labels, t->d_fin_list, t->d_ecount + 3, t->fin_cap, s.v0, nown, io->fst)) !=
            cudaSuccess ||
        (e = cudaEventRecord(evL[K - 1], io->fst)) != cudaSuccess)
        return fail(err, e, "k_finalize_list");
    stats->kernel_launches += 1;
    const eg_status os = labels_out(K - 1);
    if (os != EG_OK) return os;
    if ((e = cudaEventRecord(evS[1], io->d2h)) != cudaSuccess) return fail(err, e, "D2H event");
    io->fin_done = evL[K - 1];
    io->d2h_done = evS[1];
    io->done = true;
    return EG_OK;
}

eg_status tiled3d_local(Tiled3D *t, int ndim, const int64_t *dims, const Slab &s, const FieldView &F, int32_t *labels,
                        int *flags, cudaStream_t st, eg_stats *stats, std::string *err, cudaEvent_t ev_main0,
                        cudaEvent_t ev_main1, unsigned long long *exit_count, cudaEvent_t halo_ready,
                        ChunkIO *io) {
    if (io) io->done = false;
    int64_t d3[3] = {1, 1, 1};
    for (int i = 0; i < ndim; ++i) d3[i] = dims[i];
    cudaError_t e;
    if (!t->ready) {
        // 2-bit LUT: beta0+ >= 2 (bit 0) and empty mask (bit 1) for every 14-bit upper mask of the 3-D link,
        // in the ascending-index offset order (lexicographic in (dz, dy, dx))
        int64_t dl[3] = {4, 4, 4};
        LinkTable tab = make_link_table(3, dl);
        std::vector<uint8_t> beta = make_beta_lut3(tab);
        std::vector<uint32_t> bits(kLutWords, 0u);
        for (int m = 0; m < (1 << 14); ++m) {
            const uint32_t code = (beta[m] >= 2 ? 1u : 0u) | (m == 0 ? 2u : 0u);
            bits[m >> 4] |= code << ((m & 15) * 2);
        }
        if ((e = upload(&t->d_lut, bits)) != cudaSuccess) return fail(err, e, "lut upload");
        // pointer-box indices of the halo shell
        std::vector<uint16_t> sh;
        for (int bz = 0; bz < BZ; ++bz)
            for (int by = 0; by < BY; ++by)
                for (int bx = XO - 1; bx <= XO + TX; ++bx)
                    if (bz == 0 || bz == BZ - 1 || by == 0 || by == BY - 1 || bx == XO - 1 || bx == XO + TX)
                        sh.push_back(uint16_t(2 * (bz * PS + by * BX + bx) + bz * SKEW));
        if (int(sh.size()) != kShell) {
            if (err) *err = "shell size";
            return EG_ERR_STATE;
        }
        if ((e = upload(&t->d_shell, sh)) != cudaSuccess) return fail(err, e, "shell upload");
        {
            // smem image [kOffP, kOffM): pointer box with self-pointing shell cells, then the LUT
            std::vector<unsigned char> img(kOffM - kOffP, 0);
            for (uint16_t b : sh) std::memcpy(img.data() + b, &b, 2);
            std::memcpy(img.data() + (kOffL - kOffP), bits.data(), size_t(kLutWords) * 4);
            if ((e = upload(&t->d_tmpl, img)) != cudaSuccess) return fail(err, e, "template upload");
        }
        if ((e = cudaMalloc(&t->d_ecount, 4 * sizeof(unsigned long long))) != cudaSuccess)
            return fail(err, e, "cudaMalloc ecount");
        for (auto &ev : t->ev_io)
            if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess)
                return fail(err, e, "pipeline events");
        if ((e = cudaFuncSetAttribute(k_tile<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(kTileSmem))) != cudaSuccess ||
            (e = cudaFuncSetAttribute(k_tile<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(kTileSmem))) != cudaSuccess ||
            (e = cudaFuncSetAttribute(k_tile<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(kTileSmem))) != cudaSuccess ||
            (e = cudaFuncSetAttribute(k_tile<true, false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(kTileSmem))) != cudaSuccess ||
            (e = cudaFuncSetAttribute(k_tile<true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(kTileSmem))) != cudaSuccess ||
            (e = cudaFuncSetAttribute(k_tile<false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(kTileSmem))) != cudaSuccess)
            return fail(err, e, "smem attr");
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&t->n_sm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || t->n_sm < 1)
            t->n_sm = 148;
        const char *rs = std::getenv("EG_TILE_ROUNDS");   // tuning knob (default 2)
        if (rs && rs[0] >= '0' && rs[0] <= '6') t->rounds = rs[0] - '0';
        cudaDriverEntryPointQueryResult q;
        void *fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            t->encode = fn;
        cudaGetLastError();
        t->ready = true;
    }
    // a 1-D / 2-D grid is a 3-D grid with unit axes; its only slab is the whole grid
    const int64_t z_lo = ndim == 3 ? s.z0 : 0, z_hi = ndim == 3 ? s.z1 : 1;
    const int64_t nown = s.v1 - s.v0;
    Dims3 D{int32_t(d3[0]), int32_t(d3[1]), int32_t(d3[2])};
    const int tiles_x = int((d3[0] + TX - 1) / TX), tiles_y = int((d3[1] + TY - 1) / TY);
    const int tiles_z = int((z_hi - z_lo + TZ - 1) / TZ);
    if (tiles_x > 1024 || tiles_y > 1024 || tiles_z > 2047) {
        if (err) *err = "grid too large for the tiled path";
        return EG_ERR_UNSUPPORTED;
    }
    // "interior" tiles: every own cell inside the domain and the owned planes
    // (full tiles; the halo may be outside the domain -- NaN by TMA), and no
    // halo plane held by a neighbour slab (those tiles patch it in)
    const int nfx = int(d3[0] / TX), nfy = int(d3[1] / TY), nfz = int((z_hi - z_lo) / TZ);
    int3 lo = make_int3(0, 0, F.lo ? 1 : 0);
    int3 hi = make_int3(nfx - 1, nfy - 1, nfz - 1 - ((F.hi && int64_t(nfz) * TZ == z_hi - z_lo) ? 1 : 0));
    const bool have_interior = hi.x >= lo.x && hi.y >= lo.y && hi.z >= lo.z;
    // boundary tile list, cached per (dims, slab)
    if (t->bdims[0] != d3[0] || t->bdims[1] != d3[1] || t->bdims[2] != d3[2] || t->bz[0] != z_lo || t->bz[1] != z_hi) {
        std::vector<int32_t> bt;
        for (int bz = 0; bz < tiles_z; ++bz)
            for (int by = 0; by < tiles_y; ++by)
                for (int bx = 0; bx < tiles_x; ++bx) {
                    const bool in = have_interior && bx >= lo.x && bx <= hi.x && by >= lo.y && by <= hi.y &&
                                    bz >= lo.z && bz <= hi.z;
                    if (!in) bt.push_back((bz << 20) | (by << 10) | bx);
                }
        if (t->d_btiles) cudaFree(t->d_btiles);
        t->d_btiles = nullptr;
        if (!bt.empty() && (e = upload(&t->d_btiles, bt)) != cudaSuccess) return fail(err, e, "btiles upload");
        t->n_btiles = int64_t(bt.size());
        for (int i = 0; i < 3; ++i) t->bdims[i] = d3[i];
        t->bz[0] = z_lo;
        t->bz[1] = z_hi;
    }
    // plane table: box-plane cell (bx, by) -> by * nx + bx, bit 31 if the cell
    // is on the in-plane shell (x or y halo)
    if (t->ptab_nx != d3[0]) {
        std::vector<int32_t> pt(PL);
        for (int rr = 0; rr < PL; ++rr) {
            const int by = rr / BX, bx = rr % BX;
            const bool sh = bx < XO || bx >= XO + TX || by == 0 || by == BY - 1;
            pt[rr] = int32_t(uint32_t(by * int32_t(d3[0]) + bx) | (sh ? kFlag : 0u));
        }
        if (!t->d_ptab && (e = cudaMalloc(&t->d_ptab, PL * 4)) != cudaSuccess) return fail(err, e, "cudaMalloc ptab");
        if ((e = cudaMemcpy(t->d_ptab, pt.data(), PL * 4, cudaMemcpyHostToDevice)) != cudaSuccess)
            return fail(err, e, "ptab upload");
        t->ptab_nx = d3[0];
    }
    // exit-target list capacity: N / 8 (falls back to a per-vertex chase on overflow)
    // (EG_LIST_DIV / EG_ELIST_DIV: test knobs that start the lists small, to
    // exercise the grow-and-rerun path)
    auto env_div = [](const char *name, int64_t dflt) {
        const char *v = std::getenv(name);
        const int64_t d = v ? std::atoll(v) : 0;
        return d > 0 ? d : dflt;
    };
    const int64_t floor_cap = std::getenv("EG_LIST_DIV") ? 16 : (1 << 16);
    const int64_t want = std::max<int64_t>(nown / env_div("EG_ELIST_DIV", 8), std::getenv("EG_ELIST_DIV") ? 16 : 4096);
    if (t->ecap < want) {
        if (t->d_elist) cudaFree(t->d_elist);
        t->d_elist = nullptr;
        t->ecap = 0;
        if ((e = cudaMalloc(&t->d_elist, want * 4)) != cudaSuccess) return fail(err, e, "cudaMalloc elist");
        t->ecap = want;
    }
    // maxima / saddle list capacity: N / 4 to start with (a noisy field has
    // ~15 % saddles); on overflow the lists grow and the pass runs again
    if (t->list_cap < std::max<int64_t>(nown / env_div("EG_LIST_DIV", 4), floor_cap)) {
        const int64_t cap = std::max<int64_t>(nown / env_div("EG_LIST_DIV", 4), floor_cap);
        if ((e = grow_lists(t, cap)) != cudaSuccess) return fail(err, e, "cudaMalloc lists");
    }
    // TMA tensor map over the owned planes (needs 16-byte row and plane
    // strides); cells outside it are filled with NaN
    CUtensorMap tmap;
    std::memset(&tmap, 0, sizeof(tmap));
    bool tma = t->encode != nullptr && (d3[0] % 4) == 0 && (reinterpret_cast<uintptr_t>(F.own) % 16) == 0;
    if (tma) {
        cuuint64_t gdim[3] = {cuuint64_t(d3[0]), cuuint64_t(d3[1]), cuuint64_t(z_hi - z_lo)};
        cuuint64_t gstr[2] = {cuuint64_t(d3[0] * 4), cuuint64_t(d3[0] * d3[1] * 4)};
        cuuint32_t box[3] = {BX, BY, BZ};
        cuuint32_t es[3] = {1, 1, 1};
        CUresult r = reinterpret_cast<EncodeTiledFn>(t->encode)(
            &tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float *>(F.own), gdim, gstr, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NAN_REQUEST_ZERO_FMA);
        tma = (r == CUDA_SUCCESS);
    }
    stats->path = 1;
    for (int attempt = 0;; ++attempt) {
        if ((e = cudaMemsetAsync(t->d_ecount, 0, 4 * sizeof(unsigned long long), st)) != cudaSuccess)
            return fail(err, e, "memset counts");
        TileArgs A{};
        A.f = F.own;
        A.f_lo = F.lo;
        A.f_hi = F.hi;
        A.z_lo = int32_t(z_lo);
        A.z_hi = int32_t(z_hi);
        A.v0 = s.v0;
        A.label = labels;
        A.max_list = t->d_max;
        A.sad_list = t->d_sad;
        A.list_cap = t->list_cap;
        A.nan_flag = flags;
        A.elist = t->d_elist;
        A.ecount = t->d_ecount;
        A.ecap = t->ecap;
        A.lut = t->d_lut;
        A.tmpl = t->d_tmpl;
        A.ptab = t->d_ptab;
        A.shell = t->d_shell;
        A.btiles = t->d_btiles;
        A.rounds = t->rounds;
        A.exit_count = exit_count;
        stats->tile_rounds = t->rounds;
        // No exit list: the label pass chases (one slab: C3 0.6 ms faster;
        // with L1-cached chase loads also for L2-resident label arrays: C2
        // 2.95 vs 2.97 ms, F1-256 0.30 vs 0.34 ms; several slabs: the chase
        // stops at the first remote vertex: C3 at 2 / 4 virtual slabs 11.8 / 12.5 -> 9.9 / 10.2 ms).
        // EG_ELIST=1 builds and resolves the exit list instead.
        const char *el = std::getenv("EG_ELIST");
        A.no_elist = (el && el[0] == '1') ? 0 : 1;
        A.tma = tma ? 1 : 0;
        {
            // L2 prefetch of the box of the tile one resident-CTA count ahead (2 per SM):
            // the CTA that takes the slot next starts on an L2 hit.  C3 k_tile 5432 -> 5361 us
            // (80..296 tiles ahead all within 3 us; 592: 5399 us)
            const char *pv = std::getenv("EG_TMA_PREFETCH");   // tuning knob: distance in tiles, 0 = off
            A.prefetch = pv ? std::atoi(pv) : 2 * t->n_sm;
        }
        if (ev_main0) cudaEventRecord(ev_main0, st);
        // eg_compute_host pipeline: every tile interior, no exit list, TMA
        const char *pe = std::getenv("EG_PERSIST");
        const bool persist_req = pe && pe[0] == '1';
        const bool chunk = io && io->h_field && A.no_elist && A.tma && !persist_req && t->n_btiles == 0 &&
                           have_interior && attempt == 0;
        if (io && io->h_field && !chunk && attempt == 0) {
            // not chunkable: the whole field first
            if ((e = cudaMemcpyAsync(io->d_field, io->h_field, sizeof(float) * size_t(nown), cudaMemcpyHostToDevice,
                                     st)) != cudaSuccess)
                return fail(err, e, "H2D field");
        }
        // halo_ready (several GPUs): the neighbour slabs' halo planes arrive on
        // another stream while the interior tiles (which never read them) run;
        // the boundary tiles are launched after them
        auto boundary_tiles = [&]() -> eg_status {
            if (t->n_btiles <= 0) return EG_OK;
            if (halo_ready && (e = cudaStreamWaitEvent(st, halo_ready, 0)) != cudaSuccess)
                return fail(err, e, "halo wait");
            if (A.exit_count)
                k_tile<false, false, true><<<unsigned(t->n_btiles), kThreads, kTileSmem, st>>>(tmap, A, D);
            else
                k_tile<false, false><<<unsigned(t->n_btiles), kThreads, kTileSmem, st>>>(tmap, A, D);
            stats->kernel_launches += 1;
            if ((e = cudaGetLastError()) != cudaSuccess) return fail(err, e, "k_tile<boundary>");
            return EG_OK;
        };
        if (!halo_ready) {
            const eg_status bs = boundary_tiles();
            if (bs != EG_OK) return bs;
        }
        if (have_interior) {
            A.tiles_x = hi.x - lo.x + 1;
            A.tiles_y = hi.y - lo.y + 1;
            A.origin = lo;
            const int64_t nt = int64_t(A.tiles_x) * A.tiles_y * (hi.z - lo.z + 1);
            A.mx = ((uint64_t(1) << 32) + uint64_t(A.tiles_x) - 1) / uint64_t(A.tiles_x);
            A.my = ((uint64_t(1) << 32) + uint64_t(A.tiles_y) - 1) / uint64_t(A.tiles_y);
            A.n_tiles = int32_t(nt);
            // persistent CTAs (2 per SM) on the one-slab TMA path: measured slower
            // on C3 (6.27 vs 5.65 ms), so only on request (EG_PERSIST=1)
            const bool persist = A.no_elist && A.tma && persist_req && nt > 2 * t->n_sm;
            if (chunk) {
                const eg_status cs = pipeline_chunks(t, A, tmap, D, hi, lo, labels, s, nown, int64_t(d3[0]) * d3[1],
                                                     st, io, stats, err);
                if (cs != EG_OK) return cs;
            } else if (persist)
                k_tile<true, true><<<unsigned(2 * t->n_sm), kThreads, kTileSmem, st>>>(tmap, A, D);
            else if (A.exit_count)
                k_tile<true, false, true><<<unsigned(nt), kThreads, kTileSmem, st>>>(tmap, A, D);
            else
                if (A.no_elist)
                    k_tile<true, false, false, true><<<unsigned(nt), kThreads, kTileSmem, st>>>(tmap, A, D);
                else
                    k_tile<true, false><<<unsigned(nt), kThreads, kTileSmem, st>>>(tmap, A, D);
            stats->kernel_launches += 1;
            if ((e = cudaGetLastError()) != cudaSuccess) return fail(err, e, "k_tile<interior>");
        }
        if (halo_ready) {
            const eg_status bs = boundary_tiles();
            if (bs != EG_OK) return bs;
        }
        if (ev_main1) cudaEventRecord(ev_main1, st);
        // resolve the owned part of E
        if (!A.no_elist) {
            k_resolve_exits<<<148 * 64, 256, 0, st>>>(labels, t->d_elist, t->d_ecount, t->ecap, s.v0, s.v1);
            stats->kernel_launches += 1;
            if ((e = cudaGetLastError()) != cudaSuccess) return fail(err, e, "k_resolve_exits");
        }
        unsigned long long cnt[3] = {0, 0, 0};
        if ((e = cudaMemcpyAsync(cnt, t->d_ecount, sizeof(cnt), cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
            (e = cudaStreamSynchronize(st)) != cudaSuccess)
            return fail(err, e, "counts");
        if ((int64_t(cnt[1]) > t->list_cap || int64_t(cnt[2]) > t->list_cap) && attempt == 0) {
            // more critical points than the lists hold: grow them, run again
            const int64_t cap = std::max<int64_t>(int64_t(std::max(cnt[1], cnt[2])) * 5 / 4, t->list_cap);
            if ((e = grow_lists(t, cap)) != cudaSuccess) return fail(err, e, "cudaMalloc lists");
            if (io && io->done) {
                // the pipeline's label chunks ran on this pass's labels: let them
                // finish; the rerun is unchunked (the field is on the device now)
                if ((e = cudaStreamSynchronize(io->fst)) != cudaSuccess ||
                    (e = cudaStreamSynchronize(io->d2h)) != cudaSuccess)
                    return fail(err, e, "pipeline streams");
                io->done = false;
            }
            continue;
        }
        stats->n_exit_targets += int64_t(cnt[0]);
        t->n_max = int64_t(cnt[1]);
        t->n_sad = int64_t(cnt[2]);
        t->v0 = s.v0;
        t->v1 = s.v1;
        if (int64_t(cnt[0]) > t->ecap) {
            // E overflowed: every exiting vertex chases its own path (exact, slower)
            k_exit_chase<<<unsigned((nown + 255) / 256), 256, 0, st>>>(labels, s.v0, s.v1);
            stats->kernel_launches += 1;
            if ((e = cudaGetLastError()) != cudaSuccess) return fail(err, e, "k_exit_chase");
        }
        break;
    }
    return EG_OK;
}

int64_t tiled3d_count(const Tiled3D *t, int which) { return which == 0 ? t->n_max : t->n_sad; }

// The maxima and saddles of the last tiled3d_local, ascending (cub radix sort
// of the unordered lists over the bits of the slab's largest id).
eg_status tiled3d_lists(Tiled3D *t, int64_t *max64, int32_t *sad32, int64_t *sad64, cudaStream_t st,
                        eg_stats *stats, std::string *err) {
    cudaError_t e;
    int bits = 1;
    while (bits < 31 && (int64_t(1) << bits) < t->v1) ++bits;
    const int64_t nm = t->n_max, ns = t->n_sad;
    if (t->alt_cap < std::max<int64_t>(nm, 1)) {
        if (t->d_alt) cudaFree(t->d_alt);
        t->d_alt = nullptr;
        t->alt_cap = 0;
        if ((e = cudaMalloc(&t->d_alt, size_t(std::max<int64_t>(nm, 1)) * 4)) != cudaSuccess)
            return fail(err, e, "cudaMalloc sorted maxima");
        t->alt_cap = std::max<int64_t>(nm, 1);
    }
    size_t need = 0, b2 = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, need, t->d_max, t->d_alt, int(std::max<int64_t>(nm, 1)), 0, bits, st);
    cub::DeviceRadixSort::SortKeys(nullptr, b2, t->d_sad, sad32, int(std::max<int64_t>(ns, 1)), 0, bits, st);
    need = std::max(need, b2);
    if (t->sort_tmp_bytes < need) {
        if (t->d_sort_tmp) cudaFree(t->d_sort_tmp);
        t->d_sort_tmp = nullptr;
        t->sort_tmp_bytes = 0;
        if ((e = cudaMalloc(&t->d_sort_tmp, need)) != cudaSuccess) return fail(err, e, "cudaMalloc sort scratch");
        t->sort_tmp_bytes = need;
    }
    if (nm > 0) {
        size_t b = t->sort_tmp_bytes;
        if ((e = cub::DeviceRadixSort::SortKeys(t->d_sort_tmp, b, t->d_max, t->d_alt, int(nm), 0, bits, st)) !=
            cudaSuccess)
            return fail(err, e, "sort maxima");
        k_widen<<<unsigned((nm + 255) / 256), 256, 0, st>>>(t->d_alt, max64, nm);
        stats->kernel_launches += 5;
    }
    if (ns > 0) {
        size_t b = t->sort_tmp_bytes;
        if ((e = cub::DeviceRadixSort::SortKeys(t->d_sort_tmp, b, t->d_sad, sad32, int(ns), 0, bits, st)) !=
            cudaSuccess)
            return fail(err, e, "sort saddles");
        k_widen<<<unsigned((ns + 255) / 256), 256, 0, st>>>(sad32, sad64, ns);
        stats->kernel_launches += 5;
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return fail(err, e, "lists");
    return EG_OK;
}

}  // namespace eg
