// Tiled path for n <= 3 grids (2-D and 1-D grids are 3-D grids with unit
// axes: the Freudenthal link of a 2-D vertex is exactly the dz = 0 part of the
// 3-D link, Fig. 2).
//
// Pass T  (k_tile): one CTA per 32 x 16 x 16 tile (2 CTAs per SM).  The tile
//         plus a one-vertex halo ("ghost vertices") is brought into
//         shared memory by one TMA bulk-tensor copy; every thread walks one
//         z-column and computes, per vertex,
//           S1  the gradient = SoS argmax of the closed star,
//               separably: closed star = box(v) u box(v - 1), box(w) = w + {0,1}^3,
//               so the argmax is 2x2 in-plane maxima combined across z;
//           S3  the 14-bit upper mask -> "beta0+ >= 2" from a 2 KB bit LUT
//               (Table 1; maximum iff the mask is empty).
//         The gradients are stored as 16-bit indices into the halo box and
//         compressed by pointer doubling in shared memory (S2 inside the tile):
//         every vertex ends at an in-tile maximum (its final label) or at the
//         first halo vertex on its path (an exit: the path leaves the tile, the
//         paper's partial path P:296).  label[v] = global id of that root, with
//         bit 31 set for exits; the distinct exit targets of the tile are
//         appended to a list E.
// Pass E  (k_resolve_exits): for every e in E, follow label[] (one dependent
//         load per tile hop) to the maximum and store it in label[e].
// Pass X  (k_exit_final): every exiting vertex takes label[label[v]] (its exit
//         target is in E, hence final).
// All in-place updates are race-benign: every value ever stored on a chain is
// a later vertex of the same ascending path.
#include <cooperative_groups.h>
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "eg_tiled.h"

namespace eg {

namespace cg = cooperative_groups;

constexpr int TX = 32, TY = 16, TZ = 16;
constexpr int XO = 4;                                // box x index of the tile's first column
constexpr int BX = TX + 2 * XO;                      // 40: TMA box starts at x0 - 4 (16-byte aligned start)
constexpr int BY = TY + 2, BZ = TZ + 2;
constexpr int PL = BX * BY;
constexpr int BOX = PL * BZ;                         // 11664 < 65536: 16-bit box indices
constexpr int kThreads = TX * TY;                    // one z-column per thread
constexpr int kLutWords = (1 << 14) / 32;            // 1 bit per 14-bit upper mask: beta0+ >= 2
constexpr uint32_t kFlag = 0x80000000u;              // label bit 31: exit (not yet final)
constexpr int kFboxSlack = XO + BX + PL;             // shifted TMA boxes spill this far past the box
constexpr size_t kOffP = size_t(BOX + kFboxSlack) * 4;  // pbox after fbox
constexpr size_t kOffL = kOffP + size_t(BOX) * 2;    // lut bits
constexpr size_t kOffM = kOffL + size_t(kLutWords) * 4;
constexpr size_t kOffT = kOffM + 16 + 33 * 4 + 16;  // plane table (PL int32)
constexpr size_t kTileSmem = kOffT + size_t(PL) * 4; // ~81 KB -> 2 CTAs per SM (register-limited)

struct Tiled3D {
    uint32_t *d_lut = nullptr;
    bool ready = false;
    int64_t bdims[3] = {0, 0, 0};
    int64_t bz[2] = {-1, -1};                        // slab planes of the cached list
    bool bcluster = false;                           // cluster mode of the cached list
    bool use_cluster = false;
    int rounds = 2;
    int32_t *d_btiles = nullptr;                     // boundary tile list for the cached dims
    int32_t *d_ptab = nullptr;                       // plane table for nx = ptab_nx
    int64_t ptab_nx = -1;
    int64_t n_btiles = 0;
    int32_t *d_elist = nullptr;                      // exit targets E
    int64_t ecap = 0;
    unsigned long long *d_ecount = nullptr;
    void *encode = nullptr;                          // cuTensorMapEncodeTiled
};

Tiled3D *tiled3d_create() { return new Tiled3D(); }

void tiled3d_destroy(Tiled3D *t) {
    if (!t) return;
    if (t->d_lut) cudaFree(t->d_lut);
    if (t->d_btiles) cudaFree(t->d_btiles);
    if (t->d_ptab) cudaFree(t->d_ptab);
    if (t->d_elist) cudaFree(t->d_elist);
    if (t->d_ecount) cudaFree(t->d_ecount);
    delete t;
}

struct Dims3 {
    int32_t nx, ny, nz;
};

constexpr int kResOff = (BOX + 255) / 256 * 256;     // cluster: resolved shell values after the used bytes
constexpr int kUbitWords = (BOX + 31) / 32;          // exit-target bitmap
constexpr int kTlistOff = kUbitWords * 4;            // exit-target list (uint16 box cells) after it
static_assert(kTlistOff + BOX * 2 <= (BOX + kFboxSlack) * 4, "target list fits the dead field box");

struct TileArgs {
    const float *f;                 // owned planes [z_lo, z_hi) of the slab
    const float *f_lo, *f_hi;       // halo planes z_lo - 1 and z_hi (neighbour slabs) or null
    int32_t z_lo, z_hi;
    int64_t v0;                     // global id of the first owned vertex
    int32_t *label;                 // owned labels (index v - v0)
    uint32_t *exit_bits, *sad_bits, *max_bits;
    int *nan_flag;
    int32_t *elist;
    unsigned long long *ecount;
    int64_t ecap;
    const uint32_t *lut;
    const int32_t *ptab;            // per box-plane cell: by * nx + bx, bit 31 = in-plane shell
    const int32_t *btiles;          // boundary variant: packed tile ids
    int32_t tiles_x, tiles_y;       // interior variant: sub-box extents
    int3 origin;                    // interior variant: first interior tile
    int32_t rounds;                 // pointer-doubling rounds before the chase
};

__device__ __forceinline__ int bidx(int x, int y, int z) { return (z * BY + y) * BX + x; }

// The halo shell of a tile box (cells a path can exit to): the two z faces
// (BY rows of TX + 2 columns), the two y faces of the inner planes, and the two
// x columns of the inner rows.
constexpr int kShellW = TX + 2;
constexpr int kShellZ = 2 * BY * kShellW;
constexpr int kShellY = kShellZ + (BZ - 2) * 2 * kShellW;
constexpr int kShell = kShellY + (BZ - 2) * (BY - 2) * 2;
__device__ __forceinline__ int shell_cell(int s) {
    int bx, by, bz;
    if (s < kShellZ) {
        bz = s < BY * kShellW ? 0 : BZ - 1;
        const int t = s % (BY * kShellW);
        by = t / kShellW;
        bx = XO - 1 + t % kShellW;
    } else if (s < kShellY) {
        const int t = s - kShellZ;
        bz = 1 + t / (2 * kShellW);
        const int u = t % (2 * kShellW);
        by = u < kShellW ? 0 : BY - 1;
        bx = XO - 1 + u % kShellW;
    } else {
        const int t = s - kShellY;
        bz = 1 + t / (2 * (BY - 2));
        const int u = t % (2 * (BY - 2));
        by = 1 + (u >> 1);
        bx = (u & 1) ? XO + TX : XO - 1;
    }
    return bidx(bx, by, bz);
}

__device__ __forceinline__ bool is_shell_xyz(int bx, int by, int bz) {
    return bx < XO || bx >= XO + TX || by == 0 || by == BY - 1 || bz == 0 || bz == BZ - 1;
}
__device__ __forceinline__ bool is_shell(int r) {
    const int bz = r / PL, rr = r - bz * PL;
    const int by = rr / BX, bx = rr - by * BX;
    return is_shell_xyz(bx, by, bz);
}
// inverse of shell_cell for a shell cell (bx, by, bz)
__device__ __forceinline__ int shell_index(int bx, int by, int bz) {
    if (bz == 0 || bz == BZ - 1) return (bz ? BY * kShellW : 0) + by * kShellW + (bx - (XO - 1));
    if (by == 0 || by == BY - 1) return kShellZ + (bz - 1) * 2 * kShellW + (by ? kShellW : 0) + (bx - (XO - 1));
    return kShellY + (bz - 1) * 2 * (BY - 2) + (by - 1) * 2 + (bx == XO + TX ? 1 : 0);
}

struct Dims3;
// Follow a path that leaves tile (cx, cy, cz) of a 2x2x2 cluster at its shell
// cell i through the siblings' pointer boxes (sib[rank], rank = x + 2y + 4z)
// until it ends at a maximum inside the super-tile (final label) or leaves it
// (kUnresolved | the first vertex outside).  (sx0, sy0, sz0): global origin
// of the super-tile.
__device__ int32_t resolve_in_cluster(int i, int cx, int cy, int cz, const uint16_t *const *sib, int sx0, int sy0,
                                      int sz0, const Dims3 &D);

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

__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, uint64_t *bar, int x, int y, int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}

// ------------------------------------------------------------ the tile kernel

__device__ int32_t resolve_in_cluster(int i, int cx, int cy, int cz, const uint16_t *const *sib, int sx0, int sy0,
                                      int sz0, const Dims3 &D) {
    int idx = i;
    for (;;) {
        const int bz = idx / PL, rr = idx - bz * PL;
        const int by = rr / BX, bx = rr - by * BX;
        // super-tile coordinates of the vertex at this box cell
        const int sx = cx * TX + bx - XO, sy = cy * TY + by - 1, sz = cz * TZ + bz - 1;
        const int32_t gid = ((sz0 + sz) * D.ny + (sy0 + sy)) * D.nx + (sx0 + sx);
        if (!is_shell_xyz(bx, by, bz)) return gid;                       // a maximum of that tile
        if (sx < 0 || sx >= 2 * TX || sy < 0 || sy >= 2 * TY || sz < 0 || sz >= 2 * TZ)
            return int32_t(uint32_t(gid) | kFlag);                        // leaves the super-tile
        cx = sx / TX;
        cy = sy / TY;
        cz = sz / TZ;
        idx = sib[cx + 2 * cy + 4 * cz][bidx(sx - cx * TX + XO, sy - cy * TY + 1, sz - cz * TZ + 1)];
    }
}

struct VK {           // a value with its box-index offset from the centre vertex
    float v;
    int d;
};

// b wins ties: b is the later (higher-index) operand
__device__ __forceinline__ VK vmax(VK a, VK b) { return b.v >= a.v ? b : a; }
// the same where NaN marks a cell outside the domain: a NaN never wins
__device__ __forceinline__ VK vmaxn(VK a, VK b) { return (b.v >= a.v || a.v != a.v) ? b : a; }

// IEEE compares (no ftz: distinct denormals stay distinct, reading L2; a NaN
// compares false): m |= kBit if a > b (a >= b), one FSETP + one predicated LOP3
template <uint32_t kBit>
__device__ __forceinline__ void or_if_gt(uint32_t &m, float a, float b) {
    asm("{\n\t.reg .pred p;\n\tsetp.gt.f32 p, %1, %2;\n\t@p or.b32 %0, %0, %3;\n\t}" : "+r"(m) : "f"(a), "f"(b), "n"(kBit));
}
template <uint32_t kBit>
__device__ __forceinline__ void or_if_ge(uint32_t &m, float a, float b) {
    asm("{\n\t.reg .pred p;\n\tsetp.ge.f32 p, %1, %2;\n\t@p or.b32 %0, %0, %3;\n\t}" : "+r"(m) : "f"(a), "f"(b), "n"(kBit));
}

template <bool kInterior, bool kTma, bool kCluster>
__global__ void __launch_bounds__(kThreads, 2)
    k_tile(const __grid_constant__ CUtensorMap tmap, TileArgs A, Dims3 D) {
    extern __shared__ __align__(128) unsigned char smem[];
    float *fbox = reinterpret_cast<float *>(smem);
    uint16_t *pbox = reinterpret_cast<uint16_t *>(smem + kOffP);
    uint32_t *lut = reinterpret_cast<uint32_t *>(smem + kOffL);
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + kOffM);

    const int tid = threadIdx.x;
    const int tx = tid & 31, ty = tid >> 5;
    int bxo, byo, bzo;
    if (kCluster) {
        bxo = int(blockIdx.x) + A.origin.x;
        byo = int(blockIdx.y) + A.origin.y;
        bzo = int(blockIdx.z) + A.origin.z;
    } else if (kInterior) {
        int t = blockIdx.x;
        bxo = t % A.tiles_x + A.origin.x;
        t /= A.tiles_x;
        byo = t % A.tiles_y + A.origin.y;
        bzo = t / A.tiles_y + A.origin.z;
    } else {
        const int packed = A.btiles[blockIdx.x];     // (bz << 20) | (by << 10) | bx
        bxo = packed & 1023;
        byo = (packed >> 10) & 1023;
        bzo = packed >> 20;
    }
    const int x0 = bxo * TX, y0 = byo * TY, z0 = A.z_lo + bzo * TZ;

    // ---- stage the tile + halo: one TMA bulk-tensor copy (or plain loads).
    // A TMA box must start at a non-negative, 16-byte aligned x (measured,
    // tools/tma_probe): at the low domain faces the box starts at 0 and is
    // written shifted by one row / plane / 4 columns into the smem box (the
    // cells it then spills into are padding or never-read halo of an invalid
    // side; kFboxSlack covers the spill past the end).  Tiles whose box needs
    // a neighbour slab's halo plane take the plain loads.
    bool use_tma = kTma;
    if (kTma && !kInterior)
        use_tma = !((z0 - 1 >= 0 && z0 - 1 < A.z_lo) || (z0 + TZ < D.nz && z0 + TZ >= A.z_hi));
    if (use_tma) {
        if (tid == 0) {
            mbar_init(bar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        if (tid == 0) {
            const int xs = x0 - XO, ys = y0 - 1, zs = z0 - 1 - A.z_lo;
            const int shift = (xs < 0 ? XO : 0) + (ys < 0 ? BX : 0) + (zs < 0 ? PL : 0);
            mbar_expect_tx(bar, uint32_t(BOX * 4));
            tma_load_3d(fbox + shift, &tmap, bar, xs < 0 ? 0 : xs, ys < 0 ? 0 : ys, zs < 0 ? 0 : zs);
        }
    } else {
        // one warp per box row: the row's source (owned planes, a halo plane
        // of a neighbour slab, or nothing) is decided once per row
        // (4 rows per warp in flight: loads first, then the smem stores)
        const int lane = tid & 31;
        constexpr int kRows = BY * BZ, kWarps = kThreads / 32, kU = 4;
        for (int row0 = tid >> 5; row0 < kRows; row0 += kWarps * kU) {
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
                    const int b = lane + 32 * h;
                    const int gx = x0 + b - XO;
                    v[u][h] = (src && b < BX && gx >= 0 && gx < D.nx) ? __ldg(src + gx) : __int_as_float(0x7fffffff);
                }
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int row = row0 + u * kWarps;
                if (row >= kRows) break;
                fbox[row * BX + lane] = v[u][0];
                if (lane + 32 < BX) fbox[row * BX + lane + 32] = v[u][1];
            }
        }
    }
    // halo / padding cells of the pointer box are terminal (point to themselves);
    // two cells per store
    static_assert(BOX % 2 == 0 && kOffP % 4 == 0, "paired pbox init");
    for (int i = tid; i < BOX / 2; i += kThreads)
        reinterpret_cast<uint32_t *>(pbox)[i] = uint32_t(2 * i) | (uint32_t(2 * i + 1) << 16);
    for (int i = tid; i < kLutWords; i += kThreads) lut[i] = __ldg(A.lut + i);
    int32_t *ptab = reinterpret_cast<int32_t *>(smem + kOffT);
    for (int i = tid; i < PL; i += kThreads) ptab[i] = __ldg(A.ptab + i);
    if (use_tma) mbar_wait(bar, 0);
    __syncthreads();

    const int gx = x0 + tx, gy = y0 + ty;
    const bool col_ok = kInterior || (gx < D.nx && gy < D.ny);
    const int cb = bidx(tx + XO, ty + 1, 0);

    // 2-D star of box plane bz at this column: c, (1,0), (0,1), (1,1), (-1,0), (0,-1), (-1,-1)
    auto star = [&](int bz, float *s) {
        const float *p = fbox + cb + bz * PL;
        s[0] = p[0];
        s[1] = p[1];
        s[2] = p[BX];
        s[3] = p[BX + 1];
        s[4] = p[-1];
        s[5] = p[-BX];
        s[6] = p[-BX - 1];
    };
    // in-plane 2x2 maxima (ascending index order inside each, later wins ties).
    // Edge tiles hold NaN in the cells outside the domain: a NaN never wins
    // (vmaxn) and every compare with it is false, so the truncated link
    // (reading L3) falls out of the same code.
    auto vm = [](VK a, VK b) -> VK { return kInterior ? vmax(a, b) : vmaxn(a, b); };
    auto bplus = [&](const float *s, int dz) -> VK {    // (0,0) (1,0) (0,1) (1,1)
        VK a = vm(VK{s[0], dz * PL}, VK{s[1], 1 + dz * PL});
        VK b = vm(VK{s[2], BX + dz * PL}, VK{s[3], BX + 1 + dz * PL});
        return vm(a, b);
    };
    auto bminus = [&](const float *s, int dz) -> VK {   // (-1,-1) (0,-1) (-1,0) (0,0)
        VK a = vm(VK{s[6], -BX - 1 + dz * PL}, VK{s[5], -BX + dz * PL});
        VK b = vm(VK{s[4], -1 + dz * PL}, VK{s[0], dz * PL});
        return vm(a, b);
    };

    float pm[7], p0[7], pp[7];
    star(0, pm);
    star(1, p0);
    VK bm_prev = bminus(pm, -1);       // B-(z-1) for z = 0
    VK bp_cur = bplus(p0, 0);          // B+(z)   for z = 0
    uint32_t sad_mask = 0, max_mask = 0;
    bool nan_seen = false;
#pragma unroll 4
    for (int z = 0; z < TZ; ++z) {
        star(z + 2, pp);
        const int gz = z0 + z;
        const bool ok = col_ok && (kInterior || gz < A.z_hi);
        const float fv = p0[0];
        nan_seen |= ok && (fv != fv);
        // S1: argmax over box(v) u box(v - 1); the upper box wins ties
        const VK bp_next = bplus(pp, 1);
        const VK bm_cur = bminus(p0, 0);
        const VK U = vm(bp_cur, bp_next);
        const VK L = vm(bm_prev, bm_cur);
        const int d = vm(L, U).d;
        bp_cur = VK{bp_next.v, bp_next.d - PL};
        bm_prev = VK{bm_cur.v, bm_cur.d - PL};
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
        const int c = cb + (z + 1) * PL;
        if (ok) pbox[c] = uint16_t(c + d);
        const bool sad = (lut[mask >> 5] >> (mask & 31)) & 1u;
        sad_mask |= (ok && sad) ? (1u << z) : 0u;
        max_mask |= (ok && mask == 0) ? (1u << z) : 0u;
#pragma unroll
        for (int k = 0; k < 7; ++k) {
            pm[k] = p0[k];
            p0[k] = pp[k];
        }
    }
    if (nan_seen) atomicOr(A.nan_flag, 1);
    __syncthreads();

    // fbox is dead from here.  Cluster: 1 byte per box cell marks the shell
    // cells used as roots, resolved values after them.  Otherwise: a bitmap of
    // the exit targets (the first vertex to set a bit appends the cell to a
    // list of the tile's targets, so E needs no scan of the box).
    uint8_t *used = reinterpret_cast<uint8_t *>(fbox);
    int32_t *res = reinterpret_cast<int32_t *>(reinterpret_cast<uint8_t *>(fbox) + kResOff);   // cluster only
    uint32_t *ubits = reinterpret_cast<uint32_t *>(fbox);
    uint16_t *tlist = reinterpret_cast<uint16_t *>(reinterpret_cast<uint8_t *>(fbox) + kTlistOff);
    uint32_t *tcount = reinterpret_cast<uint32_t *>(smem + kOffM + 16 + 33 * 4 + 8);
    if constexpr (kCluster) {
        static_assert(BOX % 16 == 0, "uint4 clear of the used bytes");
        for (int i = tid; i < BOX / 16; i += kThreads) reinterpret_cast<uint4 *>(used)[i] = make_uint4(0, 0, 0, 0);
    } else {
        for (int i = tid; i < kUbitWords; i += kThreads) ubits[i] = 0u;
        if (tid == 0) *tcount = 0u;
    }

    // ---- S2 inside the tile.  Two rounds of pointer doubling (independent
    // loads, no divergence) quarter every chain; then every vertex follows the
    // rest of its chain to the local root and stores the root in its own cell
    // only.  Any other thread reads that cell as either the old pointer or the
    // root -- both lie on the same ascending path -- so nothing needs settling,
    // and chains that run into a finished cell end one hop later.
    // (measured alternatives, profiles/r01: doubling to convergence with a
    // per-vertex done mask ~50 instr/vertex; path halving + a settle pass ~45)
#pragma unroll 1
    for (int round = 0; round < A.rounds; ++round) {
#pragma unroll
        for (int z = 0; z < TZ; ++z) {
            const int c = cb + (z + 1) * PL;
            pbox[c] = pbox[pbox[c]];
        }
        __syncthreads();
    }
    auto chase = [&](int c) -> int {
        int x = pbox[c];
        for (int q; (q = pbox[x]) != x;) x = q;
        pbox[c] = uint16_t(x);
        return x;
    };

    // ---- outputs: label (bit 31 = exit), bitmaps, exit-target marks
    const bool aligned = (D.nx & 31) == 0;
    // 32-bit index arithmetic (N < 2^31): the global id of box cell (0,0,0),
    // the plane stride, and this column's owned index at z = 0
    const int32_t nxy = D.ny * D.nx;
    const int32_t g_box0 = ((z0 - 1) * D.ny + (y0 - 1)) * D.nx + (x0 - XO);
    const int32_t i_col = (z0 * D.ny + gy) * D.nx + gx - int32_t(A.v0);
    if constexpr (kCluster) {
        // The 2x2x2 tiles of a thread-block cluster form a super-tile: a path
        // that leaves this tile into a sibling is followed through the
        // sibling's pointer box in distributed shared memory, so only paths
        // leaving the super-tile remain exits.
        //   A: final roots into the own box, mark the shell cells used as roots
#pragma unroll 1
        for (int z = 0; z < TZ; ++z) chase(cb + (z + 1) * PL);
        __syncthreads();
#pragma unroll 1
        for (int z = 0; z < TZ; ++z) {
            const int r = pbox[cb + (z + 1) * PL];
            if (is_shell(r)) used[r] = 1;
        }
        cg::this_cluster().sync();
        //   B: resolve every used shell cell through the siblings
        const dim3 cbi = cg::this_cluster().block_index();
        const uint16_t *sib[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) sib[q] = cg::this_cluster().map_shared_rank(pbox, q);
        const int sx0 = x0 - int(cbi.x) * TX, sy0 = y0 - int(cbi.y) * TY, sz0 = z0 - int(cbi.z) * TZ;
        for (int s = tid; s < kShell; s += kThreads) {
            const int i = shell_cell(s);
            if (used[i]) res[s] = resolve_in_cluster(i, int(cbi.x), int(cbi.y), int(cbi.z), sib, sx0, sy0, sz0, D);
        }
        cg::this_cluster().sync();      // no sibling reads this box after this point
    }
#pragma unroll 2
    for (int z = 0; z < TZ; ++z) {
        const int gz = z0 + z;
        const bool ok = col_ok && (kInterior || gz < A.z_hi);
        const int c = cb + (z + 1) * PL;
        const int r = kCluster ? int(pbox[c]) : chase(c);   // the local root
        const int bz = r / PL, rr = r - bz * PL;
        const int32_t t = ptab[rr];
        // exit: the root is in the halo shell of the box, or (last tile of a
        // slab) in a plane the slab does not own
        bool exit = t < 0 || bz == 0 || bz == BZ - 1 || (!kInterior && z0 - 1 + bz >= A.z_hi);
        int32_t lab;
        if (kCluster && exit) {
            const int by = rr / BX, bx = rr - by * BX;
            lab = res[shell_index(bx, by, bz)];
            exit = lab < 0;
        } else {
            const int32_t root = g_box0 + bz * nxy + (t & 0x7fffffff);
            lab = exit ? int32_t(uint32_t(root) | kFlag) : root;
        }
        const int32_t i = i_col + z * nxy;               // owned index of this vertex
        if (ok) {
            A.label[i] = lab;
            if (!kCluster && exit) {
                const uint32_t bit = 1u << (r & 31);
                if (!(atomicOr(ubits + (r >> 5), bit) & bit)) tlist[atomicAdd(tcount, 1u)] = uint16_t(r);
            }
        }
        const uint32_t eb = __ballot_sync(0xffffffffu, ok && exit);
        const uint32_t sb = __ballot_sync(0xffffffffu, (sad_mask >> z) & 1u);
        const uint32_t mb = __ballot_sync(0xffffffffu, (max_mask >> z) & 1u);
        if (aligned) {
            if (tx == 0 && ok) {
                const int32_t w = i >> 5;
                A.exit_bits[w] = eb;
                A.sad_bits[w] = sb;
                A.max_bits[w] = mb;
            }
        } else {
            const int64_t r0 = int64_t((gz * D.ny + gy) * D.nx + x0) - A.v0;
            const bool row_ok = kInterior || (gy < D.ny && gz < A.z_hi);
            if (tx == 0 && row_ok && (eb | sb | mb)) {
                const int sh = int(r0 & 31);
                const int64_t w = r0 >> 5;
                atomicOr(A.exit_bits + w, eb << sh);
                atomicOr(A.sad_bits + w, sb << sh);
                atomicOr(A.max_bits + w, mb << sh);
                if (sh) {
                    atomicOr(A.exit_bits + w + 1, eb >> (32 - sh));
                    atomicOr(A.sad_bits + w + 1, sb >> (32 - sh));
                    atomicOr(A.max_bits + w + 1, mb >> (32 - sh));
                }
            }
        }
    }
    __syncthreads();
    // ---- append the tile's exit targets to E: one global atomic per tile
    if constexpr (kCluster) {
        // block scan of per-thread counts over the shell cells whose path
        // leaves the super-tile; E gets the resolved vertex outside
        uint32_t *red = reinterpret_cast<uint32_t *>(smem + kOffM + 16);   // [32] warp sums + [1] base
        auto is_target = [&](int s, int i) -> bool { return used[i] && res[s] < 0; };
        int mine = 0;
        for (int s = tid; s < kShell; s += kThreads) mine += is_target(s, shell_cell(s));
        int incl = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (tx >= o) incl += y;
        }
        if (tx == 31) red[ty] = uint32_t(incl);
        __syncthreads();
        if (ty == 0) {
            const int wsum = tx < kThreads / 32 ? int(red[tx]) : 0;
            int wincl = wsum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, wincl, o);
                if (tx >= o) wincl += y;
            }
            if (tx < kThreads / 32) red[tx] = uint32_t(wincl - wsum);   // exclusive warp offsets
            if (tx == kThreads / 32 - 1) {
                const unsigned long long b = wincl ? atomicAdd(A.ecount, (unsigned long long)wincl) : 0ull;
                reinterpret_cast<unsigned long long *>(red + 32)[0] = b;
            }
        }
        __syncthreads();
        if (mine) {
            unsigned long long slot = reinterpret_cast<unsigned long long *>(red + 32)[0] + red[ty] + (incl - mine);
            for (int s = tid; s < kShell; s += kThreads) {
                if (!is_target(s, shell_cell(s))) continue;
                if (slot < (unsigned long long)A.ecap) A.elist[slot] = res[s] & 0x7fffffff;
                ++slot;
            }
        }
    } else {
        unsigned long long *base = reinterpret_cast<unsigned long long *>(smem + kOffM + 16);
        const uint32_t nt = *tcount;
        if (tid == 0) *base = nt ? atomicAdd(A.ecount, (unsigned long long)nt) : 0ull;
        __syncthreads();
        const unsigned long long b0 = *base;
        for (uint32_t j = tid; j < nt; j += kThreads) {
            const int i = tlist[j];
            const int bz = i / PL, rr = i - bz * PL;
            if (b0 + j < (unsigned long long)A.ecap) A.elist[b0 + j] = g_box0 + bz * nxy + (ptab[rr] & 0x7fffffff);
        }
    }
}

// Pass E: resolve every owned exit target through the exit graph (bit 31 =
// not final), one dependent load per tile hop.  A path that leaves the slab
// stops at its first remote vertex (resolved later by the boundary exchange).
__global__ void __launch_bounds__(256) k_resolve_exits(int32_t *label, const int32_t *__restrict__ elist,
                                                       const unsigned long long *ecount, int64_t ecap, int64_t v0,
                                                       int64_t v1) {
    const int64_t n = int64_t(min(*ecount, (unsigned long long)ecap));
    for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += int64_t(gridDim.x) * blockDim.x) {
        const int64_t e = elist[j];
        if (e < v0 || e >= v1) continue;                 // a halo vertex: another slab's
        int32_t w = *(volatile int32_t *)(label + (e - v0));
        if (w >= 0) continue;
        for (;;) {
            const int64_t x = w & 0x7fffffff;
            if (x < v0 || x >= v1) break;                 // remote: stays unresolved
            const int32_t nw = *(volatile int32_t *)(label + (x - v0));
            w = nw;
            if (w >= 0) break;
        }
        label[e - v0] = w;
    }
}

// Pass E' (fallback when E overflowed): every exiting vertex chases its own
// path as far as the slab allows.
__global__ void __launch_bounds__(256) k_exit_chase(int32_t *label, const uint32_t *__restrict__ exit_bits, int64_t v0,
                                                    int64_t v1) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= v1 - v0) return;
    if (!((__ldg(exit_bits + (i >> 5)) >> (i & 31)) & 1u)) return;
    int32_t w = label[i];
    while (w < 0) {
        const int64_t x = w & 0x7fffffff;
        if (x < v0 || x >= v1) break;
        w = *(volatile int32_t *)(label + (x - v0));
    }
    label[i] = w;
}

__global__ void k_zero_words(uint32_t *a, uint32_t *b, uint32_t *c, int64_t n) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        a[i] = 0;
        b[i] = 0;
        c[i] = 0;
    }
}

// --------------------------------------------------------------- host side

static eg_status fail(std::string *err, cudaError_t e, const char *what) {
    if (err) *err = std::string(what) + ": " + cudaGetErrorString(e);
    return e == cudaErrorMemoryAllocation ? EG_ERR_OOM : EG_ERR_CUDA;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <bool I, bool T, bool C>
static cudaError_t set_smem_attr() {
    return cudaFuncSetAttribute(k_tile<I, T, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kTileSmem));
}

eg_status tiled3d_local(Tiled3D *t, int ndim, const int64_t *dims, const Slab &s, const FieldView &F, int32_t *labels,
                        uint32_t *sad_bits, uint32_t *max_bits, uint32_t *exit_bits, int *flags, cudaStream_t st,
                        eg_stats *stats, std::string *err, cudaEvent_t ev_main0, cudaEvent_t ev_main1) {
    int64_t d3[3] = {1, 1, 1};
    for (int i = 0; i < ndim; ++i) d3[i] = dims[i];
    cudaError_t e;
    if (!t->ready) {
        // 1-bit LUT: is beta0+ >= 2 for every 14-bit upper mask of the 3-D link,
        // in the ascending-index offset order (lexicographic in (dz, dy, dx))
        int64_t dl[3] = {4, 4, 4};
        LinkTable tab = make_link_table(3, dl);
        std::vector<uint8_t> beta = make_beta_lut3(tab);
        std::vector<uint32_t> bits(kLutWords, 0u);
        for (int m = 0; m < (1 << 14); ++m)
            if (beta[m] >= 2) bits[m >> 5] |= 1u << (m & 31);
        if ((e = cudaMalloc(&t->d_lut, kLutWords * 4)) != cudaSuccess) return fail(err, e, "cudaMalloc lut");
        if ((e = cudaMemcpy(t->d_lut, bits.data(), kLutWords * 4, cudaMemcpyHostToDevice)) != cudaSuccess)
            return fail(err, e, "lut upload");
        if ((e = cudaMalloc(&t->d_ecount, sizeof(unsigned long long))) != cudaSuccess)
            return fail(err, e, "cudaMalloc ecount");
        if ((e = set_smem_attr<false, false, false>()) != cudaSuccess ||
            (e = set_smem_attr<true, false, false>()) != cudaSuccess ||
            (e = set_smem_attr<true, true, false>()) != cudaSuccess ||
            (e = set_smem_attr<true, true, true>()) != cudaSuccess)
            return fail(err, e, "smem attr");
        // The super-tile kernel is opt-in (EG_CLUSTER=1): on C3 it cut the exit
        // targets by 25 % but made the tile kernel 62 % slower (two cluster
        // barriers per tile; profiles/r01), a net loss.
        const char *cl = std::getenv("EG_CLUSTER");
        t->use_cluster = cl && cl[0] == '1';
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
    const int64_t words = (nown + 31) / 32;
    Dims3 D{int32_t(d3[0]), int32_t(d3[1]), int32_t(d3[2])};
    const int tiles_x = int((d3[0] + TX - 1) / TX), tiles_y = int((d3[1] + TY - 1) / TY);
    const int tiles_z = int((z_hi - z_lo + TZ - 1) / TZ);
    if (tiles_x > 1024 || tiles_y > 1024 || tiles_z > 2047) {
        if (err) *err = "grid too large for the tiled path";
        return EG_ERR_UNSUPPORTED;
    }
    // interior tiles: x/y halo box inside the domain and z box inside the
    // owned planes: 1 <= b <= (extent - 1 - T) / T on every axis
    int3 lo = make_int3(1, 1, 1);
    int3 hi = make_int3(int((d3[0] - 1 - TX) / TX), int((d3[1] - 1 - TY) / TY), int((z_hi - z_lo - 1 - TZ) / TZ));
    if (d3[0] - 1 - TX < 0 || d3[1] - 1 - TY < 0 || z_hi - z_lo - 1 - TZ < 0) hi = make_int3(0, 0, 0);
    bool have_interior = hi.x >= lo.x && hi.y >= lo.y && hi.z >= lo.z;
    // thread-block clusters of 2x2x2 interior tiles (super-tiles resolved in
    // distributed shared memory) need TMA-able fields and an even number of
    // interior tiles per axis; the odd leftovers join the edge-tile list
    const bool tma_ok = t->encode != nullptr && (d3[0] % 4) == 0 && d3[0] >= 4 &&
                        (reinterpret_cast<uintptr_t>(F.own) % 16) == 0;
    const bool cluster = have_interior && tma_ok && t->use_cluster && hi.x - lo.x >= 1 && hi.y - lo.y >= 1 &&
                         hi.z - lo.z >= 1;
    if (cluster) {
        hi.x = lo.x + (hi.x - lo.x + 1) / 2 * 2 - 1;
        hi.y = lo.y + (hi.y - lo.y + 1) / 2 * 2 - 1;
        hi.z = lo.z + (hi.z - lo.z + 1) / 2 * 2 - 1;
    }
    // boundary tile list, cached per (dims, slab, cluster mode)
    if (t->bdims[0] != d3[0] || t->bdims[1] != d3[1] || t->bdims[2] != d3[2] || t->bz[0] != z_lo || t->bz[1] != z_hi ||
        t->bcluster != cluster) {
        t->bcluster = cluster;
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
        if (!bt.empty()) {
            if ((e = cudaMalloc(&t->d_btiles, bt.size() * 4)) != cudaSuccess) return fail(err, e, "cudaMalloc btiles");
            if ((e = cudaMemcpy(t->d_btiles, bt.data(), bt.size() * 4, cudaMemcpyHostToDevice)) != cudaSuccess)
                return fail(err, e, "btiles upload");
        }
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
    const int64_t want = std::max<int64_t>(nown / 8, 4096);
    if (t->ecap < want) {
        if (t->d_elist) cudaFree(t->d_elist);
        t->d_elist = nullptr;
        t->ecap = 0;
        if ((e = cudaMalloc(&t->d_elist, want * 4)) != cudaSuccess) return fail(err, e, "cudaMalloc elist");
        t->ecap = want;
    }
    if ((e = cudaMemsetAsync(t->d_ecount, 0, sizeof(unsigned long long), st)) != cudaSuccess)
        return fail(err, e, "memset ecount");
    const bool aligned = (D.nx & 31) == 0;
    if (!aligned) {
        k_zero_words<<<148 * 4, 256, 0, st>>>(exit_bits, sad_bits, max_bits, words);
        stats->kernel_launches += 1;
    }
    // TMA tensor map over the owned planes (needs 16-byte row and plane strides)
    CUtensorMap tmap;
    std::memset(&tmap, 0, sizeof(tmap));
    bool tma = tma_ok && have_interior;
    if (tma) {
        cuuint64_t gdim[3] = {cuuint64_t(d3[0]), cuuint64_t(d3[1]), cuuint64_t(z_hi - z_lo)};
        cuuint64_t gstr[2] = {cuuint64_t(d3[0] * 4), cuuint64_t(d3[0] * d3[1] * 4)};
        cuuint32_t box[3] = {BX, BY, BZ};
        cuuint32_t es[3] = {1, 1, 1};
        CUresult r = reinterpret_cast<EncodeTiledFn>(t->encode)(
            &tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float *>(F.own), gdim, gstr, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        tma = (r == CUDA_SUCCESS);
    }
    stats->path = 1;
    TileArgs A{F.own,     F.lo,     F.hi,  int32_t(z_lo), int32_t(z_hi), s.v0,    labels,   exit_bits,
               sad_bits,  max_bits, flags, t->d_elist,    t->d_ecount,   t->ecap, t->d_lut, t->d_ptab,
               t->d_btiles, 0,      0,     make_int3(0, 0, 0), t->rounds};
    if (ev_main0) cudaEventRecord(ev_main0, st);
    if (t->n_btiles > 0) {
        // boundary tiles use plain loads: a TMA box must start at a 16-byte
        // aligned, non-negative x coordinate (measured with tools/tma_probe:
        // a start of -1 is an illegal instruction), and these tiles are the
        // ones whose halo starts outside the field or in a neighbour slab
        k_tile<false, false, false><<<unsigned(t->n_btiles), kThreads, kTileSmem, st>>>(tmap, A, D);
        stats->kernel_launches += 1;
        if ((e = cudaGetLastError()) != cudaSuccess) return fail(err, e, "k_tile<boundary>");
    }
    if (have_interior && tma && cluster) {
        A.origin = lo;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(unsigned(hi.x - lo.x + 1), unsigned(hi.y - lo.y + 1), unsigned(hi.z - lo.z + 1));
        cfg.blockDim = dim3(kThreads, 1, 1);
        cfg.dynamicSmemBytes = kTileSmem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 2;
        attr[0].val.clusterDim.z = 2;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if ((e = cudaLaunchKernelEx(&cfg, k_tile<true, true, true>, tmap, A, D)) != cudaSuccess)
            return fail(err, e, "k_tile<cluster>");
        stats->kernel_launches += 1;
    } else if (have_interior) {
        A.tiles_x = hi.x - lo.x + 1;
        A.tiles_y = hi.y - lo.y + 1;
        A.origin = lo;
        const int64_t nt = int64_t(A.tiles_x) * A.tiles_y * (hi.z - lo.z + 1);
        if (tma)
            k_tile<true, true, false><<<unsigned(nt), kThreads, kTileSmem, st>>>(tmap, A, D);
        else
            k_tile<true, false, false><<<unsigned(nt), kThreads, kTileSmem, st>>>(tmap, A, D);
        stats->kernel_launches += 1;
        if ((e = cudaGetLastError()) != cudaSuccess) return fail(err, e, "k_tile<interior>");
    }
    if (ev_main1) cudaEventRecord(ev_main1, st);
    // resolve the owned part of E
    k_resolve_exits<<<148 * 64, 256, 0, st>>>(labels, t->d_elist, t->d_ecount, t->ecap, s.v0, s.v1);
    stats->kernel_launches += 1;
    if ((e = cudaGetLastError()) != cudaSuccess) return fail(err, e, "k_resolve_exits");
    unsigned long long ecount = 0;
    if ((e = cudaMemcpyAsync(&ecount, t->d_ecount, sizeof(ecount), cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
        (e = cudaStreamSynchronize(st)) != cudaSuccess)
        return fail(err, e, "ecount");
    stats->n_exit_targets += int64_t(ecount);
    if (int64_t(ecount) > t->ecap) {
        // E overflowed: every exiting vertex chases its own path (exact, slower)
        k_exit_chase<<<unsigned((nown + 255) / 256), 256, 0, st>>>(labels, exit_bits, s.v0, s.v1);
        stats->kernel_launches += 1;
        if ((e = cudaGetLastError()) != cudaSuccess) return fail(err, e, "k_exit_chase");
    }
    return EG_OK;
}

}  // namespace eg
