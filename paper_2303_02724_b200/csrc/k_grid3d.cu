// Tiled path for n <= 3 grids (2-D and 1-D grids are 3-D grids with unit
// axes: the Freudenthal link of a 2-D vertex is exactly the dz = 0 part of the
// 3-D link).
//
// Pass T  (k_tile): one CTA per 32 x 16 x 16 tile.  The tile plus a one-vertex
//         halo is staged in shared memory; every thread walks one z-column,
//         keeping the 2-D stars of three planes in registers, and computes
//           S1  the gradient (SoS argmax of the closed star),
//           S3  the 14-bit upper mask -> beta0+ from a 16 KB LUT.
//         The gradient of every tile vertex is then stored as a 16-bit index
//         into the halo box and chased in shared memory to its local root
//         (S2 inside the tile): an in-tile maximum (final label) or the first
//         halo vertex on the path (an "exit": the path leaves the tile, the
//         paper's partial path P:296).  The kernel writes label[v] = global id
//         of that root, and bit v of the exit / saddle / maximum bitmaps.
// Pass X  (k_exit_fixup): for every exiting vertex, follow label[] through
//         the exit bitmap (tile hop by tile hop) to the maximum and store it.
//         In-place and race-benign: every value ever stored on a chain is a
//         later vertex of the same ascending path.
#include <cuda_runtime.h>

#include <cstdio>

#include "eg_tiled.h"

namespace eg {

constexpr int TX = 32, TY = 16, TZ = 16;
constexpr int BX = TX + 2, BY = TY + 2, BZ = TZ + 2;
constexpr int BOX = BX * BY * BZ;                    // 11016 < 65536: 16-bit box indices
constexpr int kThreads = TX * TY;                   // one z-column per thread
constexpr int kLut = 1 << 14;
constexpr size_t kTileSmem = 6 * BOX + kLut;        // 82,480 B -> 2 CTAs per SM

struct Tiled3D {
    uint8_t *d_lut = nullptr;
    bool lut_ready = false;
};

Tiled3D *tiled3d_create() { return new Tiled3D(); }

void tiled3d_destroy(Tiled3D *t) {
    if (!t) return;
    if (t->d_lut) cudaFree(t->d_lut);
    delete t;
}

struct Dims3 {
    int32_t nx, ny, nz;
    int64_t nxy;
};

__device__ __forceinline__ int bidx(int x, int y, int z) { return (z * BY + y) * BX + x; }  // x, y, z in box coords

// The 14 link offsets of a 3-D vertex in ascending global index (lexicographic
// in (dz, dy, dx)):
//   lower group (index < v): (-1,-1,-1) (0,-1,-1) (-1,0,-1) (0,0,-1) (-1,-1,0) (0,-1,0) (-1,0,0)
//   upper group (index > v): (1,0,0) (0,1,0) (1,1,0) (0,0,1) (1,0,1) (0,1,1) (1,1,1)
// Bit k of the upper mask follows this order (lower group bits 0..6, upper 7..13),
// which is the order of LinkTable for dims >= 2 -- the LUT is built from it.
template <bool kInterior>
__global__ void __launch_bounds__(kThreads, 2) k_tile(const float *__restrict__ f, Dims3 D,
                                                      const uint8_t *__restrict__ lut_g, int32_t *__restrict__ label,
                                                      uint32_t *exit_bits, uint32_t *sad_bits, uint32_t *max_bits,
                                                      int *nan_flag, int tiles_x, int tiles_y, int3 origin,
                                                      int3 skip_lo, int3 skip_hi) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float *fbox = reinterpret_cast<float *>(smem_raw);                       // BOX floats
    uint16_t *pbox = reinterpret_cast<uint16_t *>(smem_raw + 4 * BOX);      // BOX uint16
    uint8_t *lut = smem_raw + 6 * BOX;                                        // 16 KB

    const int tid = threadIdx.x;
    const int tx = tid & 31, ty = tid >> 5;
    int t = blockIdx.x;
    const int bxi = t % tiles_x;
    t /= tiles_x;
    const int byi = t % tiles_y + origin.y;
    const int bzi = t / tiles_y + origin.z;
    const int bxo = bxi + origin.x;
    // the checked variant skips the interior sub-box (launched separately)
    if (!kInterior && bxo >= skip_lo.x && bxo <= skip_hi.x && byi >= skip_lo.y && byi <= skip_hi.y &&
        bzi >= skip_lo.z && bzi <= skip_hi.z)
        return;
    const int x0 = bxo * TX, y0 = byi * TY, z0 = bzi * TZ;

    // ---- stage the tile + halo (and the LUT) in shared memory; halo cells of
    // the pointer box point to themselves (terminal: the path leaves the tile)
    for (int i = tid; i < kLut / 16; i += kThreads)
        reinterpret_cast<uint4 *>(lut)[i] = __ldg(reinterpret_cast<const uint4 *>(lut_g) + i);
    for (int i = tid; i < BOX; i += kThreads) {
        const int bx = i % BX, r = i / BX;
        const int by = r % BY, bz = r / BY;
        const int gx = x0 + bx - 1, gy = y0 + by - 1, gz = z0 + bz - 1;
        float v = 0.f;
        if (kInterior || (gx >= 0 && gx < D.nx && gy >= 0 && gy < D.ny && gz >= 0 && gz < D.nz))
            v = __ldg(f + (int64_t(gz) * D.nxy + int64_t(gy) * D.nx + gx));
        fbox[i] = v;
        pbox[i] = uint16_t(i);
    }
    __syncthreads();

    const int gx = x0 + tx, gy = y0 + ty;
    const bool col_ok = kInterior || (gx < D.nx && gy < D.ny);
    // validity of the in-plane directions (x-1, x+1, y-1, y+1)
    const bool xm = kInterior || gx > 0, xp = kInterior || gx + 1 < D.nx;
    const bool ym = kInterior || gy > 0, yp = kInterior || gy + 1 < D.ny;

    // 2-D star of a plane at (tx, ty): c, (1,0), (0,1), (1,1), (-1,0), (0,-1), (-1,-1)
    auto star = [&](int bz, float *s) {
        const int b = bidx(tx + 1, ty + 1, bz);
        s[0] = fbox[b];
        s[1] = fbox[b + 1];
        s[2] = fbox[b + BX];
        s[3] = fbox[b + BX + 1];
        s[4] = fbox[b - 1];
        s[5] = fbox[b - BX];
        s[6] = fbox[b - BX - 1];
    };
    // box-index deltas of the 14 offsets, lower group then upper group
    constexpr int PL = BX * BY;
    constexpr int LD[7] = {-1 - BX - PL, -BX - PL, -1 - PL, -PL, -1 - BX, -BX, -1};
    constexpr int UD[7] = {1, BX, 1 + BX, PL, 1 + PL, BX + PL, 1 + BX + PL};
    float pm[7], p0[7], pp[7];
    star(0, pm);
    star(1, p0);

    uint32_t sad_mask = 0, max_mask = 0;
    bool nan_seen = false;
#pragma unroll 2
    for (int z = 0; z < TZ; ++z) {
        star(z + 2, pp);
        const int gz = z0 + z;
        const bool zm = kInterior || gz > 0, zpv = kInterior || gz + 1 < D.nz;
        const bool ok = col_ok && (kInterior || gz < D.nz);
        const float fv = p0[0];
        nan_seen |= ok && (fv != fv);
        const float lv[7] = {pm[6], pm[5], pm[4], pm[0], p0[6], p0[5], p0[4]};
        const bool lok[7] = {zm && xm && ym, zm && ym, zm && xm, zm, xm && ym, ym, xm};
        const float uv[7] = {p0[1], p0[2], p0[3], pp[0], pp[1], pp[2], pp[3]};
        const bool uok[7] = {xp, yp, xp && yp, zpv, zpv && xp, zpv && yp, zpv && xp && yp};
        uint32_t mask = 0;
        // lower neighbour u is above v iff f(u) > f(v) (its index is lower)
        float bl = -__int_as_float(0x7f800000);
        int bld = 0;
#pragma unroll
        for (int k = 0; k < 7; ++k) {
            const bool up = (kInterior || lok[k]) && (lv[k] > fv);
            mask |= up ? (1u << k) : 0u;
            if (up && lv[k] >= bl) {     // ascending index: >= keeps the highest index on ties
                bl = lv[k];
                bld = LD[k];
            }
        }
        // upper neighbour u is above v iff f(u) >= f(v)
        float bu = fv;
        int bud = 0;
#pragma unroll
        for (int k = 0; k < 7; ++k) {
            const bool up = (kInterior || uok[k]) && (uv[k] >= fv);
            mask |= up ? (1u << (7 + k)) : 0u;
            if (up && uv[k] >= bu) {
                bu = uv[k];
                bud = UD[k];
            }
        }
        // gradient = SoS max over the upper link; an upper-group winner beats a
        // lower-group one on equal values (higher index)
        const int d = (bud != 0 && (bld == 0 || bu >= bl)) ? bud : bld;
        const int c = bidx(tx + 1, ty + 1, z + 1);
        if (ok) pbox[c] = uint16_t(c + d);
        const int beta = lut[mask];
        if (ok && beta >= 2) sad_mask |= 1u << z;
        if (ok && mask == 0) max_mask |= 1u << z;
#pragma unroll
        for (int k = 0; k < 7; ++k) {
            pm[k] = p0[k];
            p0[k] = pp[k];
        }
    }
    if (nan_seen) atomicOr(nan_flag, 1);
    __syncthreads();

    // ---- S2 inside the tile: chase to the local root (path halving in smem;
    // benign races: every stored value lies further along the same path)
    const bool wrow_aligned = (D.nx & 31) == 0;
#pragma unroll 1
    for (int z = 0; z < TZ; ++z) {
        const int gz = z0 + z;
        const bool ok = col_ok && (kInterior || gz < D.nz);
        int x = bidx(tx + 1, ty + 1, z + 1);
        int p = pbox[x];
        while (p != x) {
            const int p2 = pbox[p];
            if (p2 != p) pbox[x] = uint16_t(p2);
            x = p;
            p = p2;
        }
        // root x: in-tile maximum or halo exit
        const int bx = x % BX, r = x / BX;
        const int by = r % BY, bz = r / BY;
        const bool exit = bx == 0 || bx == BX - 1 || by == 0 || by == BY - 1 || bz == 0 || bz == BZ - 1;
        const int64_t root = int64_t(z0 + bz - 1) * D.nxy + int64_t(y0 + by - 1) * D.nx + (x0 + bx - 1);
        const int64_t v = int64_t(gz) * D.nxy + int64_t(gy) * D.nx + gx;
        if (ok) label[v] = int32_t(root);
        const uint32_t eb = __ballot_sync(0xffffffffu, ok && exit);
        const uint32_t sb = __ballot_sync(0xffffffffu, ok && ((sad_mask >> z) & 1u));
        const uint32_t mb = __ballot_sync(0xffffffffu, ok && ((max_mask >> z) & 1u));
        if (wrow_aligned) {
            if (tx == 0 && ok) {
                exit_bits[v >> 5] = eb;
                sad_bits[v >> 5] = sb;
                max_bits[v >> 5] = mb;
            }
        } else {
            // rows are not 32-aligned: lane 0 scatters the ballots into (at
            // most) two words with atomics (the words were zeroed)
            const int64_t v0 = int64_t(gz) * D.nxy + int64_t(gy) * D.nx + x0;
            const bool row_ok = kInterior || (gy < D.ny && gz < D.nz);
            if (tx == 0 && row_ok && (eb | sb | mb)) {
                const int sh = int(v0 & 31);
                const int64_t w = v0 >> 5;
                atomicOr(exit_bits + w, eb << sh);
                atomicOr(sad_bits + w, sb << sh);
                atomicOr(max_bits + w, mb << sh);
                if (sh) {
                    atomicOr(exit_bits + w + 1, eb >> (32 - sh));
                    atomicOr(sad_bits + w + 1, sb >> (32 - sh));
                    atomicOr(max_bits + w + 1, mb >> (32 - sh));
                }
            }
        }
    }
}

// Pass X: resolve every exiting vertex through the exit graph.
__global__ void __launch_bounds__(256) k_exit_fixup(int32_t *label, const uint32_t *__restrict__ exit_bits, int64_t n) {
    const int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const uint32_t w = __ldg(exit_bits + (v >> 5));
    if (!((w >> (v & 31)) & 1u)) return;
    int32_t e = label[v];
    // e is a vertex of another tile; label[e] is its local root, final unless
    // e itself exits
    for (;;) {
        const uint32_t we = *(volatile const uint32_t *)(exit_bits + (e >> 5));
        const int32_t le = *(volatile int32_t *)(label + e);
        if (!((we >> (e & 31)) & 1u)) {
            e = le;
            break;
        }
        e = le;
        // if label[e] was already resolved by another thread, e is now a
        // maximum (not exiting) and the next iteration ends
    }
    label[v] = e;
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

eg_status tiled3d_labels(Tiled3D *t, int ndim, const int64_t *dims, const float *f, int32_t *labels,
                         uint32_t *sad_bits, uint32_t *max_bits, int *flags, cudaStream_t st, eg_stats *stats,
                         std::string *err, uint32_t *exit_bits) {
    int64_t d3[3] = {1, 1, 1};
    for (int i = 0; i < ndim; ++i) d3[i] = dims[i];
    cudaError_t e;
    if (!t->lut_ready) {
        int64_t dl[3] = {4, 4, 4};
        LinkTable tab = make_link_table(3, dl);
        std::vector<uint8_t> lut = make_beta_lut3(tab);
        if ((e = cudaMalloc(&t->d_lut, kLut)) != cudaSuccess) return fail(err, e, "cudaMalloc lut");
        if ((e = cudaMemcpy(t->d_lut, lut.data(), kLut, cudaMemcpyHostToDevice)) != cudaSuccess)
            return fail(err, e, "lut upload");
        if ((e = cudaFuncSetAttribute(k_tile<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kTileSmem))) !=
            cudaSuccess)
            return fail(err, e, "smem attr");
        if ((e = cudaFuncSetAttribute(k_tile<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kTileSmem))) !=
            cudaSuccess)
            return fail(err, e, "smem attr");
        t->lut_ready = true;
    }
    const int64_t N = d3[0] * d3[1] * d3[2];
    const int64_t words = (N + 31) / 32;
    Dims3 D{int32_t(d3[0]), int32_t(d3[1]), int32_t(d3[2]), d3[0] * d3[1]};
    const int tiles_x = int((d3[0] + TX - 1) / TX), tiles_y = int((d3[1] + TY - 1) / TY);
    const int tiles_z = int((d3[2] + TZ - 1) / TZ);
    const bool aligned = (D.nx & 31) == 0;
    if (!aligned) {
        k_zero_words<<<148 * 4, 256, 0, st>>>(exit_bits, sad_bits, max_bits, words);
        stats->kernel_launches += 1;
    }
    // interior tiles (halo box inside the domain) take the unchecked variant
    int3 lo = make_int3(1, 1, 1);
    int3 hi = make_int3(int((d3[0] - 1 - TX) / TX), int((d3[1] - 1 - TY) / TY), int((d3[2] - 1 - TZ) / TZ));
    // tile b is interior iff b >= 1 and (b + 1) * T + 1 <= n, i.e. b <= (n - 1 - T) / T
    const bool have_interior = hi.x >= lo.x && hi.y >= lo.y && hi.z >= lo.z;
    if (!have_interior) {
        lo = make_int3(1, 1, 1);
        hi = make_int3(0, 0, 0);
    }
    const int64_t ntiles = int64_t(tiles_x) * tiles_y * tiles_z;
    k_tile<false><<<unsigned(ntiles), kThreads, kTileSmem, st>>>(f, D, t->d_lut, labels, exit_bits, sad_bits, max_bits,
                                                         flags, tiles_x, tiles_y, make_int3(0, 0, 0), lo, hi);
    stats->kernel_launches += 1;
    if ((e = cudaGetLastError()) != cudaSuccess) return fail(err, e, "k_tile<false>");
    if (have_interior) {
        const int ix = hi.x - lo.x + 1, iy = hi.y - lo.y + 1, iz = hi.z - lo.z + 1;
        k_tile<true><<<unsigned(int64_t(ix) * iy * iz), kThreads, kTileSmem, st>>>(
            f, D, t->d_lut, labels, exit_bits, sad_bits, max_bits, flags, ix, iy, lo, lo, hi);
        stats->kernel_launches += 1;
        if ((e = cudaGetLastError()) != cudaSuccess) return fail(err, e, "k_tile<true>");
    }
    k_exit_fixup<<<unsigned((N + 255) / 256), 256, 0, st>>>(labels, exit_bits, N);
    stats->kernel_launches += 1;
    if ((e = cudaGetLastError()) != cudaSuccess) return fail(err, e, "k_exit_fixup");
    return EG_OK;
}

}  // namespace eg
