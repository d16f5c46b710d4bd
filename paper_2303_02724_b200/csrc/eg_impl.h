// Internal declarations of libeg_b200 (not part of the ABI; see include/eg.h).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "eg.h"

namespace eg {

constexpr int kMaxDim = 6;                 // generic grid kernels: n <= 6
constexpr int kMaxLink = 126;              // 2 (2^6 - 1)
constexpr int kCsrMaxDeg = 128;            // thread-per-vertex CSR kernel

// Freudenthal link of an interior vertex: the offsets d in
// {-1,0,1}^n \ 0 whose non-zero entries share one sign, i.e. the difference
// vectors Alg. 1 accepts.  Sorted by linear offset delta(d) for the actual
// dims, so that scanning in table order visits neighbours in ascending global
// index.  nbr[k] = the link offsets adjacent to offset k (Alg. 1 on offsets).
struct LinkTable {
    int32_t ndim;
    int32_t K;                             // 2 (2^n - 1)
    int32_t pad[2];
    int64_t dims[8];
    int64_t stride[8];
    int8_t d[kMaxLink][8];
    int64_t delta[kMaxLink];
    uint64_t nbr[kMaxLink][2];
};

LinkTable make_link_table(int ndim, const int64_t *dims);
// beta0+ for every 14-bit upper mask of the 3-D link (n = 3, K = 14).
std::vector<uint8_t> make_beta_lut3(const LinkTable &t);

// A slab of the grid as seen by one rank (or one virtual partition).
// Owned vertices: global ids [v0, v1) = planes [z0, z1) of the slowest axis.
// The local field buffer holds planes [h0, h1) = owned planes plus a
// one-plane halo on each side that exists (P:281 ghost vertices).
struct Slab {
    int64_t z0, z1, h0, h1;
    int64_t plane;                         // vertices per plane of the slowest axis
    int64_t v0, v1;                        // owned global ids
    int64_t base;                          // global id of local element 0 = h0 * plane
};

// --------------------------------------------------------------- kernels
// All launchers are asynchronous on `st` and return the launch error.

// S1 + S3, generic n: ptr[i] (global id) for owned i, saddle / maximum bits
// (bit i of word i/32), optional beta0+ per vertex.
cudaError_t launch_classify_grid(const LinkTable *d_tab, int ndim, const float *f_local, const Slab &s,
                                 int32_t *ptr, uint32_t *sad_bits, uint32_t *max_bits, uint8_t *beta_out,
                                 int *nan_flag, cudaStream_t st);
cudaError_t launch_classify_csr(const int64_t *row_ptr, const int32_t *col_idx, const float *f, int64_t v0,
                                int64_t v1, int32_t *ptr, uint32_t *sad_bits, uint32_t *max_bits,
                                uint8_t *beta_out, int *nan_flag, int *deg_overflow, cudaStream_t st);

// S2: in-place pointer jumping over ptr[0..n) whose entries are global ids;
// entries outside [v0, v1) are terminal (remote).  changed[r] is set when
// round r modified something; round r exits immediately if round r-1 did not.
cudaError_t launch_jump_round(int32_t *ptr, int64_t n, int64_t v0, int *changed, int round, cudaStream_t st);

// Compaction of a bitmap over owned indices [0, n) into ascending global ids
// (v0 + i) as int32 and int64.  Needs a scratch of compact_scratch_words(n).
size_t compact_scratch_bytes(int64_t n);
cudaError_t launch_compact_bits(const uint32_t *bits, int64_t n, int64_t v0, void *scratch, int32_t *out32,
                                int64_t *out64, int64_t *d_count, cudaStream_t st);

// S4 for grids and CSR.  Label lookup: label[g - v0] for owned g, else
// halo_label[g - halo_lo_base] for the lower halo plane or
// halo_label[plane + g - halo_hi_base] for the upper halo plane.
struct LabelView {
    const int32_t *own;
    int64_t v0, v1;
    const int32_t *halo;                   // [2 * plane] or null
    int64_t lo_base, hi_base, plane;       // global id of the first vertex of each halo plane
};
cudaError_t launch_saddle_beta_grid(const LinkTable *d_tab, int ndim, const float *f_local, const Slab &s,
                                    const int32_t *saddles, int64_t n_sad, int32_t *beta, cudaStream_t st);
cudaError_t launch_arcs_grid(const LinkTable *d_tab, int ndim, const float *f_local, const Slab &s,
                             const int32_t *saddles, int64_t n_sad, const int64_t *slot_off, LabelView lv,
                             int32_t *tmp_m, int32_t *tmp_mult, int32_t *n_unique, int64_t *raw_s, int64_t *raw_rep,
                             int64_t *raw_m, cudaStream_t st);
cudaError_t launch_saddle_beta_csr(const int64_t *row_ptr, const int32_t *col_idx, const float *f,
                                   const int32_t *saddles, int64_t n_sad, int32_t *beta, cudaStream_t st);
cudaError_t launch_arcs_csr(const int64_t *row_ptr, const int32_t *col_idx, const float *f, const int32_t *saddles,
                            int64_t n_sad, const int64_t *slot_off, LabelView lv, int32_t *tmp_m, int32_t *tmp_mult,
                            int32_t *n_unique, int64_t *raw_s, int64_t *raw_rep, int64_t *raw_m, cudaStream_t st);
cudaError_t launch_emit_arcs(const int32_t *saddles, int64_t n_sad, const int64_t *slot_off, const int64_t *arc_off,
                             const int32_t *tmp_m, const int32_t *tmp_mult, const int32_t *n_unique,
                             int64_t *arc_s, int64_t *arc_m, int32_t *arc_mult, cudaStream_t st);

// exclusive scan of int32 counts into int64 offsets (offsets[n] = total)
size_t scan_scratch_bytes(int64_t n);
cudaError_t launch_scan_i32(const int32_t *in, int64_t *out, int64_t n, void *scratch, size_t scratch_bytes,
                            cudaStream_t st);
cudaError_t launch_i32_to_i64(const int32_t *in, int64_t *out, int64_t n, cudaStream_t st);
cudaError_t launch_nan_scan(const float *f, int64_t n, int *flag, cudaStream_t st);

// --- tiled 3-D path (n <= 3), see k_grid3d.cu
struct Tiled3D;
}  // namespace eg
