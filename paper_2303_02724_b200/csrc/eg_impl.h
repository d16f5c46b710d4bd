// Internal declarations of libeg_b200 (not part of the ABI; see include/eg.h).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "eg.h"

namespace eg {

constexpr int kMaxDim = 8;                 // generic grid kernels: n <= 8
constexpr int kMaxLink = 510;              // 2 (2^8 - 1)
constexpr uint32_t kUnresolved = 0x80000000u;   // label bit 31: not final, low bits = a vertex further on the path

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
    uint64_t nbr[kMaxLink][2];             // (filled for K <= 128, n <= 6: the 3-D LUT builder)
};

LinkTable make_link_table(int ndim, const int64_t *dims);
// beta0+ for every 14-bit upper mask of the 3-D link (n = 3, K = 14).
std::vector<uint8_t> make_beta_lut3(const LinkTable &t);

// A slab of the grid as seen by one rank (or one virtual partition): the
// planes [z0, z1) of the slowest axis ("blocks ... along the z-axis"),
// i.e. the global ids [v0, v1).  One GPU = one slab covering the grid.
struct Slab {
    int64_t z0, z1;
    int64_t plane;                         // vertices per plane of the slowest axis
    int64_t v0, v1;                        // owned global ids
};

// Field values visible to a slab: the owned planes plus the one-plane halo on
// each side that exists ("ghost vertices"), fetched from the
// neighbours.  Grids only; on one GPU lo = hi = null and own = the field.
struct FieldView {
    const float *own, *lo, *hi;
    int64_t v0, v1, plane;
#ifdef __CUDACC__
    __device__ __forceinline__ float at(int64_t g) const {
        if (g >= v0 && g < v1) return __ldg(own + (g - v0));
        if (g < v0) return __ldg(lo + (g - v0 + plane));
        return __ldg(hi + (g - v1));
    }
#endif
};

// Labels visible to a slab: the owned labels plus the (final) labels of the
// halo planes received in the boundary exchange.  CSR: own = every vertex.
struct LabelView {
    const int32_t *own;
    int64_t v0, v1;
    const int32_t *lo, *hi;                // halo planes z0 - 1 and z1 (grid, multi-slab) or null
    int64_t plane;
    // labels still being finalised concurrently: a label with bit 31 is an
    // exit pointer, followed to the final value (every value read lies on the
    // same ascending path, so stale reads are harmless); a pointer that leaves
    // the slab lands in a halo plane, whose values (lo / hi) are final
    bool chase;
#ifdef __CUDACC__
    __device__ __forceinline__ int32_t at(int64_t g) const {
        if (chase) {
            int64_t x = g;
            for (;;) {
                if (x < v0) return lo[x - v0 + plane];
                if (x >= v1) return hi[x - v1];
                const int32_t w = __ldca(own + (x - v0));
                if (w >= 0) return w;
                x = w & 0x7fffffff;
            }
        }
        if (g >= v0 && g < v1) return own[g - v0];
        if (g < v0) return lo[g - v0 + plane];
        return hi[g - v1];
    }
#endif
};

// --------------------------------------------------------------- kernels
// All launchers are asynchronous on `st` and return the launch error.

// S1 + S3, generic n: ptr[i] (global id) for owned i, saddle / maximum bits
// (bit i of word i/32), optional beta0+ per vertex.
// pad (optional, padded_cells floats): one slab classifies on a copy padded by
// a NaN cell on each side of every axis (no per-offset domain tests)
cudaError_t launch_classify_grid(const LinkTable &tab, int ndim, FieldView F, const Slab &s, int32_t *ptr,
                                 uint32_t *sad_bits, uint32_t *max_bits, uint8_t *beta_out, int *nan_flag,
                                 cudaStream_t st, float *pad = nullptr);
int64_t padded_cells(const LinkTable &tab, int ndim);
// CSR S1 + S3 in two warp-per-vertex passes, no degree cap (k_csr.cu).
// S1 over [v0, v1): ptr[v - v0] = gradient, max_bits (nullable) = maxima of the
// range, and the upper list of every v: upl[row_ptr[v] .. + nup[v]) (upl is
// int32[nnz], nup int32[N], both indexed globally).  S3 over [v0, v1) needs
// the upper lists of every neighbour of the range (run S1 over [0, N) first):
// sad_bits, beta0+ (nullable), the saddles' reps in rep_buf[row_ptr[v] ..]
// (nullable); par = int32[nnz] scratch for vertices with |U| > 64.
cudaError_t launch_csr_upper(const int64_t *row_ptr, const int32_t *col_idx, const float *f, int64_t v0, int64_t v1,
                             int32_t *ptr, uint32_t *max_bits, int32_t *upl, int32_t *nup, int *nan_flag,
                             cudaStream_t st);
cudaError_t launch_csr_link(const int64_t *row_ptr, const int32_t *col_idx, const float *f, int64_t v0, int64_t v1,
                            const int32_t *upl, const int32_t *nup, uint32_t *sad_bits, uint8_t *beta_out,
                            int32_t *rep_buf, int32_t *par, cudaStream_t st);
// EG_CHECK_CSR: *bad |= a nonzero code if the CSR is not a sorted, symmetric,
// loop-free adjacency with a valid row_ptr (k_csr.cu)
cudaError_t launch_check_csr(const int64_t *row_ptr, const int32_t *col_idx, int64_t n, int64_t nnz, int *bad,
                             cudaStream_t st);   // saddles' component reps at rep_buf[row_ptr[v] ..]

// S2: in-place pointer jumping over ptr[0..n) whose entries are global ids;
// entries outside [v0, v0 + n) are terminal (remote).  changed[r] is set when
// round r modified something; round r exits immediately if round r-1 did not.
cudaError_t launch_jump_round(int32_t *ptr, int64_t n, int64_t v0, int *changed, int round, cudaStream_t st);

// Compaction of a bitmap over owned indices [0, n) into ascending global ids
// (v0 + i) as int32 and int64.
size_t compact_scratch_bytes(int64_t n);
cudaError_t launch_compact_bits(const uint32_t *bits, int64_t n, int64_t v0, void *scratch, int32_t *out32,
                                int64_t *out64, int64_t *d_count, cudaStream_t st);
cudaError_t launch_count_bits(const uint32_t *bits, int64_t n, void *scratch, int64_t *d_count, cudaStream_t st);
cudaError_t launch_emit_counted(const uint32_t *bits, int64_t n, int64_t v0, const void *scratch, int32_t *out32,
                                int64_t *out64, cudaStream_t st);

// S4 for grids and CSR.
cudaError_t launch_saddle_beta_grid(const LinkTable &tab, int ndim, FieldView F, const int32_t *saddles,
                                    int64_t n_sad, int32_t *beta, cudaStream_t st);
// slot_off == null: fixed slots of link size K per saddle (no beta0+ pass
// needed first) and beta0+ written to beta_out
cudaError_t launch_arcs_grid(const LinkTable &tab, int ndim, FieldView F, const int32_t *saddles, int64_t n_sad,
                             const int64_t *slot_off, LabelView lv, int32_t *tmp_m, int32_t *tmp_mult,
                             int32_t *n_unique, int64_t *raw_s, int64_t *raw_rep, int64_t *raw_m, cudaStream_t st,
                             int32_t *beta_out = nullptr);
// link size 2 (2^n - 1): the fixed slot stride of launch_arcs_grid without slot_off
inline int grid_link_size(int ndim) { return 2 * ((1 << ndim) - 1); }
// beta0+ of the saddles from a per-vertex beta0+ array written by classify
cudaError_t launch_gather_beta(const uint8_t *beta8, int64_t v0, const int32_t *saddles, int64_t n, int32_t *out,
                               cudaStream_t st);
// S4 on CSR from the representatives classify stored in rep_buf
cudaError_t launch_arcs_csr_reps(const int64_t *row_ptr, const int32_t *rep_buf, const int32_t *saddles,
                                 const int32_t *sbeta, int64_t n_sad, const int64_t *slot_off, LabelView lv,
                                 int32_t *tmp_m, int32_t *tmp_mult, int32_t *n_unique, int64_t *raw_s,
                                 int64_t *raw_rep, int64_t *raw_m, cudaStream_t st);
// int64 -> int32 ids (EG_GRAPH32 host copies; every id < 2^31)
cudaError_t launch_narrow(const int64_t *in, int32_t *out, int64_t n, cudaStream_t st);
cudaError_t launch_emit_arcs(const int32_t *saddles, int64_t n_sad, const int64_t *slot_off, const int64_t *arc_off,
                             const int32_t *tmp_m, const int32_t *tmp_mult, const int32_t *n_unique,
                             int64_t *arc_s, int64_t *arc_m, int32_t *arc_mult, cudaStream_t st,
                             int slot_stride = 0);   // slot_off == null: saddle j's slots start at j * slot_stride

// exact conversion of an EG_DTYPE_* field to float32 (reading L21)
cudaError_t launch_to_f32(const void *in, int dtype, float *out, int64_t n, cudaStream_t st);
// float64 / (u)int32 / (u)int64 -> float32 cast; *inexact |= 1 if a value is not exactly a float32
cudaError_t launch_exact_f32(const void *in, int dtype, float *out, int64_t n, int *inexact, cudaStream_t st);
// SoS-rank image of a field (reading L22; F32 too): out[v] = the float with bit
// pattern rank(v) + 2^23 (reverse: N-1-rank(v), the reversed order of L11).
// scratch == null: *bytes = the scratch size.
constexpr int64_t kRankMaxN = 0x7F000000;
cudaError_t launch_rank_f32(const void *in, int dtype, float *out, int64_t n, void *scratch, size_t *bytes,
                            bool reverse, cudaStream_t st);
// minimum graph (reading L11): g[i] = -f[n-1-i]; in-place reversal of an id
// list (entries x -> N-1-x when map_ids) or of a plain array
cudaError_t launch_reflect_negate(const float *f, float *g, int64_t n, cudaStream_t st);
cudaError_t launch_reverse_i64(int64_t *a, int64_t n, int64_t N, bool map_ids, cudaStream_t st);
cudaError_t launch_reverse_i32(int32_t *a, int64_t n, int64_t N, bool map_ids, cudaStream_t st);

// arc bundling (reading L19) of one slab's graph: inputs, scratch
// (keys / keys2 / idx / idx2 / keep / arc_cnt of ns entries, s_pos / a_pos of
// ns + 1, sort and scan scratch) and outputs (the kept saddles and arcs; the
// counts are s_pos[ns] and a_pos[ns])
struct BundleArgs {
    int64_t ns;
    const int32_t *n_unique;
    const int64_t *arc_off, *arc_s, *arc_m;
    const int32_t *arc_mult;
    const int64_t *sad64;
    const int32_t *sad32, *sbeta;
    const float *f;
    int64_t f_base;                        // global id of f[0]
    uint64_t *keys, *keys2;
    int32_t *idx, *idx2, *keep, *arc_cnt;
    int64_t *s_pos, *a_pos;
    void *sort_tmp;
    size_t sort_bytes;
    void *scan_tmp;
    size_t scan_bytes;
    int64_t *o_sad64;
    int32_t *o_sad32, *o_sbeta, *o_nu;
    int64_t *o_arc_s, *o_arc_m;
    int32_t *o_arc_mult;
};
size_t bundle_sort_bytes(int64_t ns);
cudaError_t launch_bundle(const BundleArgs &B, cudaStream_t st);

// persistence-directed cancellation (simplify.cu): host-side, serial
struct SimplifyResult {
    std::vector<int64_t> maxima, saddles, arc_s, arc_m;
    std::vector<int32_t> saddle_beta, arc_mult;
};
void simplify_graph(int64_t n_max, const int64_t *maxima, const float *fmax, int64_t n_sad, const int64_t *saddles,
                    const int32_t *sbeta, const float *fsad, int64_t n_arc, const int64_t *arc_s,
                    const int64_t *arc_m, const int32_t *arc_mult, double tau, bool minimum, SimplifyResult &out);
cudaError_t launch_gather_f(const float *f, int64_t f_base, const int64_t *ids, int64_t n, float *out,
                            cudaStream_t st);

// arc geometry (integral lines of the raw arcs): off == null -> path lengths
// into len_or_out[j]; else the vertices at len_or_out[off[j] ..]
cudaError_t launch_arc_paths_grid(const LinkTable &tab, int ndim, FieldView F, const int64_t *raw_s,
                                  const int64_t *raw_rep, int64_t n_raw, const int64_t *off, int64_t *len_or_out,
                                  cudaStream_t st, int32_t *nxt = nullptr);
cudaError_t launch_arc_paths_csr(const int64_t *row_ptr, const int32_t *col_idx, const float *f, const int64_t *raw_s,
                                 const int64_t *raw_rep, int64_t n_raw, const int64_t *off, int64_t *len_or_out,
                                 cudaStream_t st, int32_t *nxt = nullptr);
// second pass of the arc geometry: follow the next steps the first pass left in nxt (index v - v0)
cudaError_t launch_arc_paths_follow(const int64_t *raw_s, const int64_t *raw_rep, int64_t n_raw, const int64_t *off,
                                    const int32_t *nxt, int64_t v0, int64_t *out, cudaStream_t st);
// exclusive scan of int64 counts into int64 offsets (offsets[n] = total)
size_t scan64_scratch_bytes(int64_t n);
cudaError_t launch_scan_i64(const int64_t *in, int64_t *out, int64_t n, void *scratch, size_t scratch_bytes,
                            cudaStream_t st);

// exclusive scan of int32 counts into int64 offsets (offsets[n] = total)
size_t scan_scratch_bytes(int64_t n);
cudaError_t launch_scan_i32(const int32_t *in, int64_t *out, int64_t n, void *scratch, size_t scratch_bytes,
                            cudaStream_t st);

// ------------------------------------------------ cross-slab label resolution
// (k_slab.cu; the paper's partial paths P:296 become "exit
// pointers" into the neighbours' boundary planes)
//
// Label convention inside a slab after the local phase: label >= 0 is final
// (a maximum); label = kUnresolved | x means "the path continues at x", where
// x is either an owned vertex whose own label is (locally) final-or-remote,
// or a vertex of a halo plane (remote).

// generic path: after local pointer jumping, mark remote targets unresolved
cudaError_t launch_flag_remote(int32_t *label, int64_t n, int64_t v0, cudaStream_t st);
// bval[0..plane) = resolved-as-far-as-possible values of plane z0, bval[plane..2 plane) of plane z1 - 1
cudaError_t launch_bval_init(const int32_t *label, const Slab &s, int32_t *bval, cudaStream_t st);
// one exchange round: bval entries pointing into a halo plane take the
// neighbour's value (hval lo = plane z0 - 1, hi = plane z1); counts unresolved
cudaError_t launch_bval_update(int32_t *bval, const int32_t *hval_lo, const int32_t *hval_hi, const Slab &s,
                               unsigned long long *unresolved, cudaStream_t st, const unsigned long long *prev = nullptr);
// final pass: every unresolved owned label (all owned vertices, or only those
// whose bit is set in `bits`) becomes final, via owned labels and the final
// halo-plane values
// the one-slab label pass in z-chunks (eg_compute_host pipeline, k_slab.cu):
// words [w_begin, w_end) of the owned labels, chains followed only through
// local indices < lim; unfinished vertices are appended to list (capacity
// list_cap, count *list_n) for launch_finalize_list, which finishes them once
// every vertex is labelled (or every label if the list overflowed)
cudaError_t launch_finalize_chunk(int32_t *label, int64_t w_begin, int64_t w_end, int64_t n, int64_t v0, int64_t lim,
                                  int32_t *list, unsigned long long *list_n, int64_t list_cap, cudaStream_t st,
                                  unsigned long long *hist = nullptr);
cudaError_t launch_finalize_list(int32_t *label, const int32_t *list, const unsigned long long *list_n,
                                 int64_t list_cap, int64_t v0, int64_t n_all, cudaStream_t st,
                                 unsigned long long *hist = nullptr);
cudaError_t launch_gather_labels(const int32_t *label, const int32_t *list, int64_t n, int32_t *out, cudaStream_t st);
cudaError_t launch_finalize(int32_t *label, const uint32_t *bits, int64_t v0, int64_t v1, cudaStream_t st,
                            unsigned long long *hist = nullptr);
// the label pass of one 3-D slab in up to three launches (z-face plane pairs,
// y-face row pairs, the rest; tiles of tz planes x ty rows from the slab's
// first plane).  passes: bit p runs pass p.  label / v0: the slab's labels and
// its first global id; chase targets may lie outside the slab (other slabs
// of the same label array, or halo planes holding final values)
cudaError_t launch_finalize_faces(int32_t *label, int64_t v0, int64_t nx, int64_t ny, int64_t planes, int tz, int ty,
                                  int ysplit, int passes, cudaStream_t st, unsigned long long *hist = nullptr);
}  // namespace eg
