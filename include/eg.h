/*
 * include/eg.h -- C ABI of the B200 extremum-graph library (libeg_b200.so).
 *
 * Computes, for a float32 scalar field on an n-D Freudenthal grid or on a
 * symmetric CSR neighbourhood graph, the data-parallel hot path of
 * arXiv 2303.02724 ("tachyon", /root/reference/PAPER.md, cited P:<line>):
 *
 *   S1 steepest-ascent pointer  gradient(v) = highest vertex of the upper link
 *                               (P:186), v itself for a maximum; ties broken by
 *                               simulated perturbation with the lower
 *                               global linear index lower (L1).
 *   S2 labels                   label[v] = the maximum reached by following the
 *                               gradient (Alg. 2), by pointer jumping.
 *   S3 saddles                  beta0+ = #components of the upper link
 *                               (Table 1); maximum iff beta0+ = 0,
 *                               (n-1)-saddle iff beta0+ >= 2.
 *   S4 arcs                     for every saddle s and every upper-link
 *                               component C: m = label[UpperLinkRep(C)];
 *                               unique (s, m) with multiplicity.
 *
 * Conventions (all entry points):
 *  - Every function returns eg_status and never aborts.  On failure the
 *    message is available from eg_last_error(ctx).  CUDA or NCCL failures are
 *    sticky: the ctx is poisoned and only eg_destroy / eg_last_error are valid.
 *  - Vertex ids are global linear indices, axis 0 fastest.
 *  - Device pointers are borrowed for the duration of the call; every output
 *    is owned by the ctx and valid until the next eg_compute* or eg_destroy.
 *  - There is no CPU fallback: without a CUDA device eg_create fails.
 */
#ifndef EG_H
#define EG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct eg_ctx eg_ctx;

typedef enum {
    EG_OK = 0,
    EG_ERR_INVALID_ARG = 1,   /* bad dims / pointers / CSR / slab tiling        */
    EG_ERR_NAN = 2,           /* NaN in the field (reading L2: NaN is rejected) */
    EG_ERR_OOM = 3,           /* device or pinned-host allocation failed        */
    EG_ERR_CUDA = 4,          /* CUDA runtime error (sticky)                     */
    EG_ERR_NCCL = 5,          /* NCCL error (sticky)                             */
    EG_ERR_STATE = 6,         /* call out of order (e.g. get_graph before compute) */
    EG_ERR_UNSUPPORTED = 7    /* e.g. N >= 2^31, a flag combination not built   */
} eg_status;

enum { EG_DOMAIN_GRID = 0, EG_DOMAIN_CSR = 1 };

/* Regular grid.  dims[0] is the fastest axis; 1 <= ndim <= 8
 * (n <= 3: the tiled kernels; n = 4..8: the generic n-D kernels).
 * slab_begin/slab_end: the planes of the slowest axis owned by this rank
 * (multi-GPU slab partition, "blocks ... along the z-axis");
 * [0, dims[ndim-1]) on one GPU.  d_field then holds ONLY the owned planes,
 * contiguous: (slab_end - slab_begin) * prod(dims[0..ndim-2]) floats. */
typedef struct {
    int32_t ndim;
    int64_t dims[8];
    int64_t slab_begin, slab_end;
} eg_grid;

/* Symmetric CSR graph without self loops, sorted neighbour lists (reading
 * L14: the link of v is the subgraph induced on N(v)).  Device pointers,
 * replicated on every rank.  [v_begin, v_end) = vertices owned by this rank;
 * d_field is the FULL field f[n_vertices] (links touch neighbours of
 * neighbours). */
typedef struct {
    int64_t n_vertices, nnz;
    const int64_t *row_ptr;   /* [n_vertices + 1], device */
    const int32_t *col_idx;   /* [nnz], device            */
    int64_t v_begin, v_end;
} eg_csr;

typedef struct {
    int32_t kind;             /* EG_DOMAIN_GRID or EG_DOMAIN_CSR */
    eg_grid grid;
    eg_csr csr;
} eg_domain;

/* The extremum graph: host pointers owned by the ctx.  Every array is
 * ascending: maxima by id, saddles by id, arcs by (saddle, maximum).  On a
 * multi-GPU ctx this is the whole graph, identical on every rank. */
typedef struct {
    int64_t n_max, n_saddle, n_arc;
    const int64_t *maxima;
    const int64_t *saddles;
    const int32_t *saddle_beta;     /* beta0+ >= 2 */
    const int64_t *arc_saddle;
    const int64_t *arc_max;
    const int32_t *arc_mult;        /* #upper-link components of s reaching m */
} eg_graph;

typedef struct {
    /* device time (us): classify = the per-vertex pass(es); jump = pointer-
     * jumping rounds (generic / CSR paths); boundary = cross-slab exchange
     * rounds; label = the tiled path's exit-pointer label pass; arcs, graph
     * (node lists, arcs and their host copies), total */
    double us_classify, us_jump, us_boundary, us_label, us_arcs, us_graph, us_total;
    int32_t jump_rounds;            /* pointer-jumping rounds (or exit-graph rounds) */
    int32_t boundary_rounds;        /* cross-partition label rounds              */
    int32_t kernel_launches;        /* kernels launched by the last eg_compute   */
    int32_t path;                   /* 0 generic n-D grid, 1 tiled 3-D grid, 2 CSR */
    int64_t n_vertices, n_raw_arcs, n_exit_targets;
    int64_t bytes_alg;              /* algorithmic HBM bytes   */
    double us_main;                 /* device time of the main per-vertex kernel(s) */
    int64_t bytes_main;             /* their algorithmic bytes */
    /* S2 statistics (the gradient walk).
     * tile_rounds: pointer-doubling rounds inside a tile (tiled path);
     * with EG_STATS also: n_exit = vertices whose ascending path leaves their
     * tile (tiled path); chase_hist[k] = vertices whose label pass followed k
     * exit pointers (k >= 15 in the last bin), chase_max the longest. */
    int32_t tile_rounds;
    int32_t chase_max;
    int64_t n_exit;
    int64_t chase_hist[16];
} eg_stats;

/* eg_compute flags */
enum {
    EG_CHECK_NAN = 1u,        /* fused NaN scan; without it NaN input is UB  */
    EG_RAW_ARCS = 2u,         /* also keep raw (s, rep, m) per component     */
    EG_CHECK_CSR = 4u,        /* validate CSR sortedness / symmetry           */
    EG_FORCE_GENERIC = 8u,    /* grid: use the generic n-D kernels even for n <= 3 */
    EG_NO_GRAPH_D2H = 16u,    /* leave the graph (and arc paths) in HBM: one process -> eg_get_graph*,
                                 eg_get_raw_arcs and eg_get_arc_paths copy it on the first request;
                                 several ranks -> eg_get_graph* fail (EG_ERR_STATE) */
    /* The MINIMUM graph instead ("computes both maximum and
     * minimum graph"; reading L11): minima, 1-saddles (beta0 of the lower link
     * >= 2) and the descending arcs / labels -- the maximum graph under the
     * reversed total order.  eg_graph's "maxima" then hold the minima, labels
     * the minimum each descending path reaches.  Grids by point reflection;
     * CSR graphs, and grids with EG_RAW_ARCS / EG_ARC_PATHS, by the field's
     * reversed SoS-rank image (reading L22; the whole vertex range,
     * N < 2^31 - 2^24).  One GPU, one slab (EG_ERR_UNSUPPORTED otherwise). */
    EG_MINIMUM = 32u,
    /* Arc geometry (Fig. 4): the integral line of
     * every raw arc -- s, rep, then steepest-ascent steps to m -- available
     * through eg_get_arc_paths.  Implies EG_RAW_ARCS.  One GPU, one slab. */
    EG_ARC_PATHS = 64u,
    /* Arc bundling (reading L19 in DESIGN.md): of the saddles whose
     * arcs reach exactly the same two maxima, only the highest (value, then
     * index) is kept in eg_graph -- for a minimum graph the lowest.  Raw arcs
     * and paths are not filtered.  One GPU, one slab. */
    EG_BUNDLE = 128u,
    /* keep f at every maximum and saddle (for eg_simplify); one process */
    EG_NODE_VALUES = 256u,
    /* collect the S2 statistics of eg_stats (exit counts, chase histogram);
     * costs a few instructions per vertex, so it is off in timed runs */
    EG_STATS = 1024u,
    /* copy the graph to the host as 32-bit ids (12 B per arc instead of 20;
     * N < 2^31 always holds): read it with eg_get_graph32; eg_get_graph then
     * widens it on the host on first use.  One process, plain maximum graph
     * (with EG_BUNDLE / EG_MINIMUM / EG_NODE_VALUES or several ranks the graph
     * is copied as 64-bit ids and eg_get_graph32 narrows it on the host). */
    EG_GRAPH32 = 2048u
};
/* virtual partitions: process a grid as k slabs on one GPU, exchanging
 * boundaries by device copies exactly as k ranks would (partition test). */
#define EG_VIRTUAL_PARTS(k) ((uint32_t)(k) << 16)   /* k < 65536; bits 16-31, no flag uses them */

/* Create a single-GPU context on `cuda_device`, launching on `cuda_stream`
 * (a cudaStream_t, NULL = the legacy default stream).  Fails with
 * EG_ERR_CUDA if no device is present (no CPU fallback). */
eg_status eg_create(eg_ctx **out, int cuda_device, void *cuda_stream);

/* Multi-GPU: every rank calls eg_create_dist with the same 128-byte NCCL
 * unique id (from eg_nccl_unique_id on rank 0, broadcast by the caller).
 * Collective.  Calls of eg_compute on such a ctx are collective too. */
eg_status eg_nccl_unique_id(void *out128);
eg_status eg_create_dist(eg_ctx **out, int cuda_device, void *cuda_stream, const void *nccl_id128,
                         int rank, int world);

/* Compute S1..S4 for a device-resident field.  Stream-ordered on the ctx
 * stream; returns after one final synchronisation with the graph copied to
 * host memory owned by the ctx (unless EG_NO_GRAPH_D2H: then it stays in
 * ctx-owned device memory until the next compute and, on one process, the
 * first eg_get_graph / eg_get_graph32 / eg_get_raw_arcs copies it). */
eg_status eg_compute(eg_ctx *ctx, const eg_domain *domain, const float *d_field, uint32_t flags);

/* Other input types (readings L21/L22 in DESIGN.md).
 * F16, BF16, (U)INT8, (U)INT16: every value is exactly a float32, so the field
 * is converted on the device (into a buffer owned by the ctx) and the same
 * path runs -- outputs are identical to eg_compute on the converted values.
 * F64, (U)INT32, (U)INT64: the field is replaced on the device by its SoS-rank
 * image (rank of each vertex under value-then-index order, a stable radix
 * sort); the extremum graph depends on the field only through that order
 * (P:142-151), so outputs are exactly those of the type's own order, with no
 * rounding.  Rank types need one GPU and a whole domain (world size 1,
 * N < 2^31 - 2^24), are EG_ERR_UNSUPPORTED with EG_NODE_VALUES (the values at
 * the nodes have no float32 image), and use 2 x (key + 4) bytes per vertex of
 * ctx-owned scratch.  NaN (F64) is EG_ERR_NAN as for F32.  d_field: device,
 * `dtype` elements in the eg_compute layout. */
enum { EG_DTYPE_F32 = 0, EG_DTYPE_F16 = 1, EG_DTYPE_BF16 = 2, EG_DTYPE_U8 = 3, EG_DTYPE_I8 = 4, EG_DTYPE_U16 = 5,
       EG_DTYPE_I16 = 6, EG_DTYPE_F64 = 7, EG_DTYPE_I32 = 8, EG_DTYPE_U32 = 9, EG_DTYPE_I64 = 10,
       EG_DTYPE_U64 = 11 };
eg_status eg_compute_typed(eg_ctx *ctx, const eg_domain *domain, const void *d_field, int dtype, uint32_t flags);

/* Same, end to end from HOST memory: copies h_field to the device (staged
 * through pinned memory owned by the ctx), computes, and -- if h_labels is not
 * NULL -- copies the owned labels back (int32, one per owned vertex). */
eg_status eg_compute_host(eg_ctx *ctx, const eg_domain *domain, const float *h_field, int32_t *h_labels,
                          uint32_t flags);

/* S1 + S3 only, per owned vertex, into caller device buffers:
 * d_ptr[i] = gradient of vertex (first owned + i) as a global id (int32),
 * d_beta[i] = beta0+ (saturated at 255).  Single GPU, any domain. */
eg_status eg_gradient(eg_ctx *ctx, const eg_domain *domain, const float *d_field, int32_t *d_ptr,
                      uint8_t *d_beta);

eg_status eg_get_graph(eg_ctx *ctx, eg_graph *out);

/* The same graph with 32-bit ids (see EG_GRAPH32); host pointers owned by the
 * ctx, valid until the next compute / destroy. */
typedef struct {
    int64_t n_max, n_saddle, n_arc;
    const int32_t *maxima;
    const int32_t *saddles;
    const int32_t *saddle_beta;
    const int32_t *arc_saddle;
    const int32_t *arc_max;
    const int32_t *arc_mult;
} eg_graph32;
eg_status eg_get_graph32(eg_ctx *ctx, eg_graph32 *out);
/* raw arcs (EG_RAW_ARCS): one (s, rep, m) per upper-link component, ordered by
 * (s, rep); host pointers owned by the ctx; this rank's saddles only. */
eg_status eg_get_raw_arcs(eg_ctx *ctx, int64_t *n, const int64_t **s, const int64_t **rep, const int64_t **m);
/* arc geometry (EG_ARC_PATHS): path j (one per raw arc, in eg_get_raw_arcs
 * order) is vertices[offsets[j] .. offsets[j+1]): the saddle, the component's
 * representative, then every gradient step to the maximum.  Host pointers
 * owned by the ctx, valid until the next compute / destroy. */
eg_status eg_get_arc_paths(eg_ctx *ctx, int64_t *n, const int64_t **offsets, const int64_t **vertices);
/* Persistence-directed cancellation (reading L20 in
 * DESIGN.md) of the last graph (which needs EG_NODE_VALUES): saddles are
 * cancelled in increasing cost (f(lower adjacent maximum) - f(s); the second
 * highest for a multi-saddle) with lazy updates while the cost is <= tau, each
 * merging its lower maxima into its highest.  Serial on the host, as in the
 * paper.  The result is returned in `out` (host pointers owned by the ctx,
 * valid until the next call); the unsimplified graph stays available through
 * eg_get_graph.  A minimum graph is simplified in the reversed order. */
eg_status eg_simplify(eg_ctx *ctx, double tau, eg_graph *out);
/* labels of the owned vertices: device pointer owned by the ctx, int32 global
 * ids of maxima (N < 2^31). */
eg_status eg_get_labels(eg_ctx *ctx, const int32_t **d_labels, int64_t *n);
eg_status eg_get_stats(eg_ctx *ctx, eg_stats *out);
eg_status eg_destroy(eg_ctx *ctx);
const char *eg_last_error(const eg_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* EG_H */
