// C ABI (include/eg.h) and the host-side orchestration of one eg_compute.
//
// Per slab (one GPU, or one virtual partition):
//   [halo exchange of f]  -> local labels (S1 + S3 + slab-local S2)
//   [boundary exchange rounds over the two boundary planes]  -> finalize S2
//   -> compaction of maxima / saddles -> beta0+ -> arcs (S4)
// then the per-slab graphs are concatenated (rank order = id order) on every
// rank.  The field stays resident in HBM; host <-> device crossings are the
// counts needed to size outputs and the final (small) graph.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "eg_impl.h"
#include "eg_tiled.h"

using namespace eg;

namespace {

struct DevBuf {
    void *p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes) {
        if (bytes <= cap) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        size_t want = std::max<size_t>(bytes, 256);
        cudaError_t e = cudaMalloc(&p, want);
        if (e == cudaSuccess) cap = want;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    template <class T>
    T *as() const { return static_cast<T *>(p); }
};

struct HostBuf {
    void *p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes) {
        if (bytes <= cap) return cudaSuccess;
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
        size_t want = std::max<size_t>(bytes, 256);
        cudaError_t e = cudaMallocHost(&p, want);
        if (e == cudaSuccess) cap = want;
        return e;
    }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
    }
    template <class T>
    T *as() const { return static_cast<T *>(p); }
};

// One slab of a grid (or one vertex range of a CSR graph).
struct SlabState {
    Slab s{};
    FieldView F{};
    int32_t *label = nullptr;          // owned labels (a view)
    DevBuf f_lo, f_hi;                 // halo planes of f received from the neighbours
    DevBuf sad_bits, max_bits;
    DevBuf beta8;                      // CSR: beta0+ per owned vertex (from classify)
    DevBuf rep_buf;                    // CSR: the saddles' component representatives, by row_ptr
    DevBuf bval, hval_lo, hval_hi;     // boundary-plane label values (own / neighbours')
    bool has_lo = false, has_hi = false;
    Tiled3D *tiled = nullptr;
    bool tiled_lists = false;          // maxima / saddles come from the tiled path's lists
    DevBuf maxima64, saddles32, saddles64, sbeta, slot_off, tmp_m, tmp_mult, n_unique, arc_off;
    DevBuf arc_s, arc_m, arc_mult, raw_s, raw_rep, raw_m;
    DevBuf maxima32, arc_s32, arc_m32;  // EG_GRAPH32 device copies
    int64_t n_max = 0, n_sad = 0, n_arc = 0, n_raw = 0;
    ~SlabState() {
        DevBuf *b[] = {&f_lo, &f_hi, &sad_bits, &max_bits, &beta8, &rep_buf, &bval, &hval_lo, &hval_hi, &maxima64,
                       &saddles32, &saddles64, &sbeta, &slot_off, &tmp_m, &tmp_mult, &n_unique, &arc_off, &arc_s,
                       &arc_m, &arc_mult, &raw_s, &raw_rep, &raw_m, &maxima32, &arc_s32, &arc_m32};
        for (DevBuf *x : b) x->release();
        tiled3d_destroy(tiled);
    }
};

}  // namespace

struct eg_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool poisoned = false;
    std::string err;
    int rank = 0, world = 1;
    ncclComm_t comm = nullptr;

    std::vector<SlabState *> slabs;
    DevBuf label_all;                  // labels of every slab of this process
    DevBuf csr_scratch;                // CSR: int32[2 nnz + N]: upper lists, union-find parents, |U| per vertex
    DevBuf fix_dev;                    // eg_compute_host pipeline: labels patched on the host
    DevBuf field;                      // eg_compute_host staging target
    DevBuf mirror;                     // EG_MINIMUM: g[i] = -f[N-1-i]
    DevBuf typed;                      // eg_compute_typed: the field converted to float32
    DevBuf padded;                     // generic n-D grids, one slab: NaN-padded copy of the field
    DevBuf rank_scratch;               // eg_compute_typed, rank types: sort keys / indices / cub scratch
    bool minimum = false;              // the current compute is a minimum graph
    bool min_reflect = false;          // ... by point reflection (ids mapped back afterwards)
    bool bundle = false;               // the current compute bundles arcs (EG_BUNDLE)
    DevBuf bund_scratch;               // arc bundling scratch (keys, indices, scans)
    DevBuf b_sad64, b_sad32, b_sbeta, b_nu, b_arc_s, b_arc_m, b_arc_mult;   // bundled outputs (swapped in)
    DevBuf flags;                      // [0] nan, [1] deg overflow, [2..] jump-changed per round
    DevBuf counts;                     // int64 / u64 counters
    DevBuf scratch;                    // compaction / scan scratch
    DevBuf tab;                        // LinkTable
    DevBuf gsend, grecv;               // multi-GPU graph gather
    LinkTable host_tab;
    bool tab_valid = false;

    HostBuf h_maxima, h_saddles, h_sbeta, h_arc_s, h_arc_m, h_arc_mult, h_raw_s, h_raw_rep, h_raw_m, h_counts;
    HostBuf h32_maxima, h32_saddles, h32_arc_s, h32_arc_m;   // EG_GRAPH32 (sbeta / mult are int32 anyway)
    bool g32 = false;                  // the graph on the host is in the h32_* buffers (+ h_sbeta, h_arc_mult)
    bool h64_valid = false, h32_valid = false;   // which id width of the host graph is materialised
    HostBuf h_stage;
    HostBuf h_path_off, h_path_v;      // EG_ARC_PATHS
    DevBuf path_nxt;                   // EG_ARC_PATHS: next step of every visited vertex (int32[N])
    int64_t n_path_v = 0;
    bool paths_on_host = false;
    HostBuf h_fmax, h_fsad;            // EG_NODE_VALUES: f at the maxima / saddles
    DevBuf d_fnode;
    bool node_values = false, last_minimum = false;
    SimplifyResult simp;               // eg_simplify's output
    DevBuf path_len, path_off, path_v;
    int64_t n_paths = 0;
    bool paths_valid = false;
    int64_t n_max = 0, n_sad = 0, n_arc = 0, n_raw = 0, n_own = 0;
    bool have_graph = false, have_labels = false, graph_on_host = false, raw_valid = false;
    bool graph_deferred = false, deferred_raw = false;   // EG_NO_GRAPH_D2H on one process: copied on request
    const int32_t *d_labels = nullptr;
    eg_stats stats{};
    cudaEvent_t ev[8] = {};
    cudaEvent_t ev_main[2] = {};       // around the main per-vertex kernel(s) of one slab
    cudaEvent_t ev_s2[6] = {};         // S2 phases: jump rounds [0,1), boundary rounds [2,3), label pass [4,5)
    bool s2_timed[3] = {false, false, false};
    DevBuf stat_buf;                   // EG_STATS: [0] exiting vertices, [1..16] chase histogram, [17] max
    // one GPU, one slab: the node lists go to the host on a copy stream while
    // the arcs are computed (ev_d2h[0]: lists ready, [1]: beta ready, [2]: copies done)
    cudaStream_t d2h = nullptr;
    cudaEvent_t ev_d2h[3] = {};
    // one slab on one GPU: the graph stage (lists, arcs, D2H) runs on `aux`
    // while the labels are finalised on `stream` (ev_tile: local phase done,
    // ev_graph: graph stage done); gstream = the stream of the graph stage
    cudaStream_t aux = nullptr, gstream = nullptr;
    cudaStream_t cst = nullptr;        // several GPUs: the f halo exchange beside the interior tiles
    cudaStream_t h2d = nullptr, ld2h = nullptr, fst = nullptr;   // eg_compute_host pipeline streams
    ChunkIO *io = nullptr;             // set by eg_compute_host for the duration of one call
    cudaEvent_t ev_halo[2] = {};
    int prio_lo = 0, prio_hi = 0;
    cudaEvent_t ev_tile = nullptr, ev_graph = nullptr;
    bool overlap = false;
    bool early_d2h = false;            // set per compute: the node-list copies are already queued
};

static eg_status set_err(eg_ctx *c, eg_status s, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    if (c) {
        c->err = buf;
        if (s == EG_ERR_CUDA || s == EG_ERR_NCCL) c->poisoned = true;
    }
    return s;
}

#define CK(expr)                                                                                       \
    do {                                                                                               \
        cudaError_t _e = (expr);                                                                       \
        if (_e != cudaSuccess) {                                                                       \
            if (_e == cudaErrorMemoryAllocation)                                                       \
                return set_err(c, EG_ERR_OOM, "%s: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, \
                               __LINE__);                                                              \
            return set_err(c, EG_ERR_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__,  \
                           __LINE__);                                                                  \
        }                                                                                              \
    } while (0)

#define NK(expr)                                                                                             \
    do {                                                                                                     \
        ncclResult_t _r = (expr);                                                                            \
        if (_r != ncclSuccess)                                                                               \
            return set_err(c, EG_ERR_NCCL, "%s: %s (%s:%d)", #expr, ncclGetErrorString(_r), __FILE__, __LINE__); \
    } while (0)

#define ST(expr)                         \
    do {                                 \
        eg_status _s = (expr);           \
        if (_s != EG_OK) return _s;      \
    } while (0)

// ------------------------------------------------------------- validation

struct Problem {
    bool grid;
    int ndim;
    int64_t dims[8];
    int64_t N;             // total vertices
    int64_t plane;         // grid: vertices per plane of the slowest axis
    int64_t D;             // grid: extent of the slowest axis
    int64_t z0, z1;        // grid: this rank's planes
    int64_t v0, v1;        // owned range (both kinds)
    int64_t nnz;
    const int64_t *row_ptr;
    const int32_t *col_idx;
};

static bool is_device_ptr(const void *p) {
    if (!p) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

static eg_status validate(eg_ctx *c, const eg_domain *d, const float *field, bool need_device, Problem *P) {
    if (!d) return set_err(c, EG_ERR_INVALID_ARG, "domain is NULL");
    std::memset(P, 0, sizeof(*P));
    if (d->kind == EG_DOMAIN_GRID) {
        const eg_grid &g = d->grid;
        if (g.ndim < 1 || g.ndim > 8) return set_err(c, EG_ERR_INVALID_ARG, "ndim %d not in [1, 8]", g.ndim);
        if (g.ndim > kMaxDim) return set_err(c, EG_ERR_UNSUPPORTED, "ndim %d > %d is not built", g.ndim, kMaxDim);
        int64_t N = 1;
        for (int i = 0; i < g.ndim; ++i) {
            if (g.dims[i] < 1) return set_err(c, EG_ERR_INVALID_ARG, "dims[%d] = %lld < 1", i, (long long)g.dims[i]);
            if (N > INT64_MAX / g.dims[i]) return set_err(c, EG_ERR_INVALID_ARG, "vertex count overflows int64");
            N *= g.dims[i];
        }
        if (N >= (int64_t(1) << 31))
            return set_err(c, EG_ERR_UNSUPPORTED, "N = %lld >= 2^31 (int32 labels)", (long long)N);
        const int64_t D = g.dims[g.ndim - 1];
        int64_t z0 = g.slab_begin, z1 = g.slab_end;
        if (c->world == 1 && z0 == 0 && z1 == 0) z1 = D;   // convenience: 0,0 = whole grid
        if (z0 < 0 || z1 > D || z0 >= z1)
            return set_err(c, EG_ERR_INVALID_ARG, "bad slab [%lld, %lld)", (long long)z0, (long long)z1);
        if (c->world == 1 && (z0 != 0 || z1 != D))
            return set_err(c, EG_ERR_INVALID_ARG, "single-GPU ctx needs the whole grid as its slab");
        P->grid = true;
        P->ndim = g.ndim;
        for (int i = 0; i < g.ndim; ++i) P->dims[i] = g.dims[i];
        P->N = N;
        P->D = D;
        P->plane = N / D;
        P->z0 = z0;
        P->z1 = z1;
        P->v0 = z0 * P->plane;
        P->v1 = z1 * P->plane;
    } else if (d->kind == EG_DOMAIN_CSR) {
        const eg_csr &g = d->csr;
        if (g.n_vertices < 0 || g.nnz < 0) return set_err(c, EG_ERR_INVALID_ARG, "negative CSR sizes");
        if (g.n_vertices >= (int64_t(1) << 31)) return set_err(c, EG_ERR_UNSUPPORTED, "N >= 2^31");
        int64_t v0 = g.v_begin, v1 = g.v_end;
        if (c->world == 1 && v0 == 0 && v1 == 0) v1 = g.n_vertices;
        if (v0 < 0 || v1 > g.n_vertices || v0 > v1) return set_err(c, EG_ERR_INVALID_ARG, "bad vertex range");
        if (c->world == 1 && (v0 != 0 || v1 != g.n_vertices))
            return set_err(c, EG_ERR_INVALID_ARG, "single-GPU ctx needs the whole vertex range");
        if (g.n_vertices > 0 && (!is_device_ptr(g.row_ptr) || (g.nnz > 0 && !is_device_ptr(g.col_idx))))
            return set_err(c, EG_ERR_INVALID_ARG, "row_ptr / col_idx must be device pointers");
        P->grid = false;
        P->N = g.n_vertices;
        P->v0 = v0;
        P->v1 = v1;
        P->nnz = g.nnz;
        P->row_ptr = g.row_ptr;
        P->col_idx = g.col_idx;
    } else {
        return set_err(c, EG_ERR_INVALID_ARG, "unknown domain kind %d", d->kind);
    }
    if (P->N > 0 && !field) return set_err(c, EG_ERR_INVALID_ARG, "field is NULL");
    if (P->N > 0 && need_device && !is_device_ptr(field))
        return set_err(c, EG_ERR_INVALID_ARG, "field must be a device pointer");
    return EG_OK;
}

static eg_status ensure_table(eg_ctx *c, const Problem &P) {
    bool same = c->tab_valid && c->host_tab.ndim == P.ndim;
    for (int i = 0; same && i < P.ndim; ++i) same = c->host_tab.dims[i] == P.dims[i];
    if (same) return EG_OK;
    c->host_tab = make_link_table(P.ndim, P.dims);
    CK(c->tab.ensure(sizeof(LinkTable)));
    CK(cudaMemcpyAsync(c->tab.p, &c->host_tab, sizeof(LinkTable), cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    c->tab_valid = true;
    return EG_OK;
}

static float ev_us(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    return ms > 0.f ? ms * 1000.f : 0.f;     // phases on two streams may overlap
}

static void set_slab_count(eg_ctx *c, size_t k) {
    while (c->slabs.size() > k) {
        delete c->slabs.back();
        c->slabs.pop_back();
    }
    while (c->slabs.size() < k) c->slabs.push_back(new SlabState());
}

// ------------------------------------------------------- NCCL transport

static eg_status nccl_allgather_i64(eg_ctx *c, const int64_t *h_in, int n, std::vector<int64_t> &h_out) {
    CK(c->counts.ensure(sizeof(int64_t) * 16 * (c->world + 1)));
    int64_t *d = c->counts.as<int64_t>();
    CK(cudaMemcpyAsync(d, h_in, sizeof(int64_t) * n, cudaMemcpyHostToDevice, c->stream));
    NK(ncclAllGather(d, d + 16, size_t(n), ncclInt64, c->comm, c->stream));
    h_out.assign(size_t(n) * c->world, 0);
    CK(cudaMemcpyAsync(h_out.data(), d + 16, sizeof(int64_t) * n * c->world, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return EG_OK;
}

// plane exchange with the neighbour ranks: send_lo (our first plane) goes to
// rank - 1 and arrives there as its recv_hi; send_hi to rank + 1 as recv_lo
static eg_status nccl_exchange(eg_ctx *c, const void *send_lo, const void *send_hi, void *recv_lo, void *recv_hi,
                               size_t count, ncclDataType_t dt, cudaStream_t st = nullptr) {
    if (!st) st = c->stream;
    NK(ncclGroupStart());
    if (c->rank > 0) {
        NK(ncclSend(send_lo, count, dt, c->rank - 1, c->comm, st));
        NK(ncclRecv(recv_lo, count, dt, c->rank - 1, c->comm, st));
    }
    if (c->rank < c->world - 1) {
        NK(ncclSend(send_hi, count, dt, c->rank + 1, c->comm, st));
        NK(ncclRecv(recv_hi, count, dt, c->rank + 1, c->comm, st));
    }
    NK(ncclGroupEnd());
    return EG_OK;
}

// ------------------------------------------------------------ grid stages

static eg_status generic_local(eg_ctx *c, const Problem &P, SlabState &S, bool multi, bool timed) {
    const int64_t n = S.s.v1 - S.s.v0;
    int *flags = c->flags.as<int>();
    // one slab: classify on a NaN-padded copy of the field when it costs at most
    // twice the field (every axis + 2; tuning knob EG_PAD=0 turns it off)
    float *pad = nullptr;
    const char *pv = std::getenv("EG_PAD");
    if (!multi && (!pv || std::atoi(pv) != 0)) {
        const int64_t pc = padded_cells(c->host_tab, P.ndim);
        if (pc < (int64_t(1) << 31) && pc <= 2 * n + 4096) {
            CK(c->padded.ensure(sizeof(float) * size_t(pc)));
            pad = c->padded.as<float>();
        }
    }
    if (timed) CK(cudaEventRecord(c->ev_main[0], c->stream));
    CK(launch_classify_grid(c->host_tab, P.ndim, S.F, S.s, S.label, S.sad_bits.as<uint32_t>(),
                            S.max_bits.as<uint32_t>(), nullptr, flags, c->stream, pad));
    if (timed) CK(cudaEventRecord(c->ev_main[1], c->stream));
    c->stats.kernel_launches += 1;
    // S2 inside the slab: rounds are launched in batches; a round whose
    // predecessor changed nothing exits at once, so only the flag read-back
    // costs a sync.
    int *changed = flags + 2;
    CK(cudaMemsetAsync(changed, 0, sizeof(int) * 64, c->stream));
    if (timed) {
        CK(cudaEventRecord(c->ev_s2[0], c->stream));
        c->s2_timed[0] = true;
    }
    int rounds = 0;
    const int kBatch = 3;   // bounded chains: one or two rounds usually finish
    int hflag[64];
    for (int r0 = 0; r0 < 60; r0 += kBatch) {
        const int r1 = std::min(60, r0 + kBatch);
        for (int r = r0; r < r1; ++r) {
            CK(launch_jump_round(S.label, n, S.s.v0, changed, r, c->stream));
            c->stats.kernel_launches += 1;
        }
        CK(cudaMemcpyAsync(hflag, changed, sizeof(int) * r1, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        int first_zero = -1;
        for (int r = 0; r < r1; ++r)
            if (hflag[r] == 0) {
                first_zero = r;
                break;
            }
        rounds = first_zero >= 0 ? first_zero + 1 : r1;
        if (first_zero >= 0) break;
    }
    c->stats.jump_rounds = std::max(c->stats.jump_rounds, rounds);
    if (timed) CK(cudaEventRecord(c->ev_s2[1], c->stream));
    if (multi) {
        CK(launch_flag_remote(S.label, n, S.s.v0, c->stream));
        c->stats.kernel_launches += 1;
    }
    return EG_OK;
}

static eg_status grid_graph(eg_ctx *c, const Problem &P, SlabState &S, bool raw, bool early) {
    const int64_t n = S.s.v1 - S.s.v0;
    int64_t *cnt = c->counts.as<int64_t>();
    CK(c->h_counts.ensure(sizeof(int64_t) * 8));
    int64_t *hc = c->h_counts.as<int64_t>();
    if (S.tiled && S.tiled_lists) {
        // the tile kernels appended the maxima / saddles to lists: sort them
        S.n_max = tiled3d_count(S.tiled, 0);
        S.n_sad = tiled3d_count(S.tiled, 1);
        CK(S.maxima64.ensure(sizeof(int64_t) * std::max<int64_t>(S.n_max, 1)));
        CK(S.saddles32.ensure(sizeof(int32_t) * std::max<int64_t>(S.n_sad, 1)));
        CK(S.saddles64.ensure(sizeof(int64_t) * std::max<int64_t>(S.n_sad, 1)));
        eg_status st = tiled3d_lists(S.tiled, S.maxima64.as<int64_t>(), S.saddles32.as<int32_t>(),
                                     S.saddles64.as<int64_t>(), c->gstream, &c->stats, &c->err);
        if (st != EG_OK) {
            if (st == EG_ERR_CUDA) c->poisoned = true;
            return st;
        }
    } else {
        // two scratch regions: the chunk offsets of each bitmap survive until emission
        const size_t half =
            (std::max(compact_scratch_bytes(std::max<int64_t>(n, 1)), size_t(1) << 16) + 255) / 256 * 256;
        CK(c->scratch.ensure(2 * half));
        char *scr_max = c->scratch.as<char>(), *scr_sad = c->scratch.as<char>() + half;
        CK(launch_count_bits(S.max_bits.as<uint32_t>(), n, scr_max, cnt + 0, c->gstream));
        CK(launch_count_bits(S.sad_bits.as<uint32_t>(), n, scr_sad, cnt + 1, c->gstream));
        c->stats.kernel_launches += 4;
        CK(cudaMemcpyAsync(hc, cnt, sizeof(int64_t) * 2, cudaMemcpyDeviceToHost, c->gstream));
        CK(cudaStreamSynchronize(c->gstream));
        S.n_max = hc[0];
        S.n_sad = hc[1];
        CK(S.maxima64.ensure(sizeof(int64_t) * std::max<int64_t>(S.n_max, 1)));
        CK(S.saddles32.ensure(sizeof(int32_t) * std::max<int64_t>(S.n_sad, 1)));
        CK(S.saddles64.ensure(sizeof(int64_t) * std::max<int64_t>(S.n_sad, 1)));
        CK(launch_emit_counted(S.max_bits.as<uint32_t>(), n, S.s.v0, scr_max, nullptr, S.maxima64.as<int64_t>(),
                               c->gstream));
        CK(launch_emit_counted(S.sad_bits.as<uint32_t>(), n, S.s.v0, scr_sad, S.saddles32.as<int32_t>(),
                               S.saddles64.as<int64_t>(), c->gstream));
        c->stats.kernel_launches += 2;
    }
    const int64_t ns = S.n_sad;
    CK(cudaEventRecord(c->ev[3], c->gstream));
    if (early) {
        // the node lists are final: copy them while the arcs are computed
        CK(c->h_maxima.ensure(sizeof(int64_t) * std::max<int64_t>(S.n_max, 1)));
        CK(c->h_saddles.ensure(sizeof(int64_t) * std::max<int64_t>(ns, 1)));
        CK(c->h_sbeta.ensure(sizeof(int32_t) * std::max<int64_t>(ns, 1)));
        CK(cudaEventRecord(c->ev_d2h[0], c->gstream));
        CK(cudaStreamWaitEvent(c->d2h, c->ev_d2h[0], 0));
        if (c->g32) {
            CK(c->h32_maxima.ensure(sizeof(int32_t) * std::max<int64_t>(S.n_max, 1)));
            CK(c->h32_saddles.ensure(sizeof(int32_t) * std::max<int64_t>(ns, 1)));
            CK(S.maxima32.ensure(sizeof(int32_t) * std::max<int64_t>(S.n_max, 1)));
            CK(launch_narrow(S.maxima64.as<int64_t>(), S.maxima32.as<int32_t>(), S.n_max, c->d2h));
            if (S.n_max)
                CK(cudaMemcpyAsync(c->h32_maxima.p, S.maxima32.p, sizeof(int32_t) * S.n_max, cudaMemcpyDeviceToHost,
                                   c->d2h));
            if (ns)
                CK(cudaMemcpyAsync(c->h32_saddles.p, S.saddles32.p, sizeof(int32_t) * ns, cudaMemcpyDeviceToHost,
                                   c->d2h));
        } else {
            if (S.n_max)
                CK(cudaMemcpyAsync(c->h_maxima.p, S.maxima64.p, sizeof(int64_t) * S.n_max, cudaMemcpyDeviceToHost,
                                   c->d2h));
            if (ns)
                CK(cudaMemcpyAsync(c->h_saddles.p, S.saddles64.p, sizeof(int64_t) * ns, cudaMemcpyDeviceToHost,
                                   c->d2h));
        }
    }

    // beta0+ per saddle and slot offsets (sum beta0+ = raw arcs)
    CK(S.sbeta.ensure(sizeof(int32_t) * std::max<int64_t>(ns, 1)));
    CK(S.slot_off.ensure(sizeof(int64_t) * (ns + 1)));
    CK(S.arc_off.ensure(sizeof(int64_t) * (ns + 1)));
    CK(S.n_unique.ensure(sizeof(int32_t) * std::max<int64_t>(ns, 1)));
    const size_t sb = scan_scratch_bytes(std::max<int64_t>(ns, 1));
    CK(c->scratch.ensure(sb));
    LabelView lv{};
    if (P.grid) {
        lv.own = S.label;
        lv.v0 = S.s.v0;
        lv.v1 = S.s.v1;
        lv.lo = S.has_lo ? S.hval_lo.as<int32_t>() : nullptr;
        lv.hi = S.has_hi ? S.hval_hi.as<int32_t>() : nullptr;
        lv.plane = S.s.plane;
        lv.chase = c->overlap;
    } else {
        lv.own = c->label_all.as<int32_t>();     // CSR: labels of every vertex
        lv.v0 = 0;
        lv.v1 = P.N;
    }
    // grids without raw arcs: one pass computes beta0+ and the arcs into fixed
    // slots of link size per saddle (no beta0+ pass, scan or sync before it)
    const bool fused = P.grid && !raw;
    const int stride = fused ? grid_link_size(P.ndim) : 0;
    if (fused) {
        S.n_raw = 0;
        CK(S.tmp_m.ensure(sizeof(int32_t) * std::max<int64_t>(ns * stride, 1)));
        CK(S.tmp_mult.ensure(sizeof(int32_t) * std::max<int64_t>(ns * stride, 1)));
        CK(launch_arcs_grid(c->host_tab, P.ndim, S.F, S.saddles32.as<int32_t>(), ns, nullptr, lv,
                            S.tmp_m.as<int32_t>(), S.tmp_mult.as<int32_t>(), S.n_unique.as<int32_t>(), nullptr,
                            nullptr, nullptr, c->gstream, S.sbeta.as<int32_t>()));
        c->stats.kernel_launches += 1;
        if (early) {
            CK(cudaEventRecord(c->ev_d2h[1], c->gstream));
            CK(cudaStreamWaitEvent(c->d2h, c->ev_d2h[1], 0));
            if (ns)
                CK(cudaMemcpyAsync(c->h_sbeta.p, S.sbeta.p, sizeof(int32_t) * ns, cudaMemcpyDeviceToHost, c->d2h));
        }
    } else {
        if (P.grid)
            CK(launch_saddle_beta_grid(c->host_tab, P.ndim, S.F, S.saddles32.as<int32_t>(), ns,
                                       S.sbeta.as<int32_t>(), c->gstream));
        else
            CK(launch_gather_beta(S.beta8.as<uint8_t>(), S.s.v0, S.saddles32.as<int32_t>(), ns,
                                  S.sbeta.as<int32_t>(), c->gstream));
        CK(launch_scan_i32(S.sbeta.as<int32_t>(), S.slot_off.as<int64_t>(), ns, c->scratch.p, sb, c->gstream));
        c->stats.kernel_launches += 2;
        CK(cudaMemcpyAsync(hc, S.slot_off.as<int64_t>() + ns, sizeof(int64_t), cudaMemcpyDeviceToHost, c->gstream));
        CK(cudaStreamSynchronize(c->gstream));
        if (early && ns)   // beta0+ is final (the stream was just synchronised)
            CK(cudaMemcpyAsync(c->h_sbeta.p, S.sbeta.p, sizeof(int32_t) * ns, cudaMemcpyDeviceToHost, c->d2h));
        const int64_t nraw = hc[0];
        S.n_raw = nraw;
        CK(S.tmp_m.ensure(sizeof(int32_t) * std::max<int64_t>(nraw, 1)));
        CK(S.tmp_mult.ensure(sizeof(int32_t) * std::max<int64_t>(nraw, 1)));
        if (raw) {
            CK(S.raw_s.ensure(sizeof(int64_t) * std::max<int64_t>(nraw, 1)));
            CK(S.raw_rep.ensure(sizeof(int64_t) * std::max<int64_t>(nraw, 1)));
            CK(S.raw_m.ensure(sizeof(int64_t) * std::max<int64_t>(nraw, 1)));
        }
        if (P.grid)
            CK(launch_arcs_grid(c->host_tab, P.ndim, S.F, S.saddles32.as<int32_t>(), ns,
                                S.slot_off.as<int64_t>(), lv, S.tmp_m.as<int32_t>(), S.tmp_mult.as<int32_t>(),
                                S.n_unique.as<int32_t>(), raw ? S.raw_s.as<int64_t>() : nullptr,
                                raw ? S.raw_rep.as<int64_t>() : nullptr, raw ? S.raw_m.as<int64_t>() : nullptr,
                                c->gstream));
        else   // the representatives were stored by classify: no second link computation
            CK(launch_arcs_csr_reps(P.row_ptr, S.rep_buf.as<int32_t>(), S.saddles32.as<int32_t>(),
                                    S.sbeta.as<int32_t>(), ns, S.slot_off.as<int64_t>(), lv, S.tmp_m.as<int32_t>(),
                                    S.tmp_mult.as<int32_t>(), S.n_unique.as<int32_t>(),
                                    raw ? S.raw_s.as<int64_t>() : nullptr, raw ? S.raw_rep.as<int64_t>() : nullptr,
                                    raw ? S.raw_m.as<int64_t>() : nullptr, c->gstream));
        c->stats.kernel_launches += 1;
    }
    CK(launch_scan_i32(S.n_unique.as<int32_t>(), S.arc_off.as<int64_t>(), ns, c->scratch.p, sb, c->gstream));
    c->stats.kernel_launches += 2;
    CK(cudaMemcpyAsync(hc, S.arc_off.as<int64_t>() + ns, sizeof(int64_t), cudaMemcpyDeviceToHost, c->gstream));
    CK(cudaStreamSynchronize(c->gstream));
    S.n_arc = hc[0];
    CK(S.arc_s.ensure(sizeof(int64_t) * std::max<int64_t>(S.n_arc, 1)));
    CK(S.arc_m.ensure(sizeof(int64_t) * std::max<int64_t>(S.n_arc, 1)));
    CK(S.arc_mult.ensure(sizeof(int32_t) * std::max<int64_t>(S.n_arc, 1)));
    CK(launch_emit_arcs(S.saddles32.as<int32_t>(), ns, fused ? nullptr : S.slot_off.as<int64_t>(), S.arc_off.as<int64_t>(),
                        S.tmp_m.as<int32_t>(), S.tmp_mult.as<int32_t>(), S.n_unique.as<int32_t>(),
                        S.arc_s.as<int64_t>(), S.arc_m.as<int64_t>(), S.arc_mult.as<int32_t>(), c->gstream, stride));
    c->stats.kernel_launches += 1;
    return EG_OK;
}

static eg_status fail_if_flags(eg_ctx *c) {
    int h[2] = {0, 0};
    CK(cudaMemcpyAsync(h, c->flags.p, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (c->world > 1) {
        int64_t mine[2] = {h[0], h[1]};
        std::vector<int64_t> all;
        ST(nccl_allgather_i64(c, mine, 2, all));
        for (int r = 0; r < c->world; ++r) {
            h[0] |= int(all[2 * r]);
            h[1] |= int(all[2 * r + 1]);
        }
    }
    if (h[0]) return set_err(c, EG_ERR_NAN, "NaN in the scalar field (reading L2)");
    if (h[1]) return set_err(c, EG_ERR_INVALID_ARG, "CSR check failed (code %d: 1 row_ptr, 2 col_idx range, "
                             "4 unsorted / duplicate, 8 self loop, 16 asymmetric)", h[1]);
    return EG_OK;
}

// copy every slab's graph to the host (rank order = id order); multi-GPU:
// all-gather so that every rank holds the whole graph
static eg_status gather_graph(eg_ctx *c, bool raw) {
    int64_t nm = 0, ns = 0, na = 0, nr = 0;
    for (SlabState *S : c->slabs) {
        nm += S->n_max;
        ns += S->n_sad;
        na += S->n_arc;
        nr += S->n_raw;
    }
    std::vector<int64_t> all;
    int64_t mx[3] = {0, 0, 0};
    if (c->world > 1) {
        int64_t mine[3] = {nm, ns, na};
        ST(nccl_allgather_i64(c, mine, 3, all));
        nm = ns = na = 0;
        for (int r = 0; r < c->world; ++r) {
            nm += all[3 * r];
            ns += all[3 * r + 1];
            na += all[3 * r + 2];
            for (int k = 0; k < 3; ++k) mx[k] = std::max(mx[k], all[3 * r + k]);
        }
    }
    CK(c->h_maxima.ensure(sizeof(int64_t) * std::max<int64_t>(nm, 1)));
    CK(c->h_saddles.ensure(sizeof(int64_t) * std::max<int64_t>(ns, 1)));
    CK(c->h_sbeta.ensure(sizeof(int32_t) * std::max<int64_t>(ns, 1)));
    CK(c->h_arc_s.ensure(sizeof(int64_t) * std::max<int64_t>(na, 1)));
    CK(c->h_arc_m.ensure(sizeof(int64_t) * std::max<int64_t>(na, 1)));
    CK(c->h_arc_mult.ensure(sizeof(int32_t) * std::max<int64_t>(na, 1)));
    cudaStream_t st = c->gstream;
    if (c->world == 1 && c->g32) {
        // 32-bit ids: 4 B per maximum, 8 B per saddle, 12 B per arc
        CK(c->h32_maxima.ensure(sizeof(int32_t) * std::max<int64_t>(nm, 1)));
        CK(c->h32_saddles.ensure(sizeof(int32_t) * std::max<int64_t>(ns, 1)));
        CK(c->h32_arc_s.ensure(sizeof(int32_t) * std::max<int64_t>(na, 1)));
        CK(c->h32_arc_m.ensure(sizeof(int32_t) * std::max<int64_t>(na, 1)));
        int64_t om = 0, os = 0, oa = 0;
        for (SlabState *S : c->slabs) {
            if (S->n_max && !c->early_d2h) {
                CK(S->maxima32.ensure(sizeof(int32_t) * S->n_max));
                CK(launch_narrow(S->maxima64.as<int64_t>(), S->maxima32.as<int32_t>(), S->n_max, st));
                CK(cudaMemcpyAsync(c->h32_maxima.as<int32_t>() + om, S->maxima32.p, sizeof(int32_t) * S->n_max,
                                   cudaMemcpyDeviceToHost, st));
            }
            if (S->n_sad && !c->early_d2h) {
                CK(cudaMemcpyAsync(c->h32_saddles.as<int32_t>() + os, S->saddles32.p, sizeof(int32_t) * S->n_sad,
                                   cudaMemcpyDeviceToHost, st));
                CK(cudaMemcpyAsync(c->h_sbeta.as<int32_t>() + os, S->sbeta.p, sizeof(int32_t) * S->n_sad,
                                   cudaMemcpyDeviceToHost, st));
            }
            if (S->n_arc) {
                CK(S->arc_s32.ensure(sizeof(int32_t) * S->n_arc));
                CK(S->arc_m32.ensure(sizeof(int32_t) * S->n_arc));
                CK(launch_narrow(S->arc_s.as<int64_t>(), S->arc_s32.as<int32_t>(), S->n_arc, st));
                CK(launch_narrow(S->arc_m.as<int64_t>(), S->arc_m32.as<int32_t>(), S->n_arc, st));
                CK(cudaMemcpyAsync(c->h32_arc_s.as<int32_t>() + oa, S->arc_s32.p, sizeof(int32_t) * S->n_arc,
                                   cudaMemcpyDeviceToHost, st));
                CK(cudaMemcpyAsync(c->h32_arc_m.as<int32_t>() + oa, S->arc_m32.p, sizeof(int32_t) * S->n_arc,
                                   cudaMemcpyDeviceToHost, st));
                CK(cudaMemcpyAsync(c->h_arc_mult.as<int32_t>() + oa, S->arc_mult.p, sizeof(int32_t) * S->n_arc,
                                   cudaMemcpyDeviceToHost, st));
            }
            om += S->n_max;
            os += S->n_sad;
            oa += S->n_arc;
        }
        if (c->early_d2h) CK(cudaStreamWaitEvent(st, c->ev_d2h[2], 0));   // the node lists' copies
    } else if (c->world == 1) {
        int64_t om = 0, os = 0, oa = 0;
        for (SlabState *S : c->slabs) {
            if (S->n_max && !c->early_d2h)
                CK(cudaMemcpyAsync(c->h_maxima.as<int64_t>() + om, S->maxima64.p, sizeof(int64_t) * S->n_max,
                                   cudaMemcpyDeviceToHost, st));
            if (S->n_sad && !c->early_d2h) {
                CK(cudaMemcpyAsync(c->h_saddles.as<int64_t>() + os, S->saddles64.p, sizeof(int64_t) * S->n_sad,
                                   cudaMemcpyDeviceToHost, st));
                CK(cudaMemcpyAsync(c->h_sbeta.as<int32_t>() + os, S->sbeta.p, sizeof(int32_t) * S->n_sad,
                                   cudaMemcpyDeviceToHost, st));
            }
            if (S->n_arc) {
                CK(cudaMemcpyAsync(c->h_arc_s.as<int64_t>() + oa, S->arc_s.p, sizeof(int64_t) * S->n_arc,
                                   cudaMemcpyDeviceToHost, st));
                CK(cudaMemcpyAsync(c->h_arc_m.as<int64_t>() + oa, S->arc_m.p, sizeof(int64_t) * S->n_arc,
                                   cudaMemcpyDeviceToHost, st));
                CK(cudaMemcpyAsync(c->h_arc_mult.as<int32_t>() + oa, S->arc_mult.p, sizeof(int32_t) * S->n_arc,
                                   cudaMemcpyDeviceToHost, st));
            }
            om += S->n_max;
            os += S->n_sad;
            oa += S->n_arc;
        }
        if (c->early_d2h) CK(cudaStreamWaitEvent(st, c->ev_d2h[2], 0));   // the node lists' copies
    } else {
        // padded all-gather of 6 arrays through one staging buffer, 8-byte slots
        SlabState &S = *c->slabs[0];
        const int W = c->world;
        const int64_t m3[6] = {mx[0], mx[1], mx[1], mx[2], mx[2], mx[2]};
        const int64_t mine[6] = {S.n_max, S.n_sad, S.n_sad, S.n_arc, S.n_arc, S.n_arc};
        const void *src[6] = {S.maxima64.p, S.saddles64.p, S.sbeta.p, S.arc_s.p, S.arc_m.p, S.arc_mult.p};
        const size_t esz[6] = {8, 8, 4, 8, 8, 4};
        void *dst[6] = {c->h_maxima.p, c->h_saddles.p, c->h_sbeta.p, c->h_arc_s.p, c->h_arc_m.p, c->h_arc_mult.p};
        for (int a = 0; a < 6; ++a) {
            const size_t slot = size_t(std::max<int64_t>(m3[a], 1)) * esz[a];
            CK(c->gsend.ensure(slot));
            CK(c->grecv.ensure(slot * W));
            if (mine[a]) CK(cudaMemcpyAsync(c->gsend.p, src[a], mine[a] * esz[a], cudaMemcpyDeviceToDevice, st));
            NK(ncclAllGather(c->gsend.p, c->grecv.p, slot, ncclUint8, c->comm, st));
            int64_t off = 0;
            for (int r = 0; r < W; ++r) {
                const int64_t cnt = (a == 0) ? all[3 * r] : (a < 3 ? all[3 * r + 1] : all[3 * r + 2]);
                if (cnt)
                    CK(cudaMemcpyAsync(static_cast<char *>(dst[a]) + off * esz[a], c->grecv.as<char>() + r * slot,
                                       cnt * esz[a], cudaMemcpyDeviceToHost, st));
                off += cnt;
            }
        }
    }
    if (raw) {
        CK(c->h_raw_s.ensure(sizeof(int64_t) * std::max<int64_t>(nr, 1)));
        CK(c->h_raw_rep.ensure(sizeof(int64_t) * std::max<int64_t>(nr, 1)));
        CK(c->h_raw_m.ensure(sizeof(int64_t) * std::max<int64_t>(nr, 1)));
        int64_t o = 0;
        for (SlabState *S : c->slabs) {
            if (S->n_raw) {
                CK(cudaMemcpyAsync(c->h_raw_s.as<int64_t>() + o, S->raw_s.p, 8 * S->n_raw, cudaMemcpyDeviceToHost, st));
                CK(cudaMemcpyAsync(c->h_raw_rep.as<int64_t>() + o, S->raw_rep.p, 8 * S->n_raw, cudaMemcpyDeviceToHost,
                                   st));
                CK(cudaMemcpyAsync(c->h_raw_m.as<int64_t>() + o, S->raw_m.p, 8 * S->n_raw, cudaMemcpyDeviceToHost, st));
            }
            o += S->n_raw;
        }
    }
    c->n_max = nm;
    c->n_sad = ns;
    c->n_arc = na;
    c->n_raw = nr;
    return EG_OK;
}

// the boundary exchange: rounds of neighbour plane exchange and
// jumping until no boundary value of any slab is unresolved.  Rounds are
// queued in batches of kBatch with one host check per batch (paths cross a
// slab boundary only a few times: SURVEY 8(e) measured <= 4); a round whose
// predecessor left nothing unresolved returns at once on the device.
static eg_status boundary_rounds(eg_ctx *c, int *rounds_out) {
    auto &slabs = c->slabs;
    const size_t K = slabs.size();
    constexpr int kBatch = 4;
    unsigned long long *d_unres = reinterpret_cast<unsigned long long *>(c->counts.as<int64_t>() + 8);   // [kBatch]
    for (SlabState *S : slabs) {
        CK(launch_bval_init(S->label, S->s, S->bval.as<int32_t>(), c->stream));
        c->stats.kernel_launches += 1;
    }
    const int64_t plane = slabs[0]->s.plane;
    auto exchange = [&]() -> eg_status {
        // hval_lo of slab k = bval_hi of slab k-1; hval_hi = bval_lo of slab k+1
        if (c->world > 1) {
            SlabState &S = *slabs[0];
            ST(nccl_exchange(c, S.bval.as<int32_t>(), S.bval.as<int32_t>() + plane, S.hval_lo.as<int32_t>(),
                             S.hval_hi.as<int32_t>(), size_t(plane), ncclInt32));
        } else {
            for (size_t k = 0; k < K; ++k) {
                if (k > 0)
                    CK(cudaMemcpyAsync(slabs[k]->hval_lo.p, slabs[k - 1]->bval.as<int32_t>() + plane, 4 * plane,
                                       cudaMemcpyDeviceToDevice, c->stream));
                if (k + 1 < K)
                    CK(cudaMemcpyAsync(slabs[k]->hval_hi.p, slabs[k + 1]->bval.as<int32_t>(), 4 * plane,
                                       cudaMemcpyDeviceToDevice, c->stream));
            }
        }
        return EG_OK;
    };
    int rounds = 0;
    for (int batch = 0;; ++batch) {
        if (batch * kBatch > 4096) return set_err(c, EG_ERR_STATE, "boundary exchange did not converge");
        CK(cudaMemsetAsync(d_unres, 0, sizeof(unsigned long long) * kBatch, c->stream));
        for (int r = 0; r < kBatch; ++r) {
            ST(exchange());
            for (SlabState *S : slabs) {
                CK(launch_bval_update(S->bval.as<int32_t>(), S->has_lo ? S->hval_lo.as<int32_t>() : nullptr,
                                      S->has_hi ? S->hval_hi.as<int32_t>() : nullptr, S->s, d_unres + r, c->stream,
                                      r > 0 ? d_unres + r - 1 : nullptr));
                c->stats.kernel_launches += 1;
            }
            if (c->world > 1) NK(ncclAllReduce(d_unres + r, d_unres + r, 1, ncclUint64, ncclSum, c->comm, c->stream));
        }
        unsigned long long u[kBatch];
        CK(cudaMemcpyAsync(u, d_unres, sizeof(u), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        int done = -1;
        for (int r = 0; r < kBatch; ++r)
            if (u[r] == 0) {
                done = r;
                break;
            }
        if (done >= 0) {
            rounds += done + 1;
            break;
        }
        rounds += kBatch;
    }
    // one more exchange: the halo values are now the neighbours' final values
    ST(exchange());
    *rounds_out = rounds;
    return EG_OK;
}

static eg_status compute_grid(eg_ctx *c, const Problem &P, const float *f, uint32_t flags) {
    const int vparts = int((flags >> 16) & 0xffff);
    // ---- plan the slabs of this process
    std::vector<std::pair<int64_t, int64_t>> plan;
    if (c->world > 1) {
        plan.push_back({P.z0, P.z1});
        int64_t mine[2] = {P.z0, P.z1};
        std::vector<int64_t> all;
        ST(nccl_allgather_i64(c, mine, 2, all));
        for (int r = 0; r < c->world; ++r) {
            const int64_t a = all[2 * r], b = all[2 * r + 1];
            const int64_t prev = r ? all[2 * r - 1] : 0;
            if (a != prev || b - a < 2 || (r == c->world - 1 && b != P.D))
                return set_err(c, EG_ERR_INVALID_ARG, "slabs must tile the slowest axis in rank order, >= 2 planes each");
        }
    } else if (vparts > 1) {
        if (P.D < 2 * vparts) return set_err(c, EG_ERR_INVALID_ARG, "%d virtual slabs need >= %d planes", vparts, 2 * vparts);
        for (int k = 0; k < vparts; ++k) plan.push_back({P.D * k / vparts, P.D * (k + 1) / vparts});
    } else {
        plan.push_back({0, P.D});
    }
    const bool multi = plan.size() > 1 || c->world > 1;
    const bool tiled = P.ndim <= 3 && !(flags & EG_FORCE_GENERIC) && (!multi || P.ndim == 3);
    set_slab_count(c, plan.size());
    // labels: one array for every slab of this process (a view per slab)
    const int64_t nlab = (c->world > 1) ? P.v1 - P.v0 : P.N;
    // several GPUs: one halo plane of labels below and above the owned ones,
    // filled with the neighbours' final boundary values before the label pass
    const int64_t hpad = (c->world > 1) ? P.plane : 0;
    CK(c->label_all.ensure(sizeof(int32_t) * std::max<int64_t>(nlab + 2 * hpad, 1)));
    const int64_t base_v = (c->world > 1) ? P.v0 : 0;
    for (size_t k = 0; k < plan.size(); ++k) {
        SlabState &S = *c->slabs[k];
        S.s.z0 = plan[k].first;
        S.s.z1 = plan[k].second;
        S.s.plane = P.plane;
        S.s.v0 = S.s.z0 * P.plane;
        S.s.v1 = S.s.z1 * P.plane;
        const int64_t n = S.s.v1 - S.s.v0, words = (n + 31) / 32;
        S.label = c->label_all.as<int32_t>() + hpad + (S.s.v0 - base_v);
        S.F.own = f + (S.s.v0 - base_v);     // f holds the whole grid (single / virtual) or the owned planes
        S.F.v0 = S.s.v0;
        S.F.v1 = S.s.v1;
        S.F.plane = P.plane;
        S.has_lo = multi && S.s.z0 > 0;
        S.has_hi = multi && S.s.z1 < P.D;
        if (!tiled) {
            CK(S.sad_bits.ensure(sizeof(uint32_t) * std::max<int64_t>(words, 1)));
            CK(S.max_bits.ensure(sizeof(uint32_t) * std::max<int64_t>(words, 1)));
        }
        if (tiled && !S.tiled) S.tiled = tiled3d_create();
        S.tiled_lists = tiled;
        if (multi) {
            CK(S.f_lo.ensure(sizeof(float) * P.plane));
            CK(S.f_hi.ensure(sizeof(float) * P.plane));
            CK(S.bval.ensure(sizeof(int32_t) * 2 * P.plane));
            CK(S.hval_lo.ensure(sizeof(int32_t) * P.plane));
            CK(S.hval_hi.ensure(sizeof(int32_t) * P.plane));
        }
        S.F.lo = S.has_lo ? S.f_lo.as<float>() : nullptr;
        S.F.hi = S.has_hi ? S.f_hi.as<float>() : nullptr;
    }
    ST(ensure_table(c, P));
    CK(cudaEventRecord(c->ev[0], c->stream));

    // ---- halo planes of f (P:281 ghost vertices).  Several GPUs, tiled: on
    // the comm stream, overlapped with the interior tiles (halo_ev)
    cudaEvent_t halo_ev = nullptr;
    if (multi) {
        if (c->world > 1) {
            SlabState &S = *c->slabs[0];
            const int64_t np = S.s.z1 - S.s.z0;
            if (tiled) {
                CK(cudaEventRecord(c->ev_halo[0], c->stream));
                CK(cudaStreamWaitEvent(c->cst, c->ev_halo[0], 0));
                ST(nccl_exchange(c, S.F.own, S.F.own + (np - 1) * P.plane, S.f_lo.p, S.f_hi.p, size_t(P.plane),
                                 ncclFloat32, c->cst));
                CK(cudaEventRecord(c->ev_halo[1], c->cst));
                halo_ev = c->ev_halo[1];
            } else {
                ST(nccl_exchange(c, S.F.own, S.F.own + (np - 1) * P.plane, S.f_lo.p, S.f_hi.p, size_t(P.plane),
                                 ncclFloat32));
            }
        } else {
            for (size_t k = 0; k < plan.size(); ++k) {
                SlabState &S = *c->slabs[k];
                if (S.has_lo) {
                    SlabState &L = *c->slabs[k - 1];
                    CK(cudaMemcpyAsync(S.f_lo.p, L.F.own + (L.s.v1 - L.s.v0 - P.plane), 4 * P.plane,
                                       cudaMemcpyDeviceToDevice, c->stream));
                }
                if (S.has_hi)
                    CK(cudaMemcpyAsync(S.f_hi.p, c->slabs[k + 1]->F.own, 4 * P.plane, cudaMemcpyDeviceToDevice,
                                       c->stream));
            }
        }
    }
    // ---- local labels (the main kernel of slab 0 is timed for the roofline)
    c->stats.bytes_main = 8 * (c->slabs[0]->s.v1 - c->slabs[0]->s.v0);   // read f + write label once
    for (SlabState *S : c->slabs) {
        const bool first = S == c->slabs[0];
        if (tiled) {
            eg_status s = tiled3d_local(S->tiled, P.ndim, P.dims, S->s, S->F, S->label, c->flags.as<int>(),
                                        c->stream, &c->stats, &c->err, first ? c->ev_main[0] : nullptr,
                                        first ? c->ev_main[1] : nullptr,
                                        (flags & EG_STATS) ? c->stat_buf.as<unsigned long long>() : nullptr,
                                        halo_ev, !multi ? c->io : nullptr);
            if (s != EG_OK) {
                if (s == EG_ERR_CUDA) c->poisoned = true;
                return s;
            }
        } else {
            ST(generic_local(c, P, *S, multi, first));
        }
    }
    c->stats.path = tiled ? 1 : 0;
    CK(cudaEventRecord(c->ev[1], c->stream));
    const bool raw = (flags & EG_RAW_ARCS) != 0;
    // One slab on one GPU, plain maximum graph: the graph stage (node lists,
    // arcs -- which follow a representative's exit pointer themselves -- and
    // their copies to the host) runs on the aux stream while the labels are
    // finalised on the ctx stream.  The widening flags keep the serial order.
    // (several slabs in one process: after the boundary exchange, when every
    // halo value is final)
    c->overlap = tiled && c->world == 1 && !c->min_reflect && !c->bundle &&
                 !(flags & (EG_ARC_PATHS | EG_NODE_VALUES | EG_RAW_ARCS));
    c->gstream = c->overlap ? c->aux : c->stream;
    if (c->overlap && !multi) {
        CK(cudaEventRecord(c->ev_tile, c->stream));
        CK(cudaStreamWaitEvent(c->aux, c->ev_tile, 0));
    }
    // ---- cross-slab resolution, then every unresolved owned label
    if (multi) {
        int rounds = 0;
        CK(cudaEventRecord(c->ev_s2[2], c->stream));
        ST(boundary_rounds(c, &rounds));
        CK(cudaEventRecord(c->ev_s2[3], c->stream));
        c->s2_timed[1] = true;
        c->stats.boundary_rounds = rounds;
        if (c->overlap) {
            CK(cudaEventRecord(c->ev_tile, c->stream));
            CK(cudaStreamWaitEvent(c->aux, c->ev_tile, 0));
        }
    }
    if (tiled || multi) {
        CK(cudaEventRecord(c->ev_s2[4], c->stream));
        c->s2_timed[2] = true;
    }
    const bool piped = c->io && c->io->done;      // eg_compute_host pipeline: labels finished on c->io->fst
    if (piped) CK(cudaStreamWaitEvent(c->stream, c->io->fin_done, 0));
    if (multi) {
        // every boundary value is final now: each slab's own boundary planes
        // take them, and (several GPUs) the halo planes around the owned labels
        // take the neighbours'; then ONE label pass over the whole label array
        // of this process chases exactly like the one-slab pass: a chain that
        // reaches another slab stops at a final boundary value
        const int64_t pl = P.plane;
        for (SlabState *S : c->slabs) {
            const int64_t n = S->s.v1 - S->s.v0;
            CK(cudaMemcpyAsync(S->label, S->bval.p, 4 * pl, cudaMemcpyDeviceToDevice, c->stream));
            CK(cudaMemcpyAsync(S->label + n - pl, S->bval.as<int32_t>() + pl, 4 * pl, cudaMemcpyDeviceToDevice,
                               c->stream));
        }
        int64_t e0 = base_v, e1 = base_v + nlab;
        if (c->world > 1) {
            SlabState &S = *c->slabs[0];
            if (S.has_lo) {
                CK(cudaMemcpyAsync(c->label_all.p, S.hval_lo.p, 4 * pl, cudaMemcpyDeviceToDevice, c->stream));
                e0 -= pl;
            }
            if (S.has_hi) {
                CK(cudaMemcpyAsync(c->label_all.as<int32_t>() + hpad + nlab, S.hval_hi.p, 4 * pl,
                                   cudaMemcpyDeviceToDevice, c->stream));
                e1 += pl;
            }
        }
        int32_t *lab0 = c->label_all.as<int32_t>() + hpad - (base_v - e0);
        unsigned long long *hist = (flags & EG_STATS) ? c->stat_buf.as<unsigned long long>() + 1 : nullptr;
        const char *sv = std::getenv("EG_FIN_SPLIT");
        const int split = sv ? std::atoi(sv) : 2;
        bool faces = P.ndim == 3 && split && tiled;
        for (SlabState *S : c->slabs) faces = faces && S->s.z1 - S->s.z0 > kTileZ;
        if (faces) {
            // per slab (tiles start at every slab's first plane): first the z-face
            // plane pairs of every slab, then the rest of every slab; a chain that
            // reaches another slab stops at a final boundary value (or, with several
            // GPUs, at a final halo plane)
            for (int pm : {1 | (split >= 3 ? 2 : 0), 4})
                for (SlabState *S : c->slabs) {
                    CK(launch_finalize_faces(S->label, S->s.v0, P.dims[0], P.dims[1], S->s.z1 - S->s.z0, kTileZ,
                                             kTileY, split >= 3, pm, c->stream, hist));
                    c->stats.kernel_launches += pm == 4 ? 1 : (split >= 3 ? 2 : 1);
                }
        } else {
            CK(launch_finalize(lab0, nullptr, e0, e1, c->stream, hist));
            c->stats.kernel_launches += 1;
        }
    }
    for (SlabState *S : c->slabs) {
        if (!tiled && !multi) continue;           // generic single slab: already final
        if (piped || multi) continue;
        unsigned long long *hist = (flags & EG_STATS) ? c->stat_buf.as<unsigned long long>() + 1 : nullptr;
        // tuning knob EG_FIN_SPLIT: 0 = one pass over every label; 2 = the z-face
        // plane pairs first, then the rest (default; C3 8.83 -> 8.46 ms); 3 = z-face
        // planes, y-face rows, the rest (8.67 ms)
        const char *sv = std::getenv("EG_FIN_SPLIT");
        const int split = sv ? std::atoi(sv) : 2;
        if (P.ndim == 3 && split && S->s.z1 - S->s.z0 > kTileZ) {
            // a chain of the later pass that leaves its tile through a z face ends
            // one load later, at a label the first pass already finished (k_slab.cu)
            CK(launch_finalize_faces(S->label, S->s.v0, P.dims[0], P.dims[1], S->s.z1 - S->s.z0, kTileZ, kTileY,
                                     split >= 3, 7, c->stream, hist));
            c->stats.kernel_launches += split >= 3 ? 3 : 2;
        } else {
            CK(launch_finalize(S->label, nullptr, S->s.v0, S->s.v1, c->stream, hist));
            c->stats.kernel_launches += 1;
        }
    }
    if (tiled || multi) CK(cudaEventRecord(c->ev_s2[5], c->stream));
    CK(cudaEventRecord(c->ev[2], c->stream));
    if (!c->overlap) ST(fail_if_flags(c));
    c->d_labels = c->label_all.as<int32_t>() + hpad;
    c->n_own = nlab;
    c->have_labels = true;
    // one GPU, one slab, graph wanted: the node lists are copied early
    c->early_d2h =
        c->world == 1 && c->slabs.size() == 1 && !raw && !(flags & EG_NO_GRAPH_D2H) && !c->min_reflect && !c->bundle;
    for (SlabState *S : c->slabs) ST(grid_graph(c, P, *S, raw, c->early_d2h));
    if (c->early_d2h) CK(cudaEventRecord(c->ev_d2h[2], c->d2h));
    CK(cudaEventRecord(c->ev[4], c->gstream));
    // (overlap: the flags are checked once the graph copies are queued, compute_impl)
    c->raw_valid = raw;
    return EG_OK;
}

// ------------------------------------------------------------- CSR stages

static eg_status compute_csr(eg_ctx *c, const Problem &P, const float *f, uint32_t flags) {
    const int vparts = int((flags >> 16) & 0xffff);
    c->overlap = false;
    c->gstream = c->stream;
    std::vector<std::pair<int64_t, int64_t>> plan;       // vertex ranges of this process
    std::vector<int64_t> all;                            // every rank's range (multi-GPU)
    if (c->world > 1) {
        plan.push_back({P.v0, P.v1});
        int64_t mine[2] = {P.v0, P.v1};
        ST(nccl_allgather_i64(c, mine, 2, all));
        for (int r = 0; r < c->world; ++r) {
            const int64_t prev = r ? all[2 * r - 1] : 0;
            if (all[2 * r] != prev || (r == c->world - 1 && all[2 * r + 1] != P.N))
                return set_err(c, EG_ERR_INVALID_ARG, "vertex ranges must tile [0, N) in rank order");
        }
    } else if (vparts > 1) {
        for (int k = 0; k < vparts; ++k) plan.push_back({P.N * k / vparts, P.N * (k + 1) / vparts});
    } else {
        plan.push_back({0, P.N});
    }
    set_slab_count(c, plan.size());
    // every rank holds the full pointer / label array (the graph is replicated)
    CK(c->label_all.ensure(sizeof(int32_t) * std::max<int64_t>(P.N, 1)));
    for (size_t k = 0; k < plan.size(); ++k) {
        SlabState &S = *c->slabs[k];
        S.s = Slab{0, 0, 0, plan[k].first, plan[k].second};
        S.F = FieldView{f, nullptr, nullptr, 0, P.N, 0};
        S.label = c->label_all.as<int32_t>() + S.s.v0;
        const int64_t words = (S.s.v1 - S.s.v0 + 31) / 32;
        CK(S.sad_bits.ensure(sizeof(uint32_t) * std::max<int64_t>(words, 1)));
        CK(S.max_bits.ensure(sizeof(uint32_t) * std::max<int64_t>(words, 1)));
        S.tiled_lists = false;
        CK(S.beta8.ensure(std::max<int64_t>(S.s.v1 - S.s.v0, 1)));
        CK(S.rep_buf.ensure(sizeof(int32_t) * std::max<int64_t>(P.nnz, 1)));
        S.has_lo = S.has_hi = false;
    }
    const int64_t cap = std::max<int64_t>(P.nnz, 1);
    CK(c->csr_scratch.ensure(sizeof(int32_t) * (2 * cap + std::max<int64_t>(P.N, 1))));
    int32_t *upl = c->csr_scratch.as<int32_t>(), *par = upl + cap, *nup = upl + 2 * cap;
    if (flags & EG_CHECK_CSR) {
        // validated before any kernel indexes through the graph (an invalid
        // col_idx would read out of bounds)
        CK(launch_check_csr(P.row_ptr, P.col_idx, P.N, P.nnz, c->flags.as<int>() + 1, c->stream));
        c->stats.kernel_launches += 1;
        ST(fail_if_flags(c));
    }
    CK(cudaEventRecord(c->ev[0], c->stream));
    int *fl = c->flags.as<int>();
    {
        const int64_t n0 = c->slabs[0]->s.v1 - c->slabs[0]->s.v0;
        // f, the CSR rows of the range, the gradient written once
        c->stats.bytes_main = 8 * n0 + 8 * (n0 + 1) + 4 * (P.nnz * n0 / std::max<int64_t>(P.N, 1));
    }
    // S1 for every vertex of the graph on every rank (the S3 pass of a range
    // reads the upper lists of the range's neighbours, and the gradients of
    // the whole graph feed S2): cheap next to S3, and no exchange is needed
    CK(cudaEventRecord(c->ev_main[0], c->stream));
    int64_t covered = 0;
    for (SlabState *S : c->slabs) {
        if (covered < S->s.v0) {        // ranges owned by other ranks
            CK(launch_csr_upper(P.row_ptr, P.col_idx, f, covered, S->s.v0, c->label_all.as<int32_t>() + covered,
                                nullptr, upl, nup, fl, c->stream));
            c->stats.kernel_launches += 1;
        }
        CK(launch_csr_upper(P.row_ptr, P.col_idx, f, S->s.v0, S->s.v1, S->label, S->max_bits.as<uint32_t>(), upl, nup,
                            fl, c->stream));
        c->stats.kernel_launches += 1;
        covered = S->s.v1;
    }
    if (covered < P.N) {
        CK(launch_csr_upper(P.row_ptr, P.col_idx, f, covered, P.N, c->label_all.as<int32_t>() + covered, nullptr, upl,
                            nup, fl, c->stream));
        c->stats.kernel_launches += 1;
    }
    for (SlabState *S : c->slabs) {
        CK(launch_csr_link(P.row_ptr, P.col_idx, f, S->s.v0, S->s.v1, upl, nup, S->sad_bits.as<uint32_t>(),
                           S->beta8.as<uint8_t>(), S->rep_buf.as<int32_t>(), par, c->stream));
        c->stats.kernel_launches += 1;
    }
    CK(cudaEventRecord(c->ev_main[1], c->stream));
    CK(cudaEventRecord(c->ev[1], c->stream));
    // S2 on the full array (every rank; N is small for CSR workloads)
    SlabState whole;
    whole.s = Slab{0, 0, 0, 0, P.N};
    whole.label = c->label_all.as<int32_t>();
    CK(cudaEventRecord(c->ev_s2[0], c->stream));
    c->s2_timed[0] = true;
    {
        int *changed = fl + 2;
        CK(cudaMemsetAsync(changed, 0, sizeof(int) * 64, c->stream));
        int hflag[64], rounds = 0;
        for (int r0 = 0; r0 < 60; r0 += 3) {
            const int r1 = std::min(60, r0 + 3);
            for (int r = r0; r < r1; ++r) {
                CK(launch_jump_round(whole.label, P.N, 0, changed, r, c->stream));
                c->stats.kernel_launches += 1;
            }
            CK(cudaMemcpyAsync(hflag, changed, sizeof(int) * r1, cudaMemcpyDeviceToHost, c->stream));
            CK(cudaStreamSynchronize(c->stream));
            int fz = -1;
            for (int r = 0; r < r1; ++r)
                if (hflag[r] == 0) {
                    fz = r;
                    break;
                }
            rounds = fz >= 0 ? fz + 1 : r1;
            if (fz >= 0) break;
        }
        c->stats.jump_rounds = rounds;
    }
    CK(cudaEventRecord(c->ev_s2[1], c->stream));
    whole.label = nullptr;
    CK(cudaEventRecord(c->ev[2], c->stream));
    ST(fail_if_flags(c));
    c->stats.path = 2;
    c->d_labels = c->label_all.as<int32_t>() + (c->world > 1 ? P.v0 : 0);
    c->n_own = (c->world > 1) ? P.v1 - P.v0 : P.N;
    c->have_labels = true;
    const bool raw = (flags & EG_RAW_ARCS) != 0;
    c->early_d2h = c->world == 1 && c->slabs.size() == 1 && !raw && !(flags & EG_NO_GRAPH_D2H) && !c->bundle;
    for (SlabState *S : c->slabs) ST(grid_graph(c, P, *S, raw, c->early_d2h));
    if (c->early_d2h) CK(cudaEventRecord(c->ev_d2h[2], c->d2h));
    CK(cudaEventRecord(c->ev[4], c->stream));
    c->raw_valid = raw;
    return EG_OK;
}

// Arc bundling (reading L19) of the one slab's graph, on the
// device: keep the highest saddle of every pair of maxima that several
// two-maxima saddles share; the kept saddles and arcs replace the slab's.
static eg_status bundle_arcs(eg_ctx *c) {
    SlabState &S = *c->slabs[0];
    const int64_t ns = S.n_sad;
    if (ns == 0) return EG_OK;
    const size_t sort_b = (bundle_sort_bytes(ns) + 255) / 256 * 256;
    const size_t scan_b = (scan_scratch_bytes(ns) + 255) / 256 * 256;
    const size_t n8 = (8 * size_t(ns) + 255) / 256 * 256, n4 = (4 * size_t(ns) + 255) / 256 * 256,
                 p8 = (8 * size_t(ns + 1) + 255) / 256 * 256;
    CK(c->bund_scratch.ensure(2 * n8 + 4 * n4 + 2 * p8 + sort_b + scan_b));
    char *p = c->bund_scratch.as<char>();
    BundleArgs B{};
    B.ns = ns;
    B.n_unique = S.n_unique.as<int32_t>();
    B.arc_off = S.arc_off.as<int64_t>();
    B.arc_s = S.arc_s.as<int64_t>();
    B.arc_m = S.arc_m.as<int64_t>();
    B.arc_mult = S.arc_mult.as<int32_t>();
    B.sad64 = S.saddles64.as<int64_t>();
    B.sad32 = S.saddles32.as<int32_t>();
    B.sbeta = S.sbeta.as<int32_t>();
    B.f = S.F.own;
    B.f_base = S.F.v0;
    B.keys = reinterpret_cast<uint64_t *>(p);
    p += n8;
    B.keys2 = reinterpret_cast<uint64_t *>(p);
    p += n8;
    B.idx = reinterpret_cast<int32_t *>(p);
    p += n4;
    B.idx2 = reinterpret_cast<int32_t *>(p);
    p += n4;
    B.keep = reinterpret_cast<int32_t *>(p);
    p += n4;
    B.arc_cnt = reinterpret_cast<int32_t *>(p);
    p += n4;
    B.s_pos = reinterpret_cast<int64_t *>(p);
    p += p8;
    B.a_pos = reinterpret_cast<int64_t *>(p);
    p += p8;
    B.sort_tmp = p;
    B.sort_bytes = sort_b;
    p += sort_b;
    B.scan_tmp = p;
    B.scan_bytes = scan_b;
    CK(c->b_sad64.ensure(8 * std::max<int64_t>(ns, 1)));
    CK(c->b_sad32.ensure(4 * std::max<int64_t>(ns, 1)));
    CK(c->b_sbeta.ensure(4 * std::max<int64_t>(ns, 1)));
    CK(c->b_nu.ensure(4 * std::max<int64_t>(ns, 1)));
    CK(c->b_arc_s.ensure(8 * std::max<int64_t>(S.n_arc, 1)));
    CK(c->b_arc_m.ensure(8 * std::max<int64_t>(S.n_arc, 1)));
    CK(c->b_arc_mult.ensure(4 * std::max<int64_t>(S.n_arc, 1)));
    B.o_sad64 = c->b_sad64.as<int64_t>();
    B.o_sad32 = c->b_sad32.as<int32_t>();
    B.o_sbeta = c->b_sbeta.as<int32_t>();
    B.o_nu = c->b_nu.as<int32_t>();
    B.o_arc_s = c->b_arc_s.as<int64_t>();
    B.o_arc_m = c->b_arc_m.as<int64_t>();
    B.o_arc_mult = c->b_arc_mult.as<int32_t>();
    CK(launch_bundle(B, c->stream));
    c->stats.kernel_launches += 11;
    int64_t cnt[2];
    CK(cudaMemcpyAsync(&cnt[0], B.s_pos + ns, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(&cnt[1], B.a_pos + ns, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    std::swap(S.saddles64, c->b_sad64);
    std::swap(S.saddles32, c->b_sad32);
    std::swap(S.sbeta, c->b_sbeta);
    std::swap(S.n_unique, c->b_nu);
    std::swap(S.arc_s, c->b_arc_s);
    std::swap(S.arc_m, c->b_arc_m);
    std::swap(S.arc_mult, c->b_arc_mult);
    S.n_sad = cnt[0];
    S.n_arc = cnt[1];
    c->n_sad = cnt[0];
    c->n_arc = cnt[1];
    return EG_OK;
}

// EG_ARC_PATHS: offsets and vertices to the host (at once, or on the first
// eg_get_arc_paths after a compute with EG_NO_GRAPH_D2H)
static eg_status fetch_paths(eg_ctx *c) {
    if (c->paths_on_host) return EG_OK;
    const int64_t nr = c->n_paths, total = c->n_path_v;
    CK(c->h_path_off.ensure(sizeof(int64_t) * (nr + 1)));
    CK(cudaMemcpyAsync(c->h_path_off.p, c->path_off.p, sizeof(int64_t) * (nr + 1), cudaMemcpyDeviceToHost, c->stream));
    CK(c->h_path_v.ensure(sizeof(int64_t) * std::max<int64_t>(total, 1)));
    if (total)
        CK(cudaMemcpyAsync(c->h_path_v.p, c->path_v.p, sizeof(int64_t) * total, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    c->paths_on_host = true;
    return EG_OK;
}

static eg_status compute_impl(eg_ctx *c, const eg_domain *d, const float *f, uint32_t flags, bool device_field) {
    if (!c) return EG_ERR_INVALID_ARG;
    if (c->poisoned)
        return set_err(c, EG_ERR_STATE, "context is poisoned by an earlier CUDA/NCCL error: %s", c->err.c_str());
    c->have_graph = c->have_labels = c->graph_on_host = false;
    c->graph_deferred = false;
    if (c->d2h) CK(cudaStreamSynchronize(c->d2h));   // no copy of an earlier call still in flight
    Problem P;
    ST(validate(c, d, f, device_field, &P));
    CK(cudaSetDevice(c->device));
    std::memset(&c->stats, 0, sizeof(c->stats));
    c->stats.n_vertices = P.N;
    CK(c->flags.ensure(sizeof(int) * 128));
    CK(c->counts.ensure(sizeof(int64_t) * 16 * (c->world + 1)));
    CK(cudaMemsetAsync(c->flags.p, 0, sizeof(int) * 128, c->stream));
    c->s2_timed[0] = c->s2_timed[1] = c->s2_timed[2] = false;
    if (flags & EG_STATS) {
        CK(c->stat_buf.ensure(sizeof(unsigned long long) * 32));
        CK(cudaMemsetAsync(c->stat_buf.p, 0, sizeof(unsigned long long) * 32, c->stream));
    }
    // EG_MINIMUM (reading L11): the maximum graph of g[i] = -f[N-1-i], mapped
    // back by i -> N-1-i (k_common.cu)
    const float *f_user = f;           // the caller's field (device) -- f becomes the mirror for a minimum graph
    c->minimum = (flags & EG_MINIMUM) != 0;
    // On a CSR graph (no reflection maps it onto itself), and for raw arcs /
    // arc paths (whose ids and order the reflection would have to map back),
    // the maximum graph of the field's reversed SoS-rank image (reading L22)
    // is the minimum graph, with vertex ids unchanged.
    c->min_reflect = false;
    if (c->minimum) {
        if (c->world > 1 || ((flags >> 16) & 0xffff) > 1)
            return set_err(c, EG_ERR_UNSUPPORTED, "EG_MINIMUM: one GPU and one slab");
        if (!P.grid && (P.v0 != 0 || P.v1 != P.N))
            return set_err(c, EG_ERR_UNSUPPORTED, "EG_MINIMUM on a CSR graph: the whole vertex range");
        CK(c->mirror.ensure(sizeof(float) * std::max<int64_t>(P.N, 1)));
        c->min_reflect = P.grid && !(flags & (EG_RAW_ARCS | EG_ARC_PATHS));
        if (c->min_reflect) {
            CK(launch_reflect_negate(f, c->mirror.as<float>(), P.N, c->stream));
            c->stats.kernel_launches += 1;
        } else {
            if (P.N > kRankMaxN) return set_err(c, EG_ERR_UNSUPPORTED, "EG_MINIMUM by rank image: N too large");
            size_t bytes = 0;
            CK(launch_rank_f32(f, EG_DTYPE_F32, nullptr, P.N, nullptr, &bytes, true, c->stream));
            CK(c->rank_scratch.ensure(bytes));
            CK(launch_rank_f32(f, EG_DTYPE_F32, c->mirror.as<float>(), P.N, c->rank_scratch.p, &bytes, true,
                               c->stream));
            c->stats.kernel_launches += 2 + 4;   // keys, scatter + the radix sort's passes (approx.)
        }
        f = c->mirror.as<float>();
    }
    c->paths_valid = false;
    c->bundle = (flags & EG_BUNDLE) != 0;
    c->g32 = (flags & EG_GRAPH32) && c->world == 1 && !c->bundle && !(flags & (EG_MINIMUM | EG_NODE_VALUES));
    c->h64_valid = !c->g32;
    c->h32_valid = c->g32;
    if (c->bundle && (c->world > 1 || ((flags >> 16) & 0xffff) > 1))
        return set_err(c, EG_ERR_UNSUPPORTED, "EG_BUNDLE: one GPU, one slab");
    if (flags & EG_ARC_PATHS) {
        if (c->world > 1 || ((flags >> 16) & 0xffff) > 1)
            return set_err(c, EG_ERR_UNSUPPORTED, "EG_ARC_PATHS: one GPU, one slab");
        flags |= EG_RAW_ARCS;
    }
    if (P.grid) ST(compute_grid(c, P, f, flags));
    else ST(compute_csr(c, P, f, flags));
    if (flags & EG_ARC_PATHS) {
        // integral lines of the raw arcs: lengths, scan, vertices, to the host
        SlabState &S = *c->slabs[0];
        const int64_t nr = S.n_raw;
        CK(c->path_len.ensure(sizeof(int64_t) * std::max<int64_t>(nr, 1)));
        CK(c->path_off.ensure(sizeof(int64_t) * (nr + 1)));
        // pass 1 walks every path (argmax recomputed from f) for its length and
        // leaves each visited vertex's next step in path_nxt; pass 2 follows those
        CK(c->path_nxt.ensure(sizeof(int32_t) * std::max<int64_t>(P.N, 1)));
        int32_t *nxt = c->path_nxt.as<int32_t>();
        if (P.grid)
            CK(launch_arc_paths_grid(c->host_tab, P.ndim, S.F, S.raw_s.as<int64_t>(), S.raw_rep.as<int64_t>(), nr,
                                     nullptr, c->path_len.as<int64_t>(), c->stream, nxt));
        else
            CK(launch_arc_paths_csr(P.row_ptr, P.col_idx, f, S.raw_s.as<int64_t>(), S.raw_rep.as<int64_t>(), nr,
                                    nullptr, c->path_len.as<int64_t>(), c->stream, nxt));
        const size_t sb = scan64_scratch_bytes(std::max<int64_t>(nr, 1));
        CK(c->scratch.ensure(sb));
        CK(launch_scan_i64(c->path_len.as<int64_t>(), c->path_off.as<int64_t>(), nr, c->scratch.p, sb, c->stream));
        CK(c->h_path_off.ensure(sizeof(int64_t) * (nr + 1)));
        CK(cudaMemcpyAsync(c->h_path_off.as<int64_t>() + nr, c->path_off.as<int64_t>() + nr, sizeof(int64_t),
                           cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        const int64_t total = c->h_path_off.as<int64_t>()[nr];
        CK(c->path_v.ensure(sizeof(int64_t) * std::max<int64_t>(total, 1)));
        CK(launch_arc_paths_follow(S.raw_s.as<int64_t>(), S.raw_rep.as<int64_t>(), nr, c->path_off.as<int64_t>(), nxt,
                                   P.grid ? S.F.v0 : 0, c->path_v.as<int64_t>(), c->stream));
        c->n_paths = nr;
        c->n_path_v = total;
        c->paths_valid = true;
        c->paths_on_host = false;
        if (!(flags & EG_NO_GRAPH_D2H)) ST(fetch_paths(c));   // else on request (eg_get_arc_paths)
        c->stats.kernel_launches += 3;
    }
    if (c->bundle) ST(bundle_arcs(c));
    if (c->min_reflect) {
        SlabState &S = *c->slabs[0];
        const int64_t N = P.N;
        CK(launch_reverse_i32(c->label_all.as<int32_t>(), N, N, true, c->stream));
        CK(launch_reverse_i64(S.maxima64.as<int64_t>(), S.n_max, N, true, c->stream));
        CK(launch_reverse_i64(S.saddles64.as<int64_t>(), S.n_sad, N, true, c->stream));
        CK(launch_reverse_i32(S.saddles32.as<int32_t>(), S.n_sad, N, true, c->stream));
        CK(launch_reverse_i32(S.sbeta.as<int32_t>(), S.n_sad, N, false, c->stream));
        CK(launch_reverse_i64(S.arc_s.as<int64_t>(), S.n_arc, N, true, c->stream));
        CK(launch_reverse_i64(S.arc_m.as<int64_t>(), S.n_arc, N, true, c->stream));
        CK(launch_reverse_i32(S.arc_mult.as<int32_t>(), S.n_arc, N, false, c->stream));
        c->stats.kernel_launches += 8;
    }
    if (!(flags & EG_NO_GRAPH_D2H)) {
        ST(gather_graph(c, (flags & EG_RAW_ARCS) != 0));
        c->graph_on_host = true;
    } else if (c->world == 1) {
        // the graph stays in HBM (ctx-owned device arrays, valid until the next
        // compute); eg_get_graph* copies it to the host on the first request
        c->graph_deferred = true;
        c->deferred_raw = (flags & EG_RAW_ARCS) != 0;
    }
    if (c->gstream != c->stream) {             // join the graph stage (aux) into the ctx stream
        CK(cudaEventRecord(c->ev_graph, c->gstream));
        CK(cudaStreamWaitEvent(c->stream, c->ev_graph, 0));
    }
    // overlap: the arc copies above were queued while the finalize pass still
    // runs (checking the flags first would hold them until it ends)
    if (c->overlap) ST(fail_if_flags(c));
    c->node_values = false;
    c->last_minimum = c->minimum;
    if ((flags & EG_NODE_VALUES) && c->world == 1 && c->graph_on_host) {
        // f (of the caller's field) at every maximum and saddle, slab by slab
        CK(c->d_fnode.ensure(sizeof(float) * std::max<int64_t>(c->n_max + c->n_sad, 1)));
        CK(c->h_fmax.ensure(sizeof(float) * std::max<int64_t>(c->n_max, 1)));
        CK(c->h_fsad.ensure(sizeof(float) * std::max<int64_t>(c->n_sad, 1)));
        float *dm = c->d_fnode.as<float>(), *ds = dm + c->n_max;
        int64_t om = 0, os = 0;
        for (SlabState *S : c->slabs) {
            CK(launch_gather_f(f_user, 0, S->maxima64.as<int64_t>(), S->n_max, dm + om, c->stream));
            CK(launch_gather_f(f_user, 0, S->saddles64.as<int64_t>(), S->n_sad, ds + os, c->stream));
            om += S->n_max;
            os += S->n_sad;
        }
        if (c->n_max) CK(cudaMemcpyAsync(c->h_fmax.p, dm, sizeof(float) * c->n_max, cudaMemcpyDeviceToHost, c->stream));
        if (c->n_sad) CK(cudaMemcpyAsync(c->h_fsad.p, ds, sizeof(float) * c->n_sad, cudaMemcpyDeviceToHost, c->stream));
        c->stats.kernel_launches += 2 * int(c->slabs.size());
        c->node_values = true;
    }
    CK(cudaEventRecord(c->ev[5], c->stream));
    CK(cudaStreamSynchronize(c->stream));
    c->have_graph = true;
    c->stats.us_classify = ev_us(c->ev[0], c->ev[1]);
    c->stats.us_jump = c->s2_timed[0] ? ev_us(c->ev_s2[0], c->ev_s2[1]) : 0.0;
    c->stats.us_boundary = c->s2_timed[1] ? ev_us(c->ev_s2[2], c->ev_s2[3]) : 0.0;
    c->stats.us_label = c->s2_timed[2] ? ev_us(c->ev_s2[4], c->ev_s2[5]) : 0.0;
    if (flags & EG_STATS) {
        unsigned long long h[32];
        CK(cudaMemcpy(h, c->stat_buf.p, sizeof(h), cudaMemcpyDeviceToHost));
        c->stats.n_exit = int64_t(h[0]);
        for (int k = 0; k < 16; ++k) c->stats.chase_hist[k] = int64_t(h[1 + k]);
        c->stats.chase_max = int32_t(h[17]);
    }
    c->stats.us_arcs = ev_us(c->ev[2], c->ev[4]);
    c->stats.us_graph = ev_us(c->ev[4], c->ev[5]);
    c->stats.us_total = ev_us(c->ev[0], c->ev[5]);
    c->stats.us_main = ev_us(c->ev_main[0], c->ev_main[1]);
    c->stats.bytes_alg = 8 * P.N + 4 * c->n_max + 5 * c->n_sad + 12 * c->n_arc +
                         (P.grid ? 0 : 8 * (P.N + 1) + 4 * P.nnz);
    return EG_OK;
}

// ------------------------------------------------------------------- ABI

extern "C" {

eg_status eg_create(eg_ctx **out, int cuda_device, void *cuda_stream) {
    if (!out) return EG_ERR_INVALID_ARG;
    *out = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return EG_ERR_CUDA;       // no CPU fallback
    }
    if (cuda_device < 0 || cuda_device >= ndev) return EG_ERR_INVALID_ARG;
    eg_ctx *c = new (std::nothrow) eg_ctx();
    if (!c) return EG_ERR_OOM;
    c->device = cuda_device;
    c->stream = static_cast<cudaStream_t>(cuda_stream);
    if (cudaSetDevice(cuda_device) != cudaSuccess) {
        delete c;
        return EG_ERR_CUDA;
    }
    for (auto &e : c->ev)
        if (cudaEventCreate(&e) != cudaSuccess) {
            delete c;
            return EG_ERR_CUDA;
        }
    for (auto &e : c->ev_main)
        if (cudaEventCreate(&e) != cudaSuccess) {
            delete c;
            return EG_ERR_CUDA;
        }
    for (auto &e : c->ev_s2)
        if (cudaEventCreate(&e) != cudaSuccess) {
            delete c;
            return EG_ERR_CUDA;
        }
    for (auto &e : c->ev_d2h)
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
            delete c;
            return EG_ERR_CUDA;
        }
    if (cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking) != cudaSuccess ||
        cudaDeviceGetStreamPriorityRange(&c->prio_lo, &c->prio_hi) != cudaSuccess ||
        // high priority: the graph stage's few blocks run ahead of the finalize pass's queue
        cudaStreamCreateWithPriority(&c->aux, cudaStreamNonBlocking, c->prio_hi) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->cst, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->ld2h, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->fst, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_halo[0], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_halo[1], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_tile, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_graph, cudaEventDisableTiming) != cudaSuccess) {
        delete c;
        return EG_ERR_CUDA;
    }
    c->gstream = c->stream;
    *out = c;
    return EG_OK;
}

eg_status eg_nccl_unique_id(void *out128) {
    if (!out128) return EG_ERR_INVALID_ARG;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return EG_ERR_NCCL;
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(out128, &id, sizeof(id));
    return EG_OK;
}

eg_status eg_create_dist(eg_ctx **out, int cuda_device, void *cuda_stream, const void *nccl_id128, int rank,
                         int world) {
    if (!out || !nccl_id128 || world < 1 || rank < 0 || rank >= world) return EG_ERR_INVALID_ARG;
    eg_status s = eg_create(out, cuda_device, cuda_stream);
    if (s != EG_OK) return s;
    eg_ctx *c = *out;
    c->rank = rank;
    c->world = world;
    if (world > 1) {
        ncclUniqueId id;
        std::memcpy(&id, nccl_id128, sizeof(id));
        ncclResult_t r = ncclCommInitRank(&c->comm, world, id, rank);
        if (r != ncclSuccess) {
            set_err(c, EG_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
            return EG_ERR_NCCL;       // the ctx stays valid for eg_last_error / eg_destroy
        }
    }
    return EG_OK;
}

eg_status eg_compute(eg_ctx *c, const eg_domain *d, const float *d_field, uint32_t flags) {
    return compute_impl(c, d, d_field, flags, true);
}

eg_status eg_compute_typed(eg_ctx *c, const eg_domain *d, const void *d_field, int dtype, uint32_t flags) {
    if (!c || !d) return EG_ERR_INVALID_ARG;
    if (dtype == EG_DTYPE_F32) return compute_impl(c, d, static_cast<const float *>(d_field), flags, true);
    if (dtype < EG_DTYPE_F16 || dtype > EG_DTYPE_U64) return set_err(c, EG_ERR_INVALID_ARG, "dtype %d", dtype);
    const bool rank = dtype >= EG_DTYPE_F64;   // SoS-rank image (reading L22)
    if (rank && c->world != 1)
        return set_err(c, EG_ERR_UNSUPPORTED, "dtype %d: the rank image needs the whole field on one GPU", dtype);
    if (rank && (flags & EG_NODE_VALUES))
        return set_err(c, EG_ERR_UNSUPPORTED, "dtype %d: node values have no float32 image", dtype);
    if (c->poisoned) return set_err(c, EG_ERR_STATE, "context is poisoned: %s", c->err.c_str());
    if (!is_device_ptr(d_field)) return set_err(c, EG_ERR_INVALID_ARG, "d_field must be a device pointer");
    // the number of elements the domain covers on this rank
    int64_t n = 0;
    if (d->kind == EG_DOMAIN_GRID) {
        const eg_grid &g = d->grid;
        if (g.ndim < 1 || g.ndim > 8) return set_err(c, EG_ERR_INVALID_ARG, "ndim %d", g.ndim);
        int64_t plane = 1;
        for (int i = 0; i + 1 < g.ndim; ++i) plane *= g.dims[i];
        n = plane * (g.slab_end - g.slab_begin);
    } else {
        n = d->csr.n_vertices;
    }
    if (n <= 0) return set_err(c, EG_ERR_INVALID_ARG, "empty field");
    CK(cudaSetDevice(c->device));
    CK(c->typed.ensure(sizeof(float) * size_t(n)));
    if (rank) {
        // every value exactly a float32 (f32 data stored wider, integers below
        // 2^24, ...): the cast is an order isomorphism, no rank sort needed
        CK(c->flags.ensure(sizeof(int) * 128));
        CK(cudaMemsetAsync(c->flags.p, 0, sizeof(int), c->stream));
        CK(launch_exact_f32(d_field, dtype, c->typed.as<float>(), n, c->flags.as<int>(), c->stream));
        int inexact = 1;
        CK(cudaMemcpyAsync(&inexact, c->flags.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        if (!inexact) {
            c->stats.kernel_launches += 1;
            return compute_impl(c, d, c->typed.as<float>(), flags, true);
        }
    }
    if (rank) {
        if (n > kRankMaxN) return set_err(c, EG_ERR_UNSUPPORTED, "rank image: N = %lld too large", (long long)n);
        size_t bytes = 0;
        CK(launch_rank_f32(d_field, dtype, nullptr, n, nullptr, &bytes, false, c->stream));
        CK(c->rank_scratch.ensure(bytes));
        CK(launch_rank_f32(d_field, dtype, c->typed.as<float>(), n, c->rank_scratch.p, &bytes, false, c->stream));
    } else {
        CK(launch_to_f32(d_field, dtype, c->typed.as<float>(), n, c->stream));
    }
    return compute_impl(c, d, c->typed.as<float>(), flags, true);
}

static void tiled3d_fin_list_of(eg_ctx *c, const int32_t **list, const unsigned long long **n, int64_t *cap) {
    tiled3d_fin_list(c->slabs[0]->tiled, list, n, cap);
}

static bool is_pinned(const void *p) {
    cudaPointerAttributes a;
    const bool ok = p && cudaPointerGetAttributes(&a, p) == cudaSuccess && a.type == cudaMemoryTypeHost;
    cudaGetLastError();
    return ok;
}

eg_status eg_compute_host(eg_ctx *c, const eg_domain *d, const float *h_field, int32_t *h_labels, uint32_t flags) {
    if (!c) return EG_ERR_INVALID_ARG;
    if (c->poisoned) return set_err(c, EG_ERR_STATE, "context is poisoned: %s", c->err.c_str());
    Problem P;
    ST(validate(c, d, h_field, false, &P));
    if (is_device_ptr(h_field)) return set_err(c, EG_ERR_INVALID_ARG, "eg_compute_host takes a host field");
    CK(cudaSetDevice(c->device));
    const int64_t nfield = P.grid ? (P.v1 - P.v0) : P.N;
    CK(c->field.ensure(sizeof(float) * std::max<int64_t>(nfield, 1)));
    const bool pinned = is_pinned(h_field);
    // the pipeline (one 3-D slab of whole tiles on one GPU, pinned host
    // buffers, the plain maximum graph): the field arrives in z-chunks, each
    // chunk's labels leave while later chunks arrive (ChunkIO, k_grid3d.cu);
    // EG_E2E_CHUNKS = chunk count (1 = off)
    const char *ek = std::getenv("EG_E2E_CHUNKS");
    const int K = ek ? std::atoi(ek) : 16;
    const bool pipe = K >= 2 && pinned && (!h_labels || is_pinned(h_labels)) && c->world == 1 && P.grid &&
                      P.ndim == 3 && P.dims[0] % 32 == 0 && P.dims[1] % 16 == 0 && P.dims[2] % 16 == 0 &&
                      !(flags & (EG_FORCE_GENERIC | EG_MINIMUM | EG_RAW_ARCS | EG_ARC_PATHS | EG_BUNDLE |
                                 EG_NODE_VALUES)) &&
                      ((flags >> 16) & 0xffff) <= 1;
    ChunkIO io;
    if (pipe) {
        CK(cudaStreamSynchronize(c->stream));       // the previous call's uses of c->field are done
        io.K = K;
        io.h2d = c->h2d;
        io.d2h = c->ld2h;
        io.fst = c->fst;
        io.h_field = h_field;
        io.d_field = c->field.as<float>();
        io.h_labels = h_labels;
        c->io = &io;
    } else if (pinned || nfield * 4 <= (int64_t(1) << 20)) {
        CK(cudaMemcpyAsync(c->field.p, h_field, sizeof(float) * nfield, cudaMemcpyHostToDevice, c->stream));
    } else {
        // pageable source: stage through two pinned halves
        const size_t chunk = size_t(64) << 20;
        CK(c->h_stage.ensure(2 * chunk));
        char *stage = c->h_stage.as<char>();
        const char *src = reinterpret_cast<const char *>(h_field);
        char *dst = c->field.as<char>();
        const size_t total = sizeof(float) * size_t(nfield);
        cudaEvent_t done[2] = {c->ev[6], c->ev[7]};
        bool used[2] = {false, false};
        int k = 0;
        for (size_t off = 0; off < total; off += chunk, k ^= 1) {
            const size_t len = std::min(chunk, total - off);
            if (used[k]) CK(cudaEventSynchronize(done[k]));
            std::memcpy(stage + k * chunk, src + off, len);
            CK(cudaMemcpyAsync(dst + off, stage + k * chunk, len, cudaMemcpyHostToDevice, c->stream));
            CK(cudaEventRecord(done[k], c->stream));
            used[k] = true;
        }
    }
    const eg_status st = compute_impl(c, d, c->field.as<float>(), flags, true);
    c->io = nullptr;
    if (st != EG_OK) {
        if (pipe) {
            cudaStreamSynchronize(c->h2d);
            cudaStreamSynchronize(c->fst);
            cudaStreamSynchronize(c->ld2h);
        }
        return st;
    }
    if (h_labels) {
        if (pipe && io.done) {
            // the label chunks are on their way; the vertices the chunked pass
            // finished last (after their chunk was copied) are patched
            CK(cudaEventSynchronize(io.d2h_done));
            const int32_t *d_list = nullptr;
            const unsigned long long *d_n = nullptr;
            int64_t cap = 0;
            tiled3d_fin_list_of(c, &d_list, &d_n, &cap);
            unsigned long long n = 0;
            CK(cudaMemcpy(&n, d_n, sizeof(n), cudaMemcpyDeviceToHost));
            c->stats.n_exit_targets = int64_t(n);       // (reported: labels patched on the host)
            if (int64_t(n) > cap) {
                CK(cudaMemcpy(h_labels, c->d_labels, sizeof(int32_t) * c->n_own, cudaMemcpyDeviceToHost));
            } else if (n > 0) {
                CK(c->fix_dev.ensure(sizeof(int32_t) * 2 * n));
                int32_t *dv = c->fix_dev.as<int32_t>();
                CK(launch_gather_labels(c->d_labels, d_list, int64_t(n), dv, c->stream));
                CK(cudaMemcpyAsync(dv + n, d_list, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, c->stream));
                std::vector<int32_t> hv(2 * n);
                CK(cudaMemcpyAsync(hv.data(), dv, sizeof(int32_t) * 2 * n, cudaMemcpyDeviceToHost, c->stream));
                CK(cudaStreamSynchronize(c->stream));
                for (unsigned long long j = 0; j < n; ++j) h_labels[hv[n + j]] = hv[j];
            }
        } else {
            CK(cudaMemcpyAsync(h_labels, c->d_labels, sizeof(int32_t) * c->n_own, cudaMemcpyDeviceToHost,
                               c->stream));
            CK(cudaStreamSynchronize(c->stream));
        }
    } else if (pipe) {
        CK(cudaStreamSynchronize(c->ld2h));
    }
    return EG_OK;
}

eg_status eg_gradient(eg_ctx *c, const eg_domain *d, const float *d_field, int32_t *d_ptr, uint8_t *d_beta) {
    if (!c) return EG_ERR_INVALID_ARG;
    if (c->poisoned) return set_err(c, EG_ERR_STATE, "context is poisoned: %s", c->err.c_str());
    if (c->world > 1) return set_err(c, EG_ERR_UNSUPPORTED, "eg_gradient is single-GPU");
    Problem P;
    ST(validate(c, d, d_field, true, &P));
    if (!is_device_ptr(d_ptr) || !is_device_ptr(d_beta))
        return set_err(c, EG_ERR_INVALID_ARG, "d_ptr / d_beta must be device pointers");
    CK(cudaSetDevice(c->device));
    const int64_t n = P.v1 - P.v0, words = (n + 31) / 32;
    set_slab_count(c, std::max<size_t>(c->slabs.size(), 1));
    SlabState &S = *c->slabs[0];
    CK(S.sad_bits.ensure(sizeof(uint32_t) * std::max<int64_t>(words, 1)));
    CK(S.max_bits.ensure(sizeof(uint32_t) * std::max<int64_t>(words, 1)));
    CK(c->flags.ensure(sizeof(int) * 128));
    CK(cudaMemsetAsync(c->flags.p, 0, sizeof(int) * 128, c->stream));
    if (P.grid) {
        ST(ensure_table(c, P));
        const Slab s{0, P.D, P.plane, 0, P.N};
        const FieldView F{d_field, nullptr, nullptr, 0, P.N, P.plane};
        CK(launch_classify_grid(c->host_tab, P.ndim, F, s, d_ptr, S.sad_bits.as<uint32_t>(),
                                S.max_bits.as<uint32_t>(), d_beta, c->flags.as<int>(), c->stream));
    } else {
        const int64_t cap = std::max<int64_t>(P.nnz, 1);
        CK(c->csr_scratch.ensure(sizeof(int32_t) * (2 * cap + std::max<int64_t>(P.N, 1))));
        int32_t *upl = c->csr_scratch.as<int32_t>(), *par = upl + cap, *nup = upl + 2 * cap;
        CK(launch_csr_upper(P.row_ptr, P.col_idx, d_field, P.v0, P.v1, d_ptr, S.max_bits.as<uint32_t>(), upl, nup,
                            c->flags.as<int>(), c->stream));
        CK(launch_csr_link(P.row_ptr, P.col_idx, d_field, P.v0, P.v1, upl, nup, S.sad_bits.as<uint32_t>(), d_beta,
                           nullptr, par, c->stream));
    }
    return fail_if_flags(c);
}

// the host graph in the other id width, on first use (EG_GRAPH32)
static eg_status host_graph_width(eg_ctx *c, bool want64) {
    const int64_t nm = c->n_max, ns = c->n_sad, na = c->n_arc;
    if (want64 && !c->h64_valid) {
        CK(c->h_maxima.ensure(sizeof(int64_t) * std::max<int64_t>(nm, 1)));
        CK(c->h_saddles.ensure(sizeof(int64_t) * std::max<int64_t>(ns, 1)));
        CK(c->h_arc_s.ensure(sizeof(int64_t) * std::max<int64_t>(na, 1)));
        CK(c->h_arc_m.ensure(sizeof(int64_t) * std::max<int64_t>(na, 1)));
        for (int64_t i = 0; i < nm; ++i) c->h_maxima.as<int64_t>()[i] = c->h32_maxima.as<int32_t>()[i];
        for (int64_t i = 0; i < ns; ++i) c->h_saddles.as<int64_t>()[i] = c->h32_saddles.as<int32_t>()[i];
        for (int64_t i = 0; i < na; ++i) {
            c->h_arc_s.as<int64_t>()[i] = c->h32_arc_s.as<int32_t>()[i];
            c->h_arc_m.as<int64_t>()[i] = c->h32_arc_m.as<int32_t>()[i];
        }
        c->h64_valid = true;
    }
    if (!want64 && !c->h32_valid) {
        CK(c->h32_maxima.ensure(sizeof(int32_t) * std::max<int64_t>(nm, 1)));
        CK(c->h32_saddles.ensure(sizeof(int32_t) * std::max<int64_t>(ns, 1)));
        CK(c->h32_arc_s.ensure(sizeof(int32_t) * std::max<int64_t>(na, 1)));
        CK(c->h32_arc_m.ensure(sizeof(int32_t) * std::max<int64_t>(na, 1)));
        for (int64_t i = 0; i < nm; ++i) c->h32_maxima.as<int32_t>()[i] = int32_t(c->h_maxima.as<int64_t>()[i]);
        for (int64_t i = 0; i < ns; ++i) c->h32_saddles.as<int32_t>()[i] = int32_t(c->h_saddles.as<int64_t>()[i]);
        for (int64_t i = 0; i < na; ++i) {
            c->h32_arc_s.as<int32_t>()[i] = int32_t(c->h_arc_s.as<int64_t>()[i]);
            c->h32_arc_m.as<int32_t>()[i] = int32_t(c->h_arc_m.as<int64_t>()[i]);
        }
        c->h32_valid = true;
    }
    return EG_OK;
}

// EG_NO_GRAPH_D2H on one process: the first host request copies the graph
static eg_status fetch_deferred_graph(eg_ctx *c) {
    if (!c->have_graph || c->graph_on_host || !c->graph_deferred) return EG_OK;
    ST(gather_graph(c, c->deferred_raw));
    CK(cudaStreamSynchronize(c->gstream));
    CK(cudaStreamSynchronize(c->stream));
    c->graph_on_host = true;
    return EG_OK;
}

eg_status eg_get_graph32(eg_ctx *c, eg_graph32 *out) {
    if (!c || !out) return EG_ERR_INVALID_ARG;
    if (c->poisoned) return set_err(c, EG_ERR_STATE, "context is poisoned: %s", c->err.c_str());
    ST(fetch_deferred_graph(c));
    if (!c->have_graph || !c->graph_on_host) return set_err(c, EG_ERR_STATE, "no graph on the host (call eg_compute)");
    ST(host_graph_width(c, false));
    out->n_max = c->n_max;
    out->n_saddle = c->n_sad;
    out->n_arc = c->n_arc;
    out->maxima = c->h32_maxima.as<int32_t>();
    out->saddles = c->h32_saddles.as<int32_t>();
    out->saddle_beta = c->h_sbeta.as<int32_t>();
    out->arc_saddle = c->h32_arc_s.as<int32_t>();
    out->arc_max = c->h32_arc_m.as<int32_t>();
    out->arc_mult = c->h_arc_mult.as<int32_t>();
    return EG_OK;
}

eg_status eg_get_graph(eg_ctx *c, eg_graph *out) {
    if (!c || !out) return EG_ERR_INVALID_ARG;
    if (c->poisoned) return set_err(c, EG_ERR_STATE, "context is poisoned: %s", c->err.c_str());
    ST(fetch_deferred_graph(c));
    if (!c->have_graph || !c->graph_on_host) return set_err(c, EG_ERR_STATE, "no graph on the host (call eg_compute)");
    ST(host_graph_width(c, true));
    out->n_max = c->n_max;
    out->n_saddle = c->n_sad;
    out->n_arc = c->n_arc;
    out->maxima = c->h_maxima.as<int64_t>();
    out->saddles = c->h_saddles.as<int64_t>();
    out->saddle_beta = c->h_sbeta.as<int32_t>();
    out->arc_saddle = c->h_arc_s.as<int64_t>();
    out->arc_max = c->h_arc_m.as<int64_t>();
    out->arc_mult = c->h_arc_mult.as<int32_t>();
    return EG_OK;
}

eg_status eg_get_raw_arcs(eg_ctx *c, int64_t *n, const int64_t **s, const int64_t **rep, const int64_t **m) {
    if (!c || !n || !s || !rep || !m) return EG_ERR_INVALID_ARG;
    ST(fetch_deferred_graph(c));
    if (!c->have_graph || !c->raw_valid || !c->graph_on_host)
        return set_err(c, EG_ERR_STATE, "raw arcs need eg_compute with EG_RAW_ARCS");
    *n = c->n_raw;
    *s = c->h_raw_s.as<int64_t>();
    *rep = c->h_raw_rep.as<int64_t>();
    *m = c->h_raw_m.as<int64_t>();
    return EG_OK;
}

eg_status eg_simplify(eg_ctx *c, double tau, eg_graph *out) {
    if (!c || !out) return EG_ERR_INVALID_ARG;
    if (!c->have_graph || !c->graph_on_host || !c->node_values)
        return set_err(c, EG_ERR_STATE, "eg_simplify needs the last eg_compute with EG_NODE_VALUES (one process)");
    simplify_graph(c->n_max, c->h_maxima.as<int64_t>(), c->h_fmax.as<float>(), c->n_sad, c->h_saddles.as<int64_t>(),
                   c->h_sbeta.as<int32_t>(), c->h_fsad.as<float>(), c->n_arc, c->h_arc_s.as<int64_t>(),
                   c->h_arc_m.as<int64_t>(), c->h_arc_mult.as<int32_t>(), tau, c->last_minimum, c->simp);
    out->n_max = int64_t(c->simp.maxima.size());
    out->n_saddle = int64_t(c->simp.saddles.size());
    out->n_arc = int64_t(c->simp.arc_s.size());
    out->maxima = c->simp.maxima.data();
    out->saddles = c->simp.saddles.data();
    out->saddle_beta = c->simp.saddle_beta.data();
    out->arc_saddle = c->simp.arc_s.data();
    out->arc_max = c->simp.arc_m.data();
    out->arc_mult = c->simp.arc_mult.data();
    return EG_OK;
}

eg_status eg_get_arc_paths(eg_ctx *c, int64_t *n, const int64_t **offsets, const int64_t **vertices) {
    if (!c || !n || !offsets || !vertices) return EG_ERR_INVALID_ARG;
    if (!c->have_graph || !c->paths_valid) return set_err(c, EG_ERR_STATE, "arc paths need eg_compute with EG_ARC_PATHS");
    ST(fetch_paths(c));
    *n = c->n_paths;
    *offsets = c->h_path_off.as<int64_t>();
    *vertices = c->h_path_v.as<int64_t>();
    return EG_OK;
}

eg_status eg_get_labels(eg_ctx *c, const int32_t **d_labels, int64_t *n) {
    if (!c || !d_labels || !n) return EG_ERR_INVALID_ARG;
    if (!c->have_labels) return set_err(c, EG_ERR_STATE, "no labels (call eg_compute)");
    *d_labels = c->d_labels;
    *n = c->n_own;
    return EG_OK;
}

eg_status eg_get_stats(eg_ctx *c, eg_stats *out) {
    if (!c || !out) return EG_ERR_INVALID_ARG;
    *out = c->stats;
    return EG_OK;
}

eg_status eg_destroy(eg_ctx *c) {
    if (!c) return EG_OK;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    set_slab_count(c, 0);
    DevBuf *bufs[] = {&c->typed, &c->rank_scratch, &c->d_fnode, &c->bund_scratch, &c->b_sad64, &c->b_sad32, &c->b_sbeta, &c->b_nu, &c->b_arc_s, &c->b_arc_m,
                      &c->b_arc_mult, &c->label_all, &c->csr_scratch, &c->fix_dev, &c->stat_buf, &c->field, &c->mirror, &c->path_len, &c->path_off, &c->path_v, &c->flags, &c->counts, &c->scratch, &c->tab, &c->gsend, &c->grecv};
    for (DevBuf *b : bufs) b->release();
    HostBuf *hb[] = {&c->h32_maxima, &c->h32_saddles, &c->h32_arc_s, &c->h32_arc_m,
                     &c->h_fmax, &c->h_fsad, &c->h_maxima, &c->h_saddles, &c->h_sbeta, &c->h_arc_s, &c->h_arc_m, &c->h_arc_mult,
                     &c->h_raw_s, &c->h_raw_rep, &c->h_raw_m, &c->h_counts, &c->h_stage, &c->h_path_off,
                     &c->h_path_v};
    for (HostBuf *b : hb) b->release();
    for (auto &e : c->ev)
        if (e) cudaEventDestroy(e);
    for (auto &e : c->ev_s2)
        if (e) cudaEventDestroy(e);
    for (auto &e : c->ev_main)
        if (e) cudaEventDestroy(e);
    if (c->d2h) {
        cudaStreamSynchronize(c->d2h);
        cudaStreamDestroy(c->d2h);
    }
    for (cudaStream_t *sp : {&c->cst, &c->h2d, &c->ld2h, &c->fst})
        if (*sp) {
            cudaStreamSynchronize(*sp);
            cudaStreamDestroy(*sp);
        }
    for (auto &e : c->ev_halo)
        if (e) cudaEventDestroy(e);
    if (c->aux) {
        cudaStreamSynchronize(c->aux);
        cudaStreamDestroy(c->aux);
    }
    if (c->ev_tile) cudaEventDestroy(c->ev_tile);
    if (c->ev_graph) cudaEventDestroy(c->ev_graph);
    for (auto &e : c->ev_d2h)
        if (e) cudaEventDestroy(e);
    if (c->comm) ncclCommDestroy(c->comm);
    delete c;
    return EG_OK;
}

const char *eg_last_error(const eg_ctx *c) {
    if (!c) return "null context";
    return c->err.c_str();
}

}  // extern "C"
