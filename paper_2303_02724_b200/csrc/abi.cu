// C ABI (include/eg.h) and the host-side orchestration of one eg_compute.
//
// Stage order per compute:
//   classify (S1 + S3) -> pointer jumping (S2) -> compaction of maxima and
//   saddles -> per-saddle beta0+ / arcs (S4) -> graph to host.
// The field stays resident in HBM; the only host<->device crossings are the
// counts needed to size outputs and the final (small) graph.
#include <cuda_runtime.h>

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

}  // namespace

struct eg_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool poisoned = false;
    std::string err;
    int rank = 0, world = 1;
    void *nccl = nullptr;

    // device working set
    DevBuf field;                  // eg_compute_host staging target
    DevBuf ptr;                    // int32 per owned vertex: gradient, then label
    DevBuf sad_bits, max_bits;     // one bit per owned vertex
    DevBuf exit_bits;              // tiled path: vertices whose path leaves their tile
    DevBuf flags;                  // [0] nan, [1] deg overflow, [2..] jump-changed per round
    DevBuf scratch;                // compaction / scan scratch
    DevBuf counts;                 // int64 counters
    DevBuf maxima64, saddles32, saddles64, sbeta, slot_off, tmp_m, tmp_mult, n_unique, arc_off;
    DevBuf arc_s, arc_m, arc_mult, raw_s, raw_rep, raw_m;
    DevBuf tab;                    // LinkTable
    DevBuf halo_label;
    LinkTable host_tab;
    bool tab_valid = false;
    eg::Tiled3D *tiled = nullptr;

    // host outputs
    HostBuf h_maxima, h_saddles, h_sbeta, h_arc_s, h_arc_m, h_arc_mult, h_raw_s, h_raw_rep, h_raw_m, h_counts;
    HostBuf h_stage;
    int64_t n_max = 0, n_sad = 0, n_arc = 0, n_raw = 0, n_own = 0;
    bool have_graph = false, have_labels = false, graph_on_host = false, raw_valid = false;
    const int32_t *d_labels = nullptr;
    eg_stats stats{};
    cudaEvent_t ev[8] = {};
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

// ------------------------------------------------------------- validation

struct Problem {
    bool grid;
    int ndim;
    int64_t dims[8];
    int64_t N;             // total vertices
    Slab slab;             // grid
    int64_t v0, v1;        // owned range (both kinds)
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
        const int64_t plane = N / D;
        int64_t z0 = g.slab_begin, z1 = g.slab_end;
        if (c->world == 1 && z0 == 0 && z1 == 0) z1 = D;   // convenience: 0,0 = whole grid
        if (z0 < 0 || z1 > D || z0 >= z1) return set_err(c, EG_ERR_INVALID_ARG, "bad slab [%lld, %lld)", (long long)z0, (long long)z1);
        if (c->world == 1 && (z0 != 0 || z1 != D))
            return set_err(c, EG_ERR_INVALID_ARG, "single-GPU ctx needs the whole grid as its slab");
        P->grid = true;
        P->ndim = g.ndim;
        for (int i = 0; i < g.ndim; ++i) P->dims[i] = g.dims[i];
        P->N = N;
        P->slab.z0 = z0;
        P->slab.z1 = z1;
        P->slab.h0 = z0 > 0 ? z0 - 1 : 0;
        P->slab.h1 = z1 < D ? z1 + 1 : D;
        P->slab.plane = plane;
        P->slab.v0 = z0 * plane;
        P->slab.v1 = z1 * plane;
        P->slab.base = P->slab.h0 * plane;
        P->v0 = P->slab.v0;
        P->v1 = P->slab.v1;
    } else if (d->kind == EG_DOMAIN_CSR) {
        const eg_csr &g = d->csr;
        if (g.n_vertices < 0 || g.nnz < 0) return set_err(c, EG_ERR_INVALID_ARG, "negative CSR sizes");
        if (g.n_vertices >= (int64_t(1) << 31)) return set_err(c, EG_ERR_UNSUPPORTED, "N >= 2^31");
        int64_t v0 = g.v_begin, v1 = g.v_end;
        if (c->world == 1 && v0 == 0 && v1 == 0) v1 = g.n_vertices;
        if (v0 < 0 || v1 > g.n_vertices || v0 > v1) return set_err(c, EG_ERR_INVALID_ARG, "bad vertex range");
        if (g.n_vertices > 0 && (!is_device_ptr(g.row_ptr) || (g.nnz > 0 && !is_device_ptr(g.col_idx))))
            return set_err(c, EG_ERR_INVALID_ARG, "row_ptr / col_idx must be device pointers");
        P->grid = false;
        P->N = g.n_vertices;
        P->v0 = v0;
        P->v1 = v1;
        P->row_ptr = g.row_ptr;
        P->col_idx = g.col_idx;
    } else {
        return set_err(c, EG_ERR_INVALID_ARG, "unknown domain kind %d", d->kind);
    }
    if (P->N > 0 && need_device && !is_device_ptr(field))
        return set_err(c, EG_ERR_INVALID_ARG, "field must be a device pointer");
    if (P->N > 0 && !field) return set_err(c, EG_ERR_INVALID_ARG, "field is NULL");
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
    return ms * 1000.f;
}

// -------------------------------------------------------------- pipeline

// S1 + S3 + S2 on the generic path: leaves labels in c->ptr (int32, owned).
static eg_status run_generic_labels(eg_ctx *c, const Problem &P, const float *f) {
    const int64_t n = P.v1 - P.v0;
    const int64_t words = (n + 31) / 32;
    int *flags = c->flags.as<int>();
    if (P.grid) {
        CK(launch_classify_grid(c->tab.as<LinkTable>(), P.ndim, f, P.slab, c->ptr.as<int32_t>(),
                                c->sad_bits.as<uint32_t>(), c->max_bits.as<uint32_t>(), nullptr, flags, c->stream));
    } else {
        CK(launch_classify_csr(P.row_ptr, P.col_idx, f, P.v0, P.v1, c->ptr.as<int32_t>(), c->sad_bits.as<uint32_t>(),
                               c->max_bits.as<uint32_t>(), nullptr, flags, flags + 1, c->stream));
    }
    c->stats.kernel_launches += 1;
    (void)words;
    CK(cudaEventRecord(c->ev[1], c->stream));
    // S2: rounds are launched in batches; a round whose predecessor changed
    // nothing exits at once, so only the flag read-back costs a sync.
    int *changed = flags + 2;
    int rounds = 0;
    const int kBatch = 6;
    std::vector<int> hflag(64);
    for (int r0 = 0; r0 < 62; r0 += kBatch) {
        int r1 = std::min(62, r0 + kBatch);
        for (int r = r0; r < r1; ++r) {
            CK(launch_jump_round(c->ptr.as<int32_t>(), n, P.v0, changed, r, c->stream));
            c->stats.kernel_launches += 1;
        }
        CK(cudaMemcpyAsync(hflag.data(), changed, sizeof(int) * r1, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        int first_zero = -1;
        for (int r = 0; r < r1; ++r)
            if (hflag[r] == 0) {
                first_zero = r;
                break;
            }
        if (first_zero >= 0) {
            rounds = first_zero + 1;
            break;
        }
        rounds = r1;
    }
    c->stats.jump_rounds = rounds;
    return EG_OK;
}

static eg_status fail_if_flags(eg_ctx *c) {
    int h[2] = {0, 0};
    CK(cudaMemcpyAsync(h, c->flags.p, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (h[0]) return set_err(c, EG_ERR_NAN, "NaN in the scalar field (reading L2)");
    if (h[1]) return set_err(c, EG_ERR_UNSUPPORTED, "CSR vertex degree > %d", kCsrMaxDeg);
    return EG_OK;
}

// Node lists, beta0+, arcs (S3 lists + S4) for the owned range; labels in c->ptr.
static eg_status run_graph(eg_ctx *c, const Problem &P, const float *f, uint32_t flags) {
    const int64_t n = P.v1 - P.v0;
    int64_t *cnt = c->counts.as<int64_t>();
    CK(c->scratch.ensure(std::max(compact_scratch_bytes(std::max<int64_t>(n, 1)), size_t(1) << 16)));
    // maxima (ascending, int64 for the host) and saddles (int32 for the kernels)
    CK(c->maxima64.ensure(sizeof(int64_t) * 1));
    // counts first (exact sizes): two cheap compaction passes
    // pass 1: count only (out pointers null)
    CK(launch_compact_bits(c->max_bits.as<uint32_t>(), n, P.v0, c->scratch.p, nullptr, nullptr, cnt + 0, c->stream));
    CK(launch_compact_bits(c->sad_bits.as<uint32_t>(), n, P.v0, c->scratch.p, nullptr, nullptr, cnt + 1, c->stream));
    c->stats.kernel_launches += 6;
    CK(c->h_counts.ensure(sizeof(int64_t) * 8));
    int64_t *hc = c->h_counts.as<int64_t>();
    CK(cudaMemcpyAsync(hc, cnt, sizeof(int64_t) * 2, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    c->n_max = hc[0];
    c->n_sad = hc[1];
    CK(c->maxima64.ensure(sizeof(int64_t) * std::max<int64_t>(c->n_max, 1)));
    CK(c->saddles32.ensure(sizeof(int32_t) * std::max<int64_t>(c->n_sad, 1)));
    CK(c->saddles64.ensure(sizeof(int64_t) * std::max<int64_t>(c->n_sad, 1)));
    CK(launch_compact_bits(c->max_bits.as<uint32_t>(), n, P.v0, c->scratch.p, nullptr, c->maxima64.as<int64_t>(),
                           cnt + 0, c->stream));
    CK(launch_compact_bits(c->sad_bits.as<uint32_t>(), n, P.v0, c->scratch.p, c->saddles32.as<int32_t>(),
                           c->saddles64.as<int64_t>(), cnt + 1, c->stream));
    c->stats.kernel_launches += 6;
    CK(cudaEventRecord(c->ev[3], c->stream));

    // beta0+ per saddle and slot offsets (sum beta = raw arcs)
    const int64_t ns = c->n_sad;
    CK(c->sbeta.ensure(sizeof(int32_t) * std::max<int64_t>(ns, 1)));
    CK(c->slot_off.ensure(sizeof(int64_t) * (ns + 1)));
    CK(c->arc_off.ensure(sizeof(int64_t) * (ns + 1)));
    CK(c->n_unique.ensure(sizeof(int32_t) * std::max<int64_t>(ns, 1)));
    size_t sb = scan_scratch_bytes(std::max<int64_t>(ns, 1));
    CK(c->scratch.ensure(sb));
    if (P.grid)
        CK(launch_saddle_beta_grid(c->tab.as<LinkTable>(), P.ndim, f, P.slab, c->saddles32.as<int32_t>(), ns,
                                   c->sbeta.as<int32_t>(), c->stream));
    else
        CK(launch_saddle_beta_csr(P.row_ptr, P.col_idx, f, c->saddles32.as<int32_t>(), ns, c->sbeta.as<int32_t>(),
                                  c->stream));
    CK(launch_scan_i32(c->sbeta.as<int32_t>(), c->slot_off.as<int64_t>(), ns, c->scratch.p, sb, c->stream));
    c->stats.kernel_launches += 2;
    CK(cudaMemcpyAsync(hc, c->slot_off.as<int64_t>() + ns, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    const int64_t nraw = hc[0];
    c->n_raw = nraw;
    CK(c->tmp_m.ensure(sizeof(int32_t) * std::max<int64_t>(nraw, 1)));
    CK(c->tmp_mult.ensure(sizeof(int32_t) * std::max<int64_t>(nraw, 1)));
    const bool raw = (flags & EG_RAW_ARCS) != 0;
    if (raw) {
        CK(c->raw_s.ensure(sizeof(int64_t) * std::max<int64_t>(nraw, 1)));
        CK(c->raw_rep.ensure(sizeof(int64_t) * std::max<int64_t>(nraw, 1)));
        CK(c->raw_m.ensure(sizeof(int64_t) * std::max<int64_t>(nraw, 1)));
    }
    LabelView lv{};
    lv.own = c->d_labels;
    lv.v0 = P.v0;
    lv.v1 = P.v1;
    lv.halo = c->halo_label.as<int32_t>();
    if (P.grid) {
        lv.plane = P.slab.plane;
        lv.lo_base = P.slab.z0 > 0 ? (P.slab.z0 - 1) * P.slab.plane : -1;
        lv.hi_base = P.slab.z1 < P.dims[P.ndim - 1] ? P.slab.z1 * P.slab.plane : -1;
        CK(launch_arcs_grid(c->tab.as<LinkTable>(), P.ndim, f, P.slab, c->saddles32.as<int32_t>(), ns,
                            c->slot_off.as<int64_t>(), lv, c->tmp_m.as<int32_t>(), c->tmp_mult.as<int32_t>(),
                            c->n_unique.as<int32_t>(), raw ? c->raw_s.as<int64_t>() : nullptr,
                            raw ? c->raw_rep.as<int64_t>() : nullptr, raw ? c->raw_m.as<int64_t>() : nullptr,
                            c->stream));
    } else {
        CK(launch_arcs_csr(P.row_ptr, P.col_idx, f, c->saddles32.as<int32_t>(), ns, c->slot_off.as<int64_t>(), lv,
                           c->tmp_m.as<int32_t>(), c->tmp_mult.as<int32_t>(), c->n_unique.as<int32_t>(),
                           raw ? c->raw_s.as<int64_t>() : nullptr, raw ? c->raw_rep.as<int64_t>() : nullptr,
                           raw ? c->raw_m.as<int64_t>() : nullptr, c->stream));
    }
    CK(launch_scan_i32(c->n_unique.as<int32_t>(), c->arc_off.as<int64_t>(), ns, c->scratch.p, sb, c->stream));
    c->stats.kernel_launches += 2;
    CK(cudaMemcpyAsync(hc, c->arc_off.as<int64_t>() + ns, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    c->n_arc = hc[0];
    CK(c->arc_s.ensure(sizeof(int64_t) * std::max<int64_t>(c->n_arc, 1)));
    CK(c->arc_m.ensure(sizeof(int64_t) * std::max<int64_t>(c->n_arc, 1)));
    CK(c->arc_mult.ensure(sizeof(int32_t) * std::max<int64_t>(c->n_arc, 1)));
    CK(launch_emit_arcs(c->saddles32.as<int32_t>(), ns, c->slot_off.as<int64_t>(), c->arc_off.as<int64_t>(),
                        c->tmp_m.as<int32_t>(), c->tmp_mult.as<int32_t>(), c->n_unique.as<int32_t>(),
                        c->arc_s.as<int64_t>(), c->arc_m.as<int64_t>(), c->arc_mult.as<int32_t>(), c->stream));
    c->stats.kernel_launches += 1;
    CK(cudaEventRecord(c->ev[4], c->stream));
    c->stats.n_raw_arcs = nraw;
    c->raw_valid = raw;
    return EG_OK;
}

static eg_status graph_to_host(eg_ctx *c, bool raw) {
    const int64_t nm = c->n_max, ns = c->n_sad, na = c->n_arc;
    CK(c->h_maxima.ensure(sizeof(int64_t) * std::max<int64_t>(nm, 1)));
    CK(c->h_saddles.ensure(sizeof(int64_t) * std::max<int64_t>(ns, 1)));
    CK(c->h_sbeta.ensure(sizeof(int32_t) * std::max<int64_t>(ns, 1)));
    CK(c->h_arc_s.ensure(sizeof(int64_t) * std::max<int64_t>(na, 1)));
    CK(c->h_arc_m.ensure(sizeof(int64_t) * std::max<int64_t>(na, 1)));
    CK(c->h_arc_mult.ensure(sizeof(int32_t) * std::max<int64_t>(na, 1)));
    cudaStream_t st = c->stream;
    if (nm) CK(cudaMemcpyAsync(c->h_maxima.p, c->maxima64.p, sizeof(int64_t) * nm, cudaMemcpyDeviceToHost, st));
    if (ns) {
        CK(cudaMemcpyAsync(c->h_saddles.p, c->saddles64.p, sizeof(int64_t) * ns, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(c->h_sbeta.p, c->sbeta.p, sizeof(int32_t) * ns, cudaMemcpyDeviceToHost, st));
    }
    if (na) {
        CK(cudaMemcpyAsync(c->h_arc_s.p, c->arc_s.p, sizeof(int64_t) * na, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(c->h_arc_m.p, c->arc_m.p, sizeof(int64_t) * na, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(c->h_arc_mult.p, c->arc_mult.p, sizeof(int32_t) * na, cudaMemcpyDeviceToHost, st));
    }
    if (raw) {
        const int64_t nr = c->n_raw;
        CK(c->h_raw_s.ensure(sizeof(int64_t) * std::max<int64_t>(nr, 1)));
        CK(c->h_raw_rep.ensure(sizeof(int64_t) * std::max<int64_t>(nr, 1)));
        CK(c->h_raw_m.ensure(sizeof(int64_t) * std::max<int64_t>(nr, 1)));
        if (nr) {
            CK(cudaMemcpyAsync(c->h_raw_s.p, c->raw_s.p, sizeof(int64_t) * nr, cudaMemcpyDeviceToHost, st));
            CK(cudaMemcpyAsync(c->h_raw_rep.p, c->raw_rep.p, sizeof(int64_t) * nr, cudaMemcpyDeviceToHost, st));
            CK(cudaMemcpyAsync(c->h_raw_m.p, c->raw_m.p, sizeof(int64_t) * nr, cudaMemcpyDeviceToHost, st));
        }
    }
    return EG_OK;
}

static eg_status compute_impl(eg_ctx *c, const eg_domain *d, const float *f, uint32_t flags, bool device_field) {
    if (!c) return EG_ERR_INVALID_ARG;
    if (c->poisoned) return set_err(c, EG_ERR_STATE, "context is poisoned by an earlier CUDA/NCCL error: %s", c->err.c_str());
    c->have_graph = c->have_labels = c->graph_on_host = false;
    Problem P;
    eg_status s = validate(c, d, f, device_field, &P);
    if (s != EG_OK) return s;
    CK(cudaSetDevice(c->device));
    std::memset(&c->stats, 0, sizeof(c->stats));
    c->stats.n_vertices = P.N;
    const int64_t n = P.v1 - P.v0;
    c->n_own = n;
    const int64_t words = (n + 31) / 32;
    CK(c->ptr.ensure(sizeof(int32_t) * std::max<int64_t>(n, 1)));
    CK(c->sad_bits.ensure(sizeof(uint32_t) * std::max<int64_t>(words, 1)));
    CK(c->max_bits.ensure(sizeof(uint32_t) * std::max<int64_t>(words, 1)));
    CK(c->flags.ensure(sizeof(int) * 128));
    CK(c->counts.ensure(sizeof(int64_t) * 16));
    CK(c->halo_label.ensure(sizeof(int32_t) * 2));
    CK(cudaMemsetAsync(c->flags.p, 0, sizeof(int) * 128, c->stream));
    if (P.grid) {
        s = ensure_table(c, P);
        if (s != EG_OK) return s;
    }
    CK(cudaEventRecord(c->ev[0], c->stream));

    const bool tiled = P.grid && P.ndim <= 3 && !(flags & EG_FORCE_GENERIC) && c->world == 1 && c->tiled != nullptr;
    if (tiled) {
        c->stats.path = 1;
        CK(c->exit_bits.ensure(sizeof(uint32_t) * std::max<int64_t>(words, 1)));
        s = tiled3d_labels(c->tiled, P.ndim, P.dims, f, c->ptr.as<int32_t>(), c->sad_bits.as<uint32_t>(),
                           c->max_bits.as<uint32_t>(), c->flags.as<int>(), c->stream, &c->stats, &c->err,
                           c->exit_bits.as<uint32_t>());
        if (s != EG_OK) {
            if (s == EG_ERR_CUDA) c->poisoned = true;
            return s;
        }
        CK(cudaEventRecord(c->ev[1], c->stream));
    } else {
        c->stats.path = P.grid ? 0 : 2;
        s = run_generic_labels(c, P, f);
        if (s != EG_OK) return s;
    }
    CK(cudaEventRecord(c->ev[2], c->stream));
    s = fail_if_flags(c);
    if (s != EG_OK) return s;
    c->d_labels = c->ptr.as<int32_t>();
    c->have_labels = true;

    s = run_graph(c, P, f, flags);
    if (s != EG_OK) return s;
    if (!(flags & EG_NO_GRAPH_D2H)) {
        s = graph_to_host(c, (flags & EG_RAW_ARCS) != 0);
        if (s != EG_OK) return s;
        c->graph_on_host = true;
    }
    CK(cudaEventRecord(c->ev[5], c->stream));
    CK(cudaStreamSynchronize(c->stream));
    c->have_graph = true;
    c->stats.us_classify = ev_us(c->ev[0], c->ev[1]);
    c->stats.us_jump = ev_us(c->ev[1], c->ev[2]);
    c->stats.us_label = 0;
    c->stats.us_arcs = ev_us(c->ev[2], c->ev[4]);
    c->stats.us_graph = ev_us(c->ev[4], c->ev[5]);
    c->stats.us_total = ev_us(c->ev[0], c->ev[5]);
    c->stats.bytes_alg = 8 * P.N + 4 * c->n_max + 5 * c->n_sad + 12 * c->n_arc +
                         (P.grid ? 0 : 8 * (P.N + 1) + 4 * (P.row_ptr ? d->csr.nnz : 0));
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
    c->tiled = tiled3d_create();
    *out = c;
    return EG_OK;
}

eg_status eg_compute(eg_ctx *c, const eg_domain *d, const float *d_field, uint32_t flags) {
    return compute_impl(c, d, d_field, flags, true);
}

eg_status eg_compute_host(eg_ctx *c, const eg_domain *d, const float *h_field, int32_t *h_labels, uint32_t flags) {
    if (!c) return EG_ERR_INVALID_ARG;
    if (c->poisoned) return set_err(c, EG_ERR_STATE, "context is poisoned: %s", c->err.c_str());
    Problem P;
    eg_status s = validate(c, d, h_field, false, &P);
    if (s != EG_OK) return s;
    if (is_device_ptr(h_field)) return set_err(c, EG_ERR_INVALID_ARG, "eg_compute_host takes a host field");
    CK(cudaSetDevice(c->device));
    int64_t nfield;
    if (P.grid) {
        nfield = (P.slab.z1 - P.slab.z0) * P.slab.plane;
    } else {
        nfield = P.N;
    }
    CK(c->field.ensure(sizeof(float) * std::max<int64_t>(nfield, 1)));
    cudaPointerAttributes a;
    bool pinned = cudaPointerGetAttributes(&a, h_field) == cudaSuccess && a.type == cudaMemoryTypeHost;
    cudaGetLastError();
    if (pinned || nfield * 4 <= (int64_t(1) << 20)) {
        CK(cudaMemcpyAsync(c->field.p, h_field, sizeof(float) * nfield, cudaMemcpyHostToDevice, c->stream));
    } else {
        const size_t chunk = size_t(64) << 20;
        CK(c->h_stage.ensure(2 * chunk));
        char *stage = c->h_stage.as<char>();
        const char *src = reinterpret_cast<const char *>(h_field);
        char *dst = c->field.as<char>();
        size_t total = sizeof(float) * size_t(nfield);
        int k = 0;
        for (size_t off = 0; off < total; off += chunk, k ^= 1) {
            size_t len = std::min(chunk, total - off);
            // the previous copy out of this half must be complete before reuse
            CK(cudaStreamSynchronize(c->stream));
            std::memcpy(stage + k * chunk, src + off, len);
            CK(cudaMemcpyAsync(dst + off, stage + k * chunk, len, cudaMemcpyHostToDevice, c->stream));
        }
    }
    if (!P.grid) {
        // CSR: the field copy above is the full replicated field
    }
    s = compute_impl(c, d, c->field.as<float>(), flags, true);
    if (s != EG_OK) return s;
    if (h_labels) {
        CK(cudaMemcpyAsync(h_labels, c->d_labels, sizeof(int32_t) * c->n_own, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    }
    return EG_OK;
}

eg_status eg_gradient(eg_ctx *c, const eg_domain *d, const float *d_field, int32_t *d_ptr, uint8_t *d_beta) {
    if (!c) return EG_ERR_INVALID_ARG;
    if (c->poisoned) return set_err(c, EG_ERR_STATE, "context is poisoned: %s", c->err.c_str());
    Problem P;
    eg_status s = validate(c, d, d_field, true, &P);
    if (s != EG_OK) return s;
    if (!is_device_ptr(d_ptr) || !is_device_ptr(d_beta))
        return set_err(c, EG_ERR_INVALID_ARG, "d_ptr / d_beta must be device pointers");
    CK(cudaSetDevice(c->device));
    const int64_t n = P.v1 - P.v0, words = (n + 31) / 32;
    CK(c->sad_bits.ensure(sizeof(uint32_t) * std::max<int64_t>(words, 1)));
    CK(c->max_bits.ensure(sizeof(uint32_t) * std::max<int64_t>(words, 1)));
    CK(c->flags.ensure(sizeof(int) * 128));
    CK(cudaMemsetAsync(c->flags.p, 0, sizeof(int) * 128, c->stream));
    if (P.grid) {
        s = ensure_table(c, P);
        if (s != EG_OK) return s;
        CK(launch_classify_grid(c->tab.as<LinkTable>(), P.ndim, d_field, P.slab, d_ptr, c->sad_bits.as<uint32_t>(),
                                c->max_bits.as<uint32_t>(), d_beta, c->flags.as<int>(), c->stream));
    } else {
        CK(launch_classify_csr(P.row_ptr, P.col_idx, d_field, P.v0, P.v1, d_ptr, c->sad_bits.as<uint32_t>(),
                               c->max_bits.as<uint32_t>(), d_beta, c->flags.as<int>(), c->flags.as<int>() + 1,
                               c->stream));
    }
    return fail_if_flags(c);
}

eg_status eg_get_graph(eg_ctx *c, eg_graph *out) {
    if (!c || !out) return EG_ERR_INVALID_ARG;
    if (c->poisoned) return set_err(c, EG_ERR_STATE, "context is poisoned: %s", c->err.c_str());
    if (!c->have_graph || !c->graph_on_host) return set_err(c, EG_ERR_STATE, "no graph on the host (call eg_compute)");
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
    if (!c->have_graph || !c->raw_valid || !c->graph_on_host)
        return set_err(c, EG_ERR_STATE, "raw arcs need eg_compute with EG_RAW_ARCS");
    *n = c->n_raw;
    *s = c->h_raw_s.as<int64_t>();
    *rep = c->h_raw_rep.as<int64_t>();
    *m = c->h_raw_m.as<int64_t>();
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
    DevBuf *bufs[] = {&c->field, &c->ptr, &c->sad_bits, &c->max_bits, &c->exit_bits, &c->flags, &c->scratch, &c->counts,
                      &c->maxima64, &c->saddles32, &c->saddles64, &c->sbeta, &c->slot_off, &c->tmp_m, &c->tmp_mult,
                      &c->n_unique, &c->arc_off, &c->arc_s, &c->arc_m, &c->arc_mult, &c->raw_s, &c->raw_rep,
                      &c->raw_m, &c->tab, &c->halo_label};
    for (DevBuf *b : bufs) b->release();
    HostBuf *hb[] = {&c->h_maxima, &c->h_saddles, &c->h_sbeta, &c->h_arc_s, &c->h_arc_m, &c->h_arc_mult,
                     &c->h_raw_s, &c->h_raw_rep, &c->h_raw_m, &c->h_counts, &c->h_stage};
    for (HostBuf *b : hb) b->release();
    for (auto &e : c->ev)
        if (e) cudaEventDestroy(e);
    tiled3d_destroy(c->tiled);
    delete c;
    return EG_OK;
}

const char *eg_last_error(const eg_ctx *c) {
    if (!c) return "null context";
    return c->err.c_str();
}

eg_status eg_nccl_unique_id(void *out128) {
    (void)out128;
    return EG_ERR_UNSUPPORTED;
}

eg_status eg_create_dist(eg_ctx **out, int cuda_device, void *cuda_stream, const void *nccl_id128, int rank,
                         int world) {
    (void)out; (void)cuda_device; (void)cuda_stream; (void)nccl_id128; (void)rank; (void)world;
    return EG_ERR_UNSUPPORTED;
}

}  // extern "C"
