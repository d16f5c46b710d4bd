// Tiled path for n <= 3 grids: see k_grid3d.cu.
#pragma once
#include <string>

#include "eg_impl.h"

namespace eg {
struct Tiled3D;
constexpr int kTileY = 16, kTileZ = 16;   // tile rows / planes of k_tile (k_grid3d.cu: TY, TZ)

// End-to-end pipeline of eg_compute_host on one slab of one GPU (k_grid3d.cu):
// the field arrives in z-chunks on stream h2d; tile chunk k starts when chunk
// k + 1 (its halo plane) has arrived; label chunk k (stream fst) when tile
// chunk k + 1 is done; its labels leave on stream d2h while later chunks of
// the field are still arriving.  done = false if the schedule could not be
// used (the field is then fully copied first and the caller copies the labels).
struct ChunkIO {
    int K = 8;                        // chunks (z-layer ranges of tiles)
    cudaStream_t h2d = nullptr, d2h = nullptr, fst = nullptr;
    const float *h_field = nullptr;   // pinned host field (owned planes)
    float *d_field = nullptr;         // its device copy
    int32_t *h_labels = nullptr;      // pinned host labels, or null
    bool done = false;                // the chunked schedule ran (labels + list patch pending)
    cudaEvent_t fin_done = nullptr;   // (done) on fst: every owned label is final
    cudaEvent_t d2h_done = nullptr;   // (done) on d2h: every label chunk copied
};
Tiled3D *tiled3d_create();
void tiled3d_destroy(Tiled3D *t);
// S1 + S3 and the slab-local part of S2 for the owned planes of slab `s` of an
// n <= 3 grid: labels (owned, index v - s.v0) final or kUnresolved | x (see
// eg_impl.h), the maxima and saddles of the owned vertices (kept in `t`, see
// tiled3d_lists), NaN flag in flags[0].  Exiting vertices still point at
// their exit target: the caller finishes them with launch_finalize (after the
// boundary exchange when there are several slabs).
eg_status tiled3d_local(Tiled3D *t, int ndim, const int64_t *dims, const Slab &s, const FieldView &F, int32_t *labels,
                        int *flags, cudaStream_t st, eg_stats *stats, std::string *err,
                        cudaEvent_t ev_main0 = nullptr, cudaEvent_t ev_main1 = nullptr,
                        unsigned long long *exit_count = nullptr,   // EG_STATS: += exiting vertices
                        cudaEvent_t halo_ready = nullptr,            // halo planes arrive after this event
                        ChunkIO *io = nullptr);                       // eg_compute_host pipeline (one slab)
// the vertices whose labels the chunked label pass finished last (after their
// chunk had been copied to the host): device list, device count, capacity
void tiled3d_fin_list(const Tiled3D *t, const int32_t **list, const unsigned long long **count, int64_t *cap);
// number of maxima (which = 0) / saddles (which = 1) found by the last tiled3d_local
int64_t tiled3d_count(const Tiled3D *t, int which);
// the maxima (int64) and saddles (int32 and int64) of the last tiled3d_local,
// ascending; outputs sized by tiled3d_count
eg_status tiled3d_lists(Tiled3D *t, int64_t *max64, int32_t *sad32, int64_t *sad64, cudaStream_t st,
                        eg_stats *stats, std::string *err);
}  // namespace eg
