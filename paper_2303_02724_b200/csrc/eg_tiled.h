// Tiled path for n <= 3 grids: see k_grid3d.cu.
#pragma once
#include <string>

#include "eg_impl.h"

namespace eg {
struct Tiled3D;
Tiled3D *tiled3d_create();
void tiled3d_destroy(Tiled3D *t);
// S1 + S3 and the slab-local part of S2 for the owned planes of slab `s` of an
// n <= 3 grid: labels (owned, index v - s.v0) final or kUnresolved | x (see
// eg_impl.h), saddle / maximum / exit bitmaps over the owned vertices, NaN
// flag in flags[0].  Exiting vertices still point at their exit target: the
// caller finishes them with launch_finalize (after the boundary exchange when
// there are several slabs).
eg_status tiled3d_local(Tiled3D *t, int ndim, const int64_t *dims, const Slab &s, const FieldView &F, int32_t *labels,
                        uint32_t *sad_bits, uint32_t *max_bits, uint32_t *exit_bits, int *flags, cudaStream_t st,
                        eg_stats *stats, std::string *err, cudaEvent_t ev_main0 = nullptr,
                        cudaEvent_t ev_main1 = nullptr);
}  // namespace eg
