// Tiled 3-D path (n <= 3 grids on one GPU): see k_grid3d.cu.
#pragma once
#include <string>

#include "eg_impl.h"

namespace eg {
struct Tiled3D;
Tiled3D *tiled3d_create();
void tiled3d_destroy(Tiled3D *t);
// S1 + S2 + S3 for a whole n <= 3 grid: labels (int32, every vertex),
// saddle / maximum bitmaps over all vertices, NaN flag in flags[0];
// exit_bits: scratch bitmap of N bits.
eg_status tiled3d_labels(Tiled3D *t, int ndim, const int64_t *dims, const float *f, int32_t *labels,
                         uint32_t *sad_bits, uint32_t *max_bits, int *flags, cudaStream_t st, eg_stats *stats,
                         std::string *err, uint32_t *exit_bits);
}  // namespace eg
