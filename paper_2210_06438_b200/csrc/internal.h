// internal.h — entry points shared between the library's translation units
// that are not part of the public C ABI (include/taskfuse_b200.h).
#pragma once

#include <cuda.h>
#include <stdint.h>

extern "C" {
// The 4-D tensor map (slice, x, y, z) of a sub-grid pool with the minmod
// stencil box (hydro_kernels.cu pool_map, cached per pool pointer).
int tf_internal_pool_map(const double* pool, int64_t slices, int n,
                         CUtensorMap* out);
}
