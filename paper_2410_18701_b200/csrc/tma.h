// tma.h -- host-side TMA tensor-map encoding (cuTensorMapEncodeTiled through the
// runtime's driver entry point, so libbaton links only the CUDA runtime).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace baton {

// bf16 tensor of `rank` (2 to 5) dims, innermost first; strides in bytes for
// dims 1..rank-1; box sizes in elements.  SWIZZLE_128B.  False on failure.
bool encode_bf16_map(CUtensorMap *map, const void *base, int rank, const uint64_t *dims,
                     const uint64_t *strides_bytes, const uint32_t *box);

}  // namespace baton
