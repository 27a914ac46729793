// Fused HASF kernel variant: foreground adjacency 4, generic (shared or global) planes.
#include "ts_hasf_impl.cuh"

namespace ts {
TS_DEFINE_HASF_VARIANT(4, false, 4g)
}  // namespace ts
