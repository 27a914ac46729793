// Fused HASF kernel variant: foreground adjacency 8, generic (shared or global) planes.
#include "ts_hasf_impl.cuh"

namespace ts {
TS_DEFINE_HASF_VARIANT(8, false, 8g)
}  // namespace ts
