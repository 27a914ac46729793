// Fused HASF kernel variant: foreground adjacency 8, hot planes in shared memory.
#include "ts_hasf_impl.cuh"

namespace ts {
TS_DEFINE_HASF_VARIANT(8, true, 8h)
}  // namespace ts
