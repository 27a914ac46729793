// Fused HASF kernel variant: foreground adjacency 4, hot planes in shared memory.
#include "ts_hasf_impl.cuh"

namespace ts {
TS_DEFINE_HASF_VARIANT(4, true, 4h)
}  // namespace ts
