// Fused HASF kernel variant: foreground adjacency 4, generic (shared or global) planes.
#ifndef TS_BIG_THREADS
#define TS_BIG_THREADS 512
#endif
#define TS_IMPL_THREADS TS_BIG_THREADS
#define TS_IMPL_MINB 1
#define TS_IMPL_NS v512
#define TS_IMPL_E4 1   // 4 precedence planes (antisymmetry), see ts_hasf_impl.cuh
#include "ts_hasf_impl.cuh"

namespace ts {
TS_DEFINE_HASF_VARIANT(4, false, 4g)
}  // namespace ts
