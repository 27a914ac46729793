// Fused HASF kernel variant: foreground adjacency 4, hot planes in shared memory.
#ifndef TS_BIG_THREADS
#define TS_BIG_THREADS 512
#endif
#define TS_IMPL_THREADS TS_BIG_THREADS
#define TS_IMPL_MINB 1
#define TS_IMPL_NS v512
#ifdef TS_IMPL_E4_HOT
#define TS_IMPL_E4 1   // A-B experiment: 4 precedence planes in the 512-thread hot variant too
#endif
#ifndef TS_DENSE_PREFETCH
#define TS_DENSE_PREFETCH 1   // E masks (L2) of the next row requested before the current row is evaluated
#endif
#include "ts_hasf_impl.cuh"

namespace ts {
TS_DEFINE_HASF_VARIANT(4, true, 4h)
}  // namespace ts
