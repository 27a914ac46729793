// Fused HASF kernel variant: foreground adjacency 8, hot planes in shared memory,
// 256 threads per CTA, two CTAs (images) per SM (small images).
#define TS_IMPL_THREADS 256
#define TS_IMPL_MINB 2
#define TS_IMPL_NS v256
#define TS_IMPL_E4 1   // 4 precedence planes (antisymmetry), see ts_hasf_impl.cuh
#define TS_DENSE_BATCH 1   // measured: c4 2.79 -> 2.74 ms (E in shared memory: no latency to batch)
#include "ts_hasf_impl.cuh"

namespace ts {
TS_DEFINE_HASF_VARIANT(8, true, 8h256)
}  // namespace ts
