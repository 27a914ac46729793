// Fused HASF kernel variant: foreground adjacency 8, planes in global memory (L2),
// 1024 threads per CTA (64 registers): the cluster teams of large images are
// bound by L2 / DRAM latency, twice the warps per SM hide more of it
// (c2: 45.8 -> 38.1 ms against the 512-thread variant).
#define TS_IMPL_THREADS 1024
#define TS_IMPL_MINB 1
#define TS_IMPL_NS v1024
#define TS_IMPL_E4 1   // 4 precedence planes (antisymmetry), see ts_hasf_impl.cuh
#include "ts_hasf_impl.cuh"

namespace ts {
TS_DEFINE_HASF_VARIANT(8, false, 8g1024)
}  // namespace ts
