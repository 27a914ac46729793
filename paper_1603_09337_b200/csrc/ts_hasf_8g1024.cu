// Fused HASF kernel variant: foreground adjacency 8, planes in global memory (L2),
// TS_WIDE_THREADS (768) threads per CTA: the cluster teams of large images are
// bound by L2 / DRAM latency, more warps per SM hide more of it while 80
// registers still hold the strip walk (see ts_internal.h for the measurements).
#include "ts_internal.h"
#define TS_IMPL_THREADS TS_WIDE_THREADS
#define TS_IMPL_MINB 1
#define TS_IMPL_NS v1024
#ifndef TS_WIDE_PIPE
#define TS_WIDE_PIPE 0
#endif
#define TS_DENSE_PIPE TS_WIDE_PIPE   // the pipelined strip walk measured slower here (c2 35.1 vs 37.0 ms)
#define TS_IMPL_E4 1   // 4 precedence planes (antisymmetry), see ts_hasf_impl.cuh
#include "ts_hasf_impl.cuh"

namespace ts {
TS_DEFINE_HASF_VARIANT(8, false, 8g1024)
}  // namespace ts
