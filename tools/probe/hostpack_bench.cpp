// Host packing throughput probe (GPU box CPU): per-chunk calls vs one call.
//   g++ -O3 -fopenmp -I paper_1603_09337_b200/csrc tools/probe/hostpack_bench.cpp paper_1603_09337_b200/csrc/ts_hostpack.cpp -o /tmp/hpb && /tmp/hpb
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <omp.h>
#include "ts_hostpack.h"
using clk = std::chrono::steady_clock;
static double us(clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::micro>(b - a).count(); }
int main() {
    const int n = 256, h = 512, w = 512, ww = 16;
    std::vector<uint8_t> in((size_t)n * h * w), out((size_t)n * h * w);
    std::vector<uint32_t> bits((size_t)n * h * ww);
    for (size_t i = 0; i < in.size(); ++i) in[i] = (uint8_t)((i * 2654435761u >> 13) & 1);
    printf("omp threads %d\n", omp_get_max_threads());
    for (int chunk : {256, 64, 16, 8, 4}) {
        double best_p = 1e30, best_u = 1e30;
        for (int rep = 0; rep < 8; ++rep) {
            auto t0 = clk::now();
            for (int i = 0; i < n; i += chunk) ts::pack_images(in.data() + (size_t)i * h * w, bits.data() + (size_t)i * h * ww, chunk, h, w, ww);
            auto t1 = clk::now();
            for (int i = 0; i < n; i += chunk) ts::unpack_images(bits.data() + (size_t)i * h * ww, out.data() + (size_t)i * h * w, chunk, h, w, ww);
            auto t2 = clk::now();
            best_p = std::min(best_p, us(t0, t1));
            best_u = std::min(best_u, us(t1, t2));
        }
        printf("chunk %3d images: pack %.0f us total (%.1f us/chunk, %.1f GB/s)  unpack %.0f us total (%.1f us/chunk, %.1f GB/s)\n", chunk,
               best_p, best_p / (n / chunk), in.size() / best_p / 1e3, best_u, best_u / (n / chunk), in.size() / best_u / 1e3);
    }
    return memcmp(in.data(), out.data(), in.size()) != 0;
}
