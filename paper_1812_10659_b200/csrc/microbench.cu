// Integer-pipe roof for the roofline: sustained Harvey/Shoup butterflies per
// second with every operand register resident (no memory traffic at all).
// MEASURED_PEAKS.json carries only HBM and bf16 peaks; SURVEY.md §8(d) asks
// for this number as the denominator of integer-bound kernels.
#include <cuda_runtime.h>

#include "../../include/lola_b200.h"
#include "context.hpp"
#include "ntt.cuh"

namespace lb {

// Same butterfly sequence as fwd_group<4> (radix-16 pass: 32 butterflies),
// twiddles held in registers, repeated `iters` times. Results folded into
// `sink` so nothing is dead code.
template <class W>
__global__ void __launch_bounds__(256) butterfly_peak_kernel(W q, PairT<W> w0, PairT<W> w1, int iters,
                                                               uint64_t* sink) {
    const W two_q = 2 * q;
    W r[kE];
#pragma unroll
    for (int k = 0; k < kE; ++k) r[k] = static_cast<W>((threadIdx.x * 2654435761ull + k * 97ull) % q);
    PairT<W> w[4] = {w0, w1, w0, w1};
    w[2].x ^= 1;
    w[3].x ^= 1;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int l = 0; l < kLogE; ++l) {
            const int half = 1 << (kLogE - 1 - l);
#pragma unroll
            for (int k = 0; k < kE; ++k) {
                if (k & half) continue;
                ct_bfly(r[k], r[k + half], w[(k + l) & 3], q, two_q);
            }
        }
    }
    W acc = 0;
#pragma unroll
    for (int k = 0; k < kE; ++k) acc ^= r[k];
    if (acc == static_cast<W>(0x5555555555555555ull)) sink[0] = acc;
}

}  // namespace lb

extern "C" int lb_bench_butterfly_peak(uint64_t q, int blocks_per_sm, int iters, double* bfly_per_s) {
    try {
        int dev = 0, sms = 0;
        LB_CUDA(cudaGetDevice(&dev));
        LB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        uint64_t* sink = nullptr;
        LB_CUDA(cudaMalloc(&sink, 8));
        const uint64_t w = 0x123456789abcdefull % q, w2 = 0x0fedcba987654321ull % q;
        const int grid = sms * blocks_per_sm;
        // q < 2^30: the 32-bit word butterfly the NTT kernels use for such primes
        const bool w32 = q < lb::kWord32Bound;
        auto launch = [&](int it) {
            if (w32) {
                const uint2 w0 = make_uint2(uint32_t(w), lb::shoup_companion32(w, q));
                const uint2 w1 = make_uint2(uint32_t(w2), lb::shoup_companion32(w2, q));
                lb::butterfly_peak_kernel<uint32_t><<<grid, 256>>>(uint32_t(q), w0, w1, it, sink);
            } else {
                const ulonglong2 w0 = make_ulonglong2(w, lb::shoup_companion(w, q));
                const ulonglong2 w1 = make_ulonglong2(w2, lb::shoup_companion(w2, q));
                lb::butterfly_peak_kernel<uint64_t><<<grid, 256>>>(q, w0, w1, it, sink);
            }
        };
        launch(iters / 10 + 1);  // warm-up
        cudaEvent_t a, b;
        LB_CUDA(cudaEventCreate(&a));
        LB_CUDA(cudaEventCreate(&b));
        LB_CUDA(cudaEventRecord(a));
        launch(iters);
        LB_CUDA(cudaEventRecord(b));
        LB_CUDA(cudaEventSynchronize(b));
        float ms = 0;
        LB_CUDA(cudaEventElapsedTime(&ms, a, b));
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        cudaFree(sink);
        const double bflies = double(grid) * 256.0 * iters * (lb::kE / 2) * lb::kLogE;
        *bfly_per_s = bflies / (ms * 1e-3);
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}
