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

// Raw issue rates of the instructions a 32-bit Shoup butterfly is made of,
// for the cross-check of the butterfly roof against the pipe limits:
// op 0 = IMAD (mad.lo.u32), 1 = IMAD.HI (mul.hi.u32), 2 = IADD3 (3-input
// add), 3 = VIADDMNMX (min(x, x - m)). 8 independent chains per thread.
template <int OP>
__global__ void __launch_bounds__(256) int_pipe_kernel(uint32_t b, uint32_t c, int iters, uint32_t* sink) {
    uint32_t a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 2654435761u + k * 97u;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if constexpr (OP == 0) {
                asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[k]) : "r"(b), "r"(c));
            } else if constexpr (OP == 1) {
                asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(a[k]) : "r"(b));
            } else if constexpr (OP == 2) {
                asm volatile("add.u32 %0, %0, %1;\n\tadd.u32 %0, %0, %2;" : "+r"(a[k]) : "r"(b), "r"(c));
            } else if constexpr (OP == 3) {
                a[k] = csub<uint32_t>(a[k] ^ b, c);
            } else {
                uint64_t w;
                asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(w) : "r"(a[k]), "r"(b));
                a[k] = static_cast<uint32_t>(w >> 32) ^ static_cast<uint32_t>(w);
            }
        }
    }
    uint32_t acc = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) acc ^= a[k];
    if (acc == 0x55555555u) sink[0] = acc;
}

}  // namespace lb

extern "C" int lb_bench_int_pipes(int iters, double* ops_per_s) {
    try {
        int dev = 0, sms = 0;
        LB_CUDA(cudaGetDevice(&dev));
        LB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        uint32_t* sink = nullptr;
        LB_CUDA(cudaMalloc(&sink, 4));
        const int grid = sms * 8;
        cudaEvent_t a, b;
        LB_CUDA(cudaEventCreate(&a));
        LB_CUDA(cudaEventCreate(&b));
        auto run = [&](auto kernel, int it) {
            kernel<<<grid, 256>>>(0x9E3779B9u, 0x1234567u, it / 10 + 1, sink);
            LB_CUDA(cudaEventRecord(a));
            kernel<<<grid, 256>>>(0x9E3779B9u, 0x1234567u, it, sink);
            LB_CUDA(cudaEventRecord(b));
            LB_CUDA(cudaEventSynchronize(b));
            float ms = 0;
            LB_CUDA(cudaEventElapsedTime(&ms, a, b));
            return double(grid) * 256.0 * it * 8 / (ms * 1e-3);
        };
        ops_per_s[0] = run(lb::int_pipe_kernel<0>, iters);
        ops_per_s[1] = run(lb::int_pipe_kernel<1>, iters);
        // OP 2 issues two dependent adds per chain step (PTX add.u32 pairs
        // may fuse into one IADD3): reported per chain step
        ops_per_s[2] = run(lb::int_pipe_kernel<2>, iters);
        ops_per_s[3] = run(lb::int_pipe_kernel<3>, iters);
        ops_per_s[4] = run(lb::int_pipe_kernel<4>, iters);  // IMAD.WIDE.U32 (+ a LOP3 fold)
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        cudaFree(sink);
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

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
