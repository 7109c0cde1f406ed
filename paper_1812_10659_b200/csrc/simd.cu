// Record-tensor (SIMD) dense layer: out_r = sum_i W[r][i] * x_i over whole
// ciphertexts, for every row r at once — the batched form of the reference's
// per-value weighted sums (proj/src/kernels.cpp:302-318), where each message
// holds one feature of up to n records in its slots.
//
// It is a modular GEMM [R x F] * [F x C] with C = every coefficient of a
// message (all plaintext instances, both components, every limb). Weights are
// small signed integers, so each thread keeps, per row of its tile, the sums
// of the positive and the negative products in 128 bits and reduces once.
#include <cuda_runtime.h>

#include <stdexcept>

#include "bfv.hpp"
#include "bfv_kernels.cuh"

namespace lb {

namespace {

constexpr int kRowTile = 8;     // rows per thread
constexpr int kColThreads = 256;
constexpr int kChunk = 256;     // weights staged in smem per tile row and pass

template <class St>
__global__ void __launch_bounds__(kColThreads) k_weighted_sums(BfvDev d, const St* const* __restrict__ xs,
                                                                  uint32_t F, St* const* __restrict__ outs,
                                                                  uint32_t R, const int64_t* __restrict__ W,
                                                                  uint64_t cols) {
    __shared__ int64_t wsh[kRowTile][kChunk];
    const uint64_t c = blockIdx.x * uint64_t(kColThreads) + threadIdx.x;
    const uint32_t r0 = blockIdx.y * kRowTile;
    const bool live = c < cols;
    const uint32_t limb = static_cast<uint32_t>((c >> d.logn) % d.L);
    uint64_t plo[kRowTile] = {}, phi[kRowTile] = {}, nlo[kRowTile] = {}, nhi[kRowTile] = {};
    for (uint32_t f0 = 0; f0 < F; f0 += kChunk) {
        const uint32_t fc = min(uint32_t(kChunk), F - f0);
        __syncthreads();
        for (uint32_t k = threadIdx.x; k < kRowTile * kChunk; k += kColThreads) {
            const uint32_t rr = k / kChunk, ff = k % kChunk;
            wsh[rr][ff] = (r0 + rr < R && ff < fc) ? W[uint64_t(r0 + rr) * F + f0 + ff] : 0;
        }
        __syncthreads();
        if (!live) continue;
        for (uint32_t ff = 0; ff < fc; ++ff) {
            const uint64_t x = __ldg(&xs[f0 + ff][c]);  // widened
#pragma unroll
            for (int rr = 0; rr < kRowTile; ++rr) {
                const int64_t w = wsh[rr][ff];
                const uint64_t aw = w < 0 ? uint64_t(-w) : uint64_t(w);
                uint64_t h, l;
                mul_wide(x, aw, h, l);
                if (w < 0) {
                    nlo[rr] += l;
                    nhi[rr] += h + (nlo[rr] < l ? 1 : 0);
                } else {
                    plo[rr] += l;
                    phi[rr] += h + (plo[rr] < l ? 1 : 0);
                }
            }
        }
    }
    if (!live) return;
    const Modulus m = modulus_of(d.primes[limb]);
#pragma unroll
    for (int rr = 0; rr < kRowTile; ++rr) {
        if (r0 + rr >= R) break;
        const uint64_t p = barrett_reduce_128(phi[rr], plo[rr], m);
        const uint64_t q = barrett_reduce_128(nhi[rr], nlo[rr], m);
        outs[r0 + rr][c] = static_cast<St>(sub_mod(p, q, m.q));
    }
}

// 32-bit residues (every q < 2^30) and |W| < 2^15: each product is exact in a
// signed 64-bit accumulator (|sum| < 2^17 * 2^15 * 2^30 = 2^62), one
// IMAD.WIDE per term; up to 16 rows per thread divide the x loads per
// product (fewer when R is small: the conv layers have 5 maps).
template <int kRowTile32, class St>
__global__ void __launch_bounds__(kColThreads) k_weighted_sums32(BfvDev d, const St* const* __restrict__ xs,
                                                                    uint32_t F, St* const* __restrict__ outs,
                                                                    uint32_t R, const int64_t* __restrict__ W,
                                                                    uint64_t cols) {
    __shared__ int32_t wsh[kChunk][kRowTile32];
    const uint64_t c = blockIdx.x * uint64_t(kColThreads) + threadIdx.x;
    const uint32_t r0 = blockIdx.y * kRowTile32;
    const bool live = c < cols;
    const uint32_t limb = static_cast<uint32_t>((c >> d.logn) % d.L);
    int64_t acc[kRowTile32] = {};
    for (uint32_t f0 = 0; f0 < F; f0 += kChunk) {
        const uint32_t fc = min(uint32_t(kChunk), F - f0);
        __syncthreads();
        for (uint32_t k = threadIdx.x; k < kRowTile32 * kChunk; k += kColThreads) {
            const uint32_t rr = k / kChunk, ff = k % kChunk;
            wsh[ff][rr] = (r0 + rr < R && ff < fc) ? static_cast<int32_t>(W[uint64_t(r0 + rr) * F + f0 + ff]) : 0;
        }
        __syncthreads();
        if (!live) continue;
#pragma unroll 4
        for (uint32_t ff = 0; ff < fc; ++ff) {
            const int32_t x = static_cast<int32_t>(__ldg(&xs[f0 + ff][c]));  // < 2^30
#pragma unroll
            for (int rr = 0; rr < kRowTile32; ++rr) acc[rr] += static_cast<int64_t>(x) * wsh[ff][rr];
        }
    }
    if (!live) return;
    const Modulus m = modulus_of(d.primes[limb]);
#pragma unroll
    for (int rr = 0; rr < kRowTile32; ++rr) {
        if (r0 + rr >= R) break;
        const int64_t v = acc[rr];
        const uint64_t a = reduce_u64(static_cast<uint64_t>(v < 0 ? -v : v), m);
        outs[r0 + rr][c] = static_cast<St>(v < 0 ? neg_mod(a, m.q) : a);
    }
}

}  // namespace

template <class St>
static void weighted_sums_words(Context& cx, const St* const* xs, uint32_t F, St* const* outs, uint32_t R,
                                const int64_t* W, bool small_weights, uint32_t cts, cudaStream_t s) {
    const BfvDev& d = cx.bfv()->dev;
    const uint64_t cols = uint64_t(cts) * 2 * d.L * d.n;
    if (small_weights && cx.primes_small(0, d.L)) {
        const int tile = R <= 4 ? 4 : R <= 8 ? 8 : 16;
        const dim3 grid(static_cast<unsigned>((cols + kColThreads - 1) / kColThreads), (R + tile - 1) / tile);
        if (grid.y > 65535) throw std::invalid_argument("weighted sums: too many rows");
        if (tile == 4)
            k_weighted_sums32<4, St><<<grid, kColThreads, 0, s>>>(d, xs, F, outs, R, W, cols);
        else if (tile == 8)
            k_weighted_sums32<8, St><<<grid, kColThreads, 0, s>>>(d, xs, F, outs, R, W, cols);
        else
            k_weighted_sums32<16, St><<<grid, kColThreads, 0, s>>>(d, xs, F, outs, R, W, cols);
    } else {
        const dim3 grid(static_cast<unsigned>((cols + kColThreads - 1) / kColThreads), (R + kRowTile - 1) / kRowTile);
        if (grid.y > 65535) throw std::invalid_argument("weighted sums: too many rows");
        k_weighted_sums<St><<<grid, kColThreads, 0, s>>>(d, xs, F, outs, R, W, cols);
    }
    LB_KERNEL_DONE();
}

void simd_weighted_sums(Context& cx, const void* const* xs, uint32_t F, void* const* outs, uint32_t R,
                        const int64_t* W, bool small_weights, uint32_t cts, cudaStream_t s) {
    if (!F || !R) return;
    if (F >= (1u << 17)) throw std::invalid_argument("weighted sums: fan-in above 2^17");
    // xs / outs: device arrays of device pointers to residue words
    if (cx.bfv()->dev.ks32)
        weighted_sums_words(cx, reinterpret_cast<const uint32_t* const*>(xs), F, reinterpret_cast<uint32_t* const*>(outs),
                            R, W, small_weights, cts, s);
    else
        weighted_sums_words(cx, reinterpret_cast<const uint64_t* const*>(xs), F, reinterpret_cast<uint64_t* const*>(outs),
                            R, W, small_weights, cts, s);
}

}  // namespace lb
