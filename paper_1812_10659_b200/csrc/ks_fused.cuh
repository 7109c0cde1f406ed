// Fused hybrid key switching on top of the cluster NTT core.
//
//   ks_inner_kernel  one cluster per (ciphertext, target prime r of Q∪P):
//                    for every digit j: ModUp of the digit to r computed on
//                    the fly in the transform's first pass (digit
//                    decomposition), forward NTT in distributed smem, then the
//                    key inner product accumulated in smem — the extended
//                    digits never touch HBM. Digits whose own primes contain r
//                    skip the transform and read the input's evaluations.
//   moddown_kernel   one cluster per (ciphertext, component, q_r): the P->q_r
//                    conversion in the first pass, forward NTT, then
//                    (acc - conv) * P^-1 (+ the other ciphertext component,
//                    through the automorphism for rotations) in the epilogue.
#pragma once

#include "bfv_kernels.cuh"
#include "ntt.cuh"

namespace lb {

struct KsInnerArgs {
    const void* dc;          // [count][L][n] coefficients of the input (word-sized: u64 or u32)
    const void* dn;          // input evaluations (residue words == the kernel word), poly stride d_stride
    uint64_t d_stride;
    uint64_t d_galois;       // automorphism applied to dn reads (0 = none)
    const void* key;         // [dnum][2][L+K][n] (value, Shoup companion): PairT<W>
    void* acc;               // [count][2][L+K][n] evaluations (word-sized)
    uint32_t count;
};

// a + b for a, b in [0, 2q) -> [0, 2q)
template <class W>
__device__ __forceinline__ W add_lazy2(W a, W b, W two_q) {
    const W s = a + b;
    return csub<W>(s, two_q);
}

// Word-specific views of the key-switch constant tables.
template <class W> struct KsTables;
template <> struct KsTables<uint64_t> {
    __device__ static const ulonglong2* dhat(const BfvDev& d) { return d.dhat_mod_sh; }
    __device__ static const ulonglong2* phat(const BfvDev& d) { return d.phat_mod_sh; }
};
template <> struct KsTables<uint32_t> {
    __device__ static const uint2* dhat(const BfvDev& d) { return d.dhat_mod_sh32; }
    __device__ static const uint2* phat(const BfvDev& d) { return d.phat_mod_sh32; }
};

// x mod q in [0, 6q) for a sum x < 2^61 of products, q in (2^28, 2^29) and
// mu = floor(2^60 / q): the quotient of x by 2q is estimated from the top 32
// bits of x / 2^29 (low by at most 3), so the remainder fits 32 bits.
__device__ __forceinline__ uint32_t barrett61_lazy(uint64_t x, uint32_t mu, uint32_t two_q) {
    const uint32_t xh = static_cast<uint32_t>(x >> 29);
    return static_cast<uint32_t>(x) - __umulhi(xh, mu) * two_q;
}

// Per-kernel constants of the 29-bit fast path (BfvDev::ks29): base
// conversions and the key inner product accumulate plain 32x32 -> 64-bit
// products (one IMAD.WIDE per term) and reduce once per output.
struct Wide29 {
    bool on = false;
    uint32_t mu = 0;  // floor(2^60 / q_r)
};

#ifndef LB_WIDE_CONV
#define LB_WIDE_CONV 1
#endif
#ifndef LB_MD_L2PF
#define LB_MD_L2PF 1  // bulk L2 prefetch of operands read late from HBM (key switch 1.421 -> 1.408 ms)
#endif
#ifndef LB_WIDE_MAC
#define LB_WIDE_MAC 1  // packed Shoup-free keys; BfvDev::ks29 contexts store them (bfv.cu ensure_key)
#endif

// Fast base conversion of A source limbs (limb stride n) to one target
// prime: sum_i y_i w_i with Shoup pairs w_i, in [0, 4r). A == 1 passes the
// raw residue (< 4r: every prime of Q and P is within a factor 4 of every
// other). A is a compile-time constant so all A loads of an element are
// independent (a runtime loop serializes them).
// WIDE (32-bit words, every prime in (2^28, 2^29), A <= 8): the sum of the A
// plain products y_i w_i < 2^61 is accumulated in 64 bits and reduced once.
// NT > 1: transform u converts the sources at src + u * pair_stride (same
// target prime and weights), all NT side by side (fwd_core).
template <int A, bool WIDE, int LOGN, int NT, class W, class St, class Last = std::nullptr_t>
__device__ __forceinline__ void fwd_conv_n(W* sm, const PrimeView<W>& P, uint32_t rank, const St* __restrict__ src,
                                           const PairT<W>* w, uint32_t w_stride, bool start_sync, Xchg xc,
                                           uint32_t mu, uint64_t pair_stride, Last&& last = nullptr,
                                           uint32_t w_pair = 0) {
    const W q = P.q, two_q = 2 * q;
    constexpr uint64_t n = 1ull << LOGN;
    if constexpr (A == 1) {
        fwd_core<LOGN, NT>(sm, P, rank, [&](uint32_t u, uint32_t rho, uint32_t off) {
            return static_cast<W>(__ldg(&(src + u * pair_stride + rho)[off]));
        }, start_sync, xc, last);
    } else if constexpr (WIDE && sizeof(W) == 4) {
        static_assert(A <= 8, "wide accumulation holds at most 8 products below 2^58");
        // (w_pair: transform u uses the weights at w + u * w_pair — two digits
        // of one ciphertext to the same target prime; 0: the same weights)
        uint32_t ww[NT][A];
#pragma unroll
        for (int u = 0; u < NT; ++u)
#pragma unroll
            for (int i = 0; i < A; ++i) ww[u][i] = w[u * w_pair + i * w_stride].x;
        const uint32_t four_q = 4 * q;
        fwd_core<LOGN, NT>(sm, P, rank, [&](uint32_t u, uint32_t rho, uint32_t off) {
            const St* s0 = src + u * pair_stride + rho;
            uint32_t v[A];
#pragma unroll
            for (int i = 0; i < A; ++i) v[i] = static_cast<uint32_t>(__ldg(&s0[i * n + off]));
            uint64_t acc = static_cast<uint64_t>(v[0]) * ww[u][0];
#pragma unroll
            for (int i = 1; i < A; ++i) acc += static_cast<uint64_t>(v[i]) * ww[u][i];
            return csub<uint32_t>(barrett61_lazy(acc, mu, two_q), four_q);
        }, start_sync, xc, last);
    } else {
        PairT<W> ww[A];
#pragma unroll
        for (int i = 0; i < A; ++i) ww[i] = w[i * w_stride];
        fwd_core<LOGN, NT>(sm, P, rank, [&](uint32_t u, uint32_t rho, uint32_t off) {
            const St* s0 = src + u * pair_stride + rho;
            W v[A];
#pragma unroll
            for (int i = 0; i < A; ++i) v[i] = static_cast<W>(__ldg(&s0[i * n + off]));
            W acc = shoup_lazy<W>(v[0], ww[0].x, ww[0].y, q) + shoup_lazy<W>(v[1], ww[1].x, ww[1].y, q);
#pragma unroll
            for (int i = 2; i < A; ++i) {
                acc = csub<W>(acc, two_q);
                acc += shoup_lazy<W>(v[i], ww[i].x, ww[i].y, q);
            }
            return acc;
        }, start_sync, xc, last);
    }
}

template <int LOGN, class W, bool WIDE = false, int NT = 1, class St, class Last = std::nullptr_t>
__device__ __forceinline__ void fwd_conv(W* sm, const PrimeView<W>& P, uint32_t rank, const St* src, uint32_t A,
                                         const PairT<W>* w, uint32_t w_stride, bool start_sync = true,
                                         Xchg xc = Xchg{}, uint32_t mu = 0, Last&& last = nullptr,
                                         uint64_t pair_stride = 0, uint32_t w_pair = 0) {
    switch (A) {
        case 1: fwd_conv_n<1, WIDE, LOGN, NT, W, St>(sm, P, rank, src, w, w_stride, start_sync, xc, mu, pair_stride, last, w_pair); break;
        case 2: fwd_conv_n<2, WIDE, LOGN, NT, W, St>(sm, P, rank, src, w, w_stride, start_sync, xc, mu, pair_stride, last, w_pair); break;
        // (64-bit words: unrolling 3 and 4 costs registers the common
        // K, alpha <= 2 configurations need)
        case 3: if constexpr (sizeof(W) == 4) { fwd_conv_n<3, WIDE, LOGN, NT, W, St>(sm, P, rank, src, w, w_stride, start_sync, xc, mu, pair_stride, last, w_pair); break; }
        [[fallthrough]];
        case 4: if constexpr (sizeof(W) == 4) { if (A == 4) { fwd_conv_n<4, WIDE, LOGN, NT, W, St>(sm, P, rank, src, w, w_stride, start_sync, xc, mu, pair_stride, last, w_pair); break; } }
        [[fallthrough]];
        case 5: if constexpr (sizeof(W) == 4) { if (A == 5) { fwd_conv_n<5, WIDE, LOGN, NT, W, St>(sm, P, rank, src, w, w_stride, start_sync, xc, mu, pair_stride, last, w_pair); break; } }
        [[fallthrough]];
        default: {
            const W q = P.q, two_q = 2 * q;
            constexpr uint64_t n = 1ull << LOGN;
            fwd_core<LOGN, NT>(sm, P, rank, [&](uint32_t u, uint32_t rho, uint32_t off) {
                const uint32_t x = rho + off;
                const St* su = src + u * pair_stride;
                W v = 0;
                for (uint32_t i = 0; i < A; ++i) {
                    const PairT<W> wi = w[i * w_stride];
                    v = add_lazy2<W>(v, shoup_lazy<W>(static_cast<W>(__ldg(&su[i * n + x])), wi.x, wi.y, q), two_q);
                }
                return v;
            }, start_sync, xc, last);
        }
    }
}

#ifndef LB_KS32_MINB
#define LB_KS32_MINB 3
#endif
#ifndef LB_KS_PLANES_MINB
#define LB_KS_PLANES_MINB 4  // 64 registers, 4 CTAs/SM: 138.3 vs 135.4 img/s at 3 CTAs/SM (80 registers)
#endif
// 64-bit words: three 32 KiB smem planes per CTA -> 2 CTAs/SM; 32-bit words
// halve the planes, so registers decide
template <class W> constexpr int ks_min_blocks() { return sizeof(W) == 8 ? 2 : LB_KS32_MINB; }

template <int LOGN, class W>
__global__ void __launch_bounds__(NttShape<LOGN>::T, ks_min_blocks<W>()) ks_inner_kernel(BfvDev d, KsInnerArgs a) {
    using S = NttShape<LOGN>;
    using Pr = PairT<W>;
    extern __shared__ __align__(16) uint8_t smem_raw[];
    W* sm = reinterpret_cast<W*>(smem_raw);
    W* acc0 = sm + plane_words<LOGN, W>();  // linear accumulator planes behind the transform plane
    W* acc1 = acc0 + S::M;
    const uint32_t LK = d.L + d.K;
    const uint32_t rank = S::CL > 1 ? cluster_rank() : 0;
    const uint32_t id = blockIdx.x / S::CL;
    const uint32_t c = id / LK, r = id % LK;
    const PrimeView<W> P = prime_view<W>(d.primes[r]);
    const W q = P.q, two_q = 2 * q;
    const uint32_t cta_base = rank * S::M;
    const uint64_t n = 1ull << LOGN;
    const Pr* key = static_cast<const Pr*>(a.key);
#pragma unroll
    for (int jj = 0; jj < kE; ++jj) {
        const uint32_t y = threadIdx.x + jj * S::T;
        acc0[y] = 0;
        acc1[y] = 0;
    }
    // acc_h[y] += v_jj * key_j[h][r][x] for the thread's 16 final-pass
    // elements; key loads (L2-resident, shared by every ciphertext of the
    // batch) are issued a half at a time ahead of their use.
    auto mac_all = [&](uint32_t j, auto&& value_of) {
        const Pr* k0 = key + ((uint64_t(j) * 2 * LK + r) << LOGN);
        const Pr* k1 = k0 + (uint64_t(LK) << LOGN);
        constexpr int kHalf = 8;  // elements whose key loads are in flight together
#pragma unroll
        for (int part = 0; part < kE / kHalf; ++part) {
            Pr w0[kHalf], w1[kHalf];
#pragma unroll
            for (int jj = 0; jj < kHalf; ++jj) {
                const uint32_t x = cta_base + threadIdx.x + (part * kHalf + jj) * S::T;
                w0[jj] = __ldg(&k0[x]);
                w1[jj] = __ldg(&k1[x]);
            }
#pragma unroll
            for (int jj = 0; jj < kHalf; ++jj) {
                const uint32_t y = threadIdx.x + (part * kHalf + jj) * S::T;
                const W v = value_of(y, cta_base + y);
                acc0[y] = add_lazy2<W>(acc0[y], shoup_lazy<W>(v, w0[jj].x, w0[jj].y, q), two_q);
                acc1[y] = add_lazy2<W>(acc1[y], shoup_lazy<W>(v, w1[jj].x, w1[jj].y, q), two_q);
            }
        }
    };
    __shared__ uint64_t mbar;
    Xchg xc = xchg_init<S::CL>(&mbar, 1);
    for (uint32_t j = 0; j < d.dnum; ++j) {
        const uint32_t lo = j * d.alpha, hi = min(d.L, lo + d.alpha);
        if (r >= lo && r < hi) {
            // the digit already lives in this prime: use the input's evaluations
            const W* dn = static_cast<const W*>(a.dn) + c * a.d_stride + (uint64_t(r) << LOGN);
            mac_all(j, [&](uint32_t, uint32_t x) {
                return __ldg(&dn[a.d_galois ? galois_src(x, a.d_galois, LOGN) : x]);
            });
            continue;
        }
        // src limbs hold y_i = [d_i (D_j/q_i)^-1]_{q_i} (a single-prime digit:
        // d itself); ModUp = sum_i y_i [D_j/q_i]_r computed in the loader
        const W* src = static_cast<const W*>(a.dc) + (uint64_t(c) * d.L + lo) * n;
        fwd_conv<LOGN, W>(sm, P, rank, src, hi - lo, KsTables<W>::dhat(d) + lo * LK + r, LK, true, xc);
        xc.parity ^= 1;  // the same plane (and mbarrier) serves every digit
        const uint32_t sbt = swb<W, LOGN>(threadIdx.x);
        mac_all(j, [&](uint32_t y, uint32_t) { return reduce_4q<W>(sm_at<LOGN>(sm, sbt, y - threadIdx.x), q, two_q); });
    }
    W* out0 = static_cast<W*>(a.acc) + (uint64_t(c) * 2 * LK + r) * n + cta_base;
    W* out1 = out0 + uint64_t(LK) * n;
#pragma unroll
    for (int jj = 0; jj < kE; ++jj) {
        const uint32_t y = threadIdx.x + jj * S::T;
        const W v0 = acc0[y], v1 = acc1[y];
        out0[y] = csub<W>(v0, q);
        out1[y] = csub<W>(v1, q);
    }
    // no trailing cluster barrier: the last remote access to this CTA's smem
    // (a scatter) is ordered before the cluster sync inside fwd_core
}


// ---- plane variant (32-bit words, dnum <= 3) ---------------------------------------
// Same result as ks_inner_kernel. Each foreign digit's transform lands in its
// own smem plane (dnum x 16 KiB = the accumulator kernel's footprint), so
// the key inner product runs once at the end with the accumulators in
// registers (no smem read-modify-write per digit), and transforms after the
// first skip the start barrier (nothing they overwrite is still being read).
constexpr uint32_t kMaxPlanes = 3;

template <int LOGN, bool K29 = false>
__global__ void __launch_bounds__(NttShape<LOGN>::T, LB_KS_PLANES_MINB) ks_inner_planes_kernel(BfvDev d,
                                                                                                     KsInnerArgs a) {
    using S = NttShape<LOGN>;
    using W = uint32_t;
    using Pr = uint2;
    extern __shared__ __align__(16) uint8_t smem_raw[];
    W* planes = reinterpret_cast<W*>(smem_raw);
    const uint32_t LK = d.L + d.K;
    const uint32_t rank = S::CL > 1 ? cluster_rank() : 0;
    const uint32_t r = blockIdx.x / S::CL, c = block_yz();
    if (c >= a.count) return;  // whole cluster
    const PrimeView<W> P = prime_view<W, LOGN>(d.tab32, d.primes, r);
    const W q = P.q, two_q = 2 * q;
    const uint64_t n = 1ull << LOGN;
    const uint32_t xt = rank * S::M + threadIdx.x;
    int own = -1;
    bool first = true;
    const uint32_t mu = K29 ? d.mu60[r] : 0u;
    __shared__ uint64_t mbar[kMaxPlanes];
    const Xchg xc0 = xchg_init<S::CL>(mbar, kMaxPlanes);
    for (uint32_t j = 0; j < d.dnum; ++j) {
        const uint32_t lo = j * d.alpha, hi = min(d.L, lo + d.alpha);
        if (r >= lo && r < hi) {
            own = static_cast<int>(j);
            continue;
        }
        const W* src = static_cast<const W*>(a.dc) + (uint64_t(c) * d.L + lo) * n;
        const Xchg xc{xc0.mbar ? xc0.mbar + 8 * j : 0u, 0u};
        fwd_conv<LOGN, W, K29 && LB_WIDE_CONV>(planes + j * plane_words<LOGN, W>(), P, rank, src, hi - lo,
                                               KsTables<W>::dhat(d) + lo * LK + r, LK, first, xc, mu);
        first = false;
    }
    const W* dn = static_cast<const W*>(a.dn) + c * a.d_stride + (uint64_t(r) << LOGN);
    const uint32_t sbt = swb<W, LOGN>(threadIdx.x);
    W* out0 = static_cast<W*>(a.acc) + (uint64_t(c) * 2 * LK + r) * n + xt;
    W* out1 = out0 + uint64_t(LK) * n;
    constexpr int kChunk = 4;
    if constexpr (K29 && LB_WIDE_MAC) {
        // packed keys [dnum][L+K][n] of (key_j[0], key_j[1]) words, no Shoup
        // companions: acc_h = sum_j v_j key_j[h] as 64-bit sums of at most
        // three products below 2^59 (v_j < 2q), one reduction per output.
        // Q limbs leave lazily (< 6 q_r: ModDown's epilogue multiplies them),
        // P limbs below 2 p (the inverse transform's input range).
        const Pr* key = static_cast<const Pr*>(a.key) + (uint64_t(r) << LOGN) + xt;
        const uint64_t kstride_j = uint64_t(LK) << LOGN;
        const bool to_p = r >= d.L;
        const W four_q = 4 * q;
#pragma unroll
        for (int e0 = 0; e0 < kE; e0 += kChunk) {
            uint64_t acc0[kChunk] = {}, acc1[kChunk] = {};
#pragma unroll
            for (uint32_t j = 0; j < kMaxPlanes; ++j) {
                if (j >= d.dnum) break;
                Pr kk[kChunk];
                W v[kChunk];
#pragma unroll
                for (int e = 0; e < kChunk; ++e) {
                    const uint32_t off = (e0 + e) * S::T;
                    kk[e] = __ldg(&key[j * kstride_j + off]);
                    if (static_cast<int>(j) == own) {
                        const uint32_t x = xt + off;
                        v[e] = __ldg(&dn[a.d_galois ? galois_src(x, a.d_galois, LOGN) : x]);
                    } else {
                        v[e] = csub<W>(sm_at<LOGN>(planes + j * plane_words<LOGN, W>(), sbt, off), two_q);
                    }
                }
#pragma unroll
                for (int e = 0; e < kChunk; ++e) {
                    acc0[e] += static_cast<uint64_t>(v[e]) * kk[e].x;
                    acc1[e] += static_cast<uint64_t>(v[e]) * kk[e].y;
                }
            }
#pragma unroll
            for (int e = 0; e < kChunk; ++e) {
                W u0 = barrett61_lazy(acc0[e], mu, two_q), u1 = barrett61_lazy(acc1[e], mu, two_q);
                if (to_p) {
                    u0 = csub<W>(csub<W>(u0, four_q), two_q);
                    u1 = csub<W>(csub<W>(u1, four_q), two_q);
                }
                out0[(e0 + e) * S::T] = u0;
                out1[(e0 + e) * S::T] = u1;
            }
        }
    } else {
    // acc_h[x] = sum_j v_j[x] * key_j[h][r][x], four elements at a time
    const Pr* key = static_cast<const Pr*>(a.key) + (uint64_t(r) << LOGN) + xt;
    const uint64_t kstride_j = uint64_t(2 * LK) << LOGN, kstride_h = uint64_t(LK) << LOGN;
#pragma unroll
    for (int e0 = 0; e0 < kE; e0 += kChunk) {
        W acc0[kChunk] = {}, acc1[kChunk] = {};
#pragma unroll
        for (uint32_t j = 0; j < kMaxPlanes; ++j) {
            if (j >= d.dnum) break;
            Pr w0[kChunk], w1[kChunk];
            W v[kChunk];
#pragma unroll
            for (int e = 0; e < kChunk; ++e) {
                const uint32_t off = (e0 + e) * S::T;
                w0[e] = __ldg(&key[j * kstride_j + off]);
                w1[e] = __ldg(&key[j * kstride_j + kstride_h + off]);
                if (static_cast<int>(j) == own) {
                    const uint32_t x = xt + off;
                    v[e] = __ldg(&dn[a.d_galois ? galois_src(x, a.d_galois, LOGN) : x]);
                } else {
                    v[e] = reduce_4q<W>(sm_at<LOGN>(planes + j * plane_words<LOGN, W>(), sbt, off), q, two_q);
                }
            }
#pragma unroll
            for (int e = 0; e < kChunk; ++e) {
                acc0[e] = add_lazy2<W>(acc0[e], shoup_lazy<W>(v[e], w0[e].x, w0[e].y, q), two_q);
                acc1[e] = add_lazy2<W>(acc1[e], shoup_lazy<W>(v[e], w1[e].x, w1[e].y, q), two_q);
            }
        }
#pragma unroll
        for (int e = 0; e < kChunk; ++e) {
            out0[(e0 + e) * S::T] = csub<W>(acc0[e], q);
            out1[(e0 + e) * S::T] = csub<W>(acc1[e], q);
        }
    }
    }
}

// ---- paired plane variant (29-bit fast path) ---------------------------------------
// One cluster per (ciphertext pair, target prime): the ModUp transforms of
// ciphertexts c and c + 1 run side by side (fwd_core NT = 2: shared twiddles,
// conversion weights, addresses, exchange) and the inner product loads every
// key word and automorphism position once for both. Planes: dnum foreign
// digits x 2 ciphertexts (64 KiB at dnum = 2: 3 CTAs per SM, which the 80
// registers per thread allow anyway); r = r_first + blockIdx.x / CL.
#ifndef LB_KS_PAIR_MINB
#define LB_KS_PAIR_MINB 3
#endif
constexpr uint32_t kPairDigits = 2;  // the paired kernel covers dnum <= 2 (launch_ks_inner)

template <int LOGN>
__global__ void __launch_bounds__(NttShape<LOGN>::T, LB_KS_PAIR_MINB) ks_inner_pair_kernel(BfvDev d, KsInnerArgs a,
                                                                                          uint32_t r_first) {
    using S = NttShape<LOGN>;
    using W = uint32_t;
    using Pr = uint2;
    extern __shared__ __align__(16) uint8_t smem_raw[];
    W* planes = reinterpret_cast<W*>(smem_raw);  // [foreign digit][pair member][M]
    const uint32_t LK = d.L + d.K;
    const uint32_t rank = S::CL > 1 ? cluster_rank() : 0;
    const uint32_t r = r_first + blockIdx.x / S::CL, c = 2 * block_yz();
    if (c >= a.count) return;  // whole cluster (count is even)
    const PrimeView<W> P = prime_view<W, LOGN>(d.tab32, d.primes, r);
    const W q = P.q, two_q = 2 * q, four_q = 4 * q;
    const uint64_t n = 1ull << LOGN;
    const uint32_t xt = rank * S::M + threadIdx.x;
    const uint32_t mu = d.mu60[r];
    int own = -1;
    bool first = true;
    uint32_t pl = 0;
    __shared__ uint64_t mbar[kPairDigits];
    const Xchg xc0 = xchg_init<S::CL>(mbar, kPairDigits);
    for (uint32_t j = 0; j < d.dnum; ++j) {
        const uint32_t lo = j * d.alpha, hi = min(d.L, lo + d.alpha);
        if (r >= lo && r < hi) {
            own = static_cast<int>(j);
            continue;
        }
        const W* src = static_cast<const W*>(a.dc) + (uint64_t(c) * d.L + lo) * n;
        const Xchg xc{xc0.mbar ? xc0.mbar + 8 * pl : 0u, 0u};
        fwd_conv<LOGN, W, true, 2>(planes + pl * 2 * plane_words<LOGN, W>(), P, rank, src, hi - lo, KsTables<W>::dhat(d) + lo * LK + r, LK,
                                   first, xc, mu, nullptr, uint64_t(d.L) * n);
        first = false;
        ++pl;
    }
    const Pr* key = static_cast<const Pr*>(a.key) + (uint64_t(r) << LOGN) + xt;
    const uint64_t kstride_j = uint64_t(LK) << LOGN;
    const W* dn = static_cast<const W*>(a.dn) + c * a.d_stride + (uint64_t(r) << LOGN);
    const uint32_t sbt = swb<W, LOGN>(threadIdx.x);
    W* out = static_cast<W*>(a.acc) + (uint64_t(c) * 2 * LK + r) * n + xt;
    const uint64_t out_h = uint64_t(LK) * n, out_u = 2 * out_h;
    const bool to_p = r >= d.L;
    constexpr int kChunk = 4;
#pragma unroll
    for (int e0 = 0; e0 < kE; e0 += kChunk) {
        Pr kk[kPairDigits][kChunk];
        uint32_t xs[kChunk];
#pragma unroll
        for (uint32_t j = 0; j < kPairDigits; ++j) {
            if (j >= d.dnum) break;
#pragma unroll
            for (int e = 0; e < kChunk; ++e) kk[j][e] = __ldg(&key[j * kstride_j + (e0 + e) * S::T]);
        }
        if (own >= 0) {
#pragma unroll
            for (int e = 0; e < kChunk; ++e) {
                const uint32_t x = xt + (e0 + e) * S::T;
                xs[e] = a.d_galois ? galois_src(x, a.d_galois, LOGN) : x;
            }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            uint64_t acc0[kChunk] = {}, acc1[kChunk] = {};
            uint32_t pj = 0;
#pragma unroll
            for (uint32_t j = 0; j < kPairDigits; ++j) {
                if (j >= d.dnum) break;
                W v[kChunk];
                if (static_cast<int>(j) == own) {
#pragma unroll
                    for (int e = 0; e < kChunk; ++e) v[e] = __ldg(&(dn + u * a.d_stride)[xs[e]]);
                } else {
#pragma unroll
                    for (int e = 0; e < kChunk; ++e)
                        v[e] = csub<W>(sm_at<LOGN>(planes + (pj * 2 + u) * plane_words<LOGN, W>(), sbt, (e0 + e) * S::T), two_q);
                    ++pj;
                }
#pragma unroll
                for (int e = 0; e < kChunk; ++e) {
                    acc0[e] += static_cast<uint64_t>(v[e]) * kk[j][e].x;
                    acc1[e] += static_cast<uint64_t>(v[e]) * kk[j][e].y;
                }
            }
#pragma unroll
            for (int e = 0; e < kChunk; ++e) {
                W u0 = barrett61_lazy(acc0[e], mu, two_q), u1 = barrett61_lazy(acc1[e], mu, two_q);
                if (to_p) {
                    u0 = csub<W>(csub<W>(u0, four_q), two_q);
                    u1 = csub<W>(csub<W>(u1, four_q), two_q);
                }
                out[u * out_u + (e0 + e) * S::T] = u0;
                out[u * out_u + out_h + (e0 + e) * S::T] = u1;
            }
        }
    }
}

// ---- mixed variant (29-bit fast path, dnum = 2) ---------------------------------------
// Every cluster needs exactly two smem planes, so 4 CTAs fit per SM (the
// paired kernel above needs four planes for the targets in P: 3 CTAs):
//   targets in Q (one foreign digit + the own digit): ciphertexts 2y, 2y+1
//     side by side, as in the paired kernel;
//   targets in P (two foreign digits): ONE ciphertext per cluster, its two
//     digit transforms side by side in the two planes (same prime: they
//     pair up like two ciphertexts do).
// grid.x = CL * (L + 2K) virtual targets v: v < L is q_v for the pair;
// v >= L is p_{(v-L)/2} for ciphertext 2y + ((v-L) & 1). grid.y/z = pairs.
#ifndef LB_KS_MIX_MINB
#define LB_KS_MIX_MINB 4
#endif
template <int LOGN>
__global__ void __launch_bounds__(NttShape<LOGN>::T, LB_KS_MIX_MINB) ks_inner_mix_kernel(BfvDev d, KsInnerArgs a) {
    using S = NttShape<LOGN>;
    using W = uint32_t;
    using Pr = uint2;
    constexpr uint32_t kPlane = plane_words<LOGN, W>();
    __shared__ __align__(16) W planes[2 * kPlane];
    __shared__ uint64_t mbar[2];
    const uint32_t LK = d.L + d.K;
    const uint32_t rank = S::CL > 1 ? cluster_rank() : 0;
    const uint32_t v = blockIdx.x / S::CL, y = block_yz();
    if (2 * y >= a.count) return;  // whole cluster (count is even)
    const bool in_q = v < d.L;
    const uint32_t r = in_q ? v : d.L + ((v - d.L) >> 1);
    const uint32_t c = 2 * y + (in_q ? 0u : ((v - d.L) & 1u));
    const PrimeView<W> P = prime_view<W, LOGN>(d.tab32, d.primes, r);
    const W q = P.q, two_q = 2 * q, four_q = 4 * q;
    const uint64_t n = 1ull << LOGN;
    const uint32_t xt = rank * S::M + threadIdx.x;
    const uint32_t mu = d.mu60[r];
    const Xchg xc0 = xchg_init<S::CL>(mbar, 2);
    const Pr* key = static_cast<const Pr*>(a.key) + (uint64_t(r) << LOGN) + xt;
    const uint64_t kstride_j = uint64_t(LK) << LOGN;
    const uint32_t sbt = swb<W, LOGN>(threadIdx.x);
    W* out = static_cast<W*>(a.acc) + (uint64_t(c) * 2 * LK + r) * n + xt;
    const uint64_t out_h = uint64_t(LK) * n;
    constexpr int kChunk = 4;
    if (in_q) {
        // one foreign digit (pair of transforms in the two planes) + the own digit
        const uint32_t own = r / d.alpha, fj = own ^ 1u;
        const uint32_t lo = fj * d.alpha, hi = min(d.L, lo + d.alpha);
        const W* dn = static_cast<const W*>(a.dn) + c * a.d_stride + (uint64_t(r) << LOGN);
        const uint64_t out_u = 2 * out_h;
#if LB_MD_L2PF
        // the own digit's evaluations (the input ciphertext, in HBM) are only
        // read after the transform: bulk L2 prefetch of this CTA's chunk of
        // both ciphertexts (the automorphism maps a chunk into one chunk)
        if (threadIdx.x == 0) {
            const uint32_t cb = rank * S::M;
            const uint32_t gb = a.d_galois ? (galois_src(cb, a.d_galois, LOGN) & ~uint32_t(S::M - 1)) : cb;
            prefetch_l2(dn + gb, S::M * sizeof(W));
            prefetch_l2(dn + a.d_stride + gb, S::M * sizeof(W));
        }
#endif
        const W* src = static_cast<const W*>(a.dc) + (uint64_t(c) * d.L + lo) * n;
        fwd_conv<LOGN, W, true, 2>(planes, P, rank, src, hi - lo, KsTables<W>::dhat(d) + lo * LK + r, LK, true,
                                   Xchg{xc0.mbar, 0u}, mu, nullptr, uint64_t(d.L) * n);
#pragma unroll
        for (int e0 = 0; e0 < kE; e0 += kChunk) {
            Pr ko[kChunk], kf[kChunk];
            uint32_t xs[kChunk];
#pragma unroll
            for (int e = 0; e < kChunk; ++e) {
                ko[e] = __ldg(&key[own * kstride_j + (e0 + e) * S::T]);
                kf[e] = __ldg(&key[fj * kstride_j + (e0 + e) * S::T]);
                const uint32_t x = xt + (e0 + e) * S::T;
                xs[e] = a.d_galois ? galois_src(x, a.d_galois, LOGN) : x;
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                W vo[kChunk], vf[kChunk];
#pragma unroll
                for (int e = 0; e < kChunk; ++e) {
                    vo[e] = __ldg(&(dn + u * a.d_stride)[xs[e]]);
                    vf[e] = csub<W>(sm_at<LOGN>(planes + u * kPlane, sbt, (e0 + e) * S::T), two_q);
                }
#pragma unroll
                for (int e = 0; e < kChunk; ++e) {
                    const uint64_t a0 = static_cast<uint64_t>(vo[e]) * ko[e].x + static_cast<uint64_t>(vf[e]) * kf[e].x;
                    const uint64_t a1 = static_cast<uint64_t>(vo[e]) * ko[e].y + static_cast<uint64_t>(vf[e]) * kf[e].y;
                    // Q limbs leave lazily (< 6 q_r: ModDown's epilogue multiplies them)
                    out[u * out_u + (e0 + e) * S::T] = barrett61_lazy(a0, mu, two_q);
                    out[u * out_u + out_h + (e0 + e) * S::T] = barrett61_lazy(a1, mu, two_q);
                }
            }
        }
    } else {
        // two foreign digits of one ciphertext, one plane each: both go to
        // the same prime, so they run as a transform pair too (u = digit; its
        // alpha source limbs and conversion weights follow digit 0's)
        const W* src = static_cast<const W*>(a.dc) + uint64_t(c) * d.L * n;
        fwd_conv<LOGN, W, true, 2>(planes, P, rank, src, d.alpha, KsTables<W>::dhat(d) + r, LK, true,
                                   Xchg{xc0.mbar, 0u}, mu, nullptr, uint64_t(d.alpha) * n, d.alpha * LK);
#pragma unroll
        for (int e0 = 0; e0 < kE; e0 += kChunk) {
            Pr k0[kChunk], k1[kChunk];
            W v0[kChunk], v1[kChunk];
#pragma unroll
            for (int e = 0; e < kChunk; ++e) {
                k0[e] = __ldg(&key[(e0 + e) * S::T]);
                k1[e] = __ldg(&key[kstride_j + (e0 + e) * S::T]);
                v0[e] = csub<W>(sm_at<LOGN>(planes, sbt, (e0 + e) * S::T), two_q);
                v1[e] = csub<W>(sm_at<LOGN>(planes + kPlane, sbt, (e0 + e) * S::T), two_q);
            }
#pragma unroll
            for (int e = 0; e < kChunk; ++e) {
                const uint64_t a0 = static_cast<uint64_t>(v0[e]) * k0[e].x + static_cast<uint64_t>(v1[e]) * k1[e].x;
                const uint64_t a1 = static_cast<uint64_t>(v0[e]) * k0[e].y + static_cast<uint64_t>(v1[e]) * k1[e].y;
                // P limbs below 2p: the inverse transform's input range
                out[(e0 + e) * S::T] = csub<W>(csub<W>(barrett61_lazy(a0, mu, two_q), four_q), two_q);
                out[out_h + (e0 + e) * S::T] = csub<W>(csub<W>(barrett61_lazy(a1, mu, two_q), four_q), two_q);
            }
        }
    }
}

// ---- TMEM-accumulator variant ------------------------------------------------------
// Same algorithm as ks_inner_kernel; the two accumulators of every element
// live in Tensor Memory instead of shared memory (128 TMEM columns per CTA:
// warp w owns lanes 32*(w%4).. of column block w/4, each thread 16 elements x
// 2 components x 2 words). Shared memory then holds only the 32 KiB
// transform chunk, so three CTAs fit per SM (registers allowing) instead of
// two.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void tmem_ld8(uint32_t addr, uint32_t (&r)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

__device__ __forceinline__ void tmem_st8(uint32_t addr, const uint32_t (&r)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(addr), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t addr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

__device__ __forceinline__ void tmem_st16(uint32_t addr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n"
        ::"r"(addr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
          "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}

constexpr int kTmemCols = 128;
#ifndef LB_KS_TMEM_MINB
#define LB_KS_TMEM_MINB 3
#endif

template <int LOGN>
__global__ void __launch_bounds__(NttShape<LOGN>::T, LB_KS_TMEM_MINB) ks_inner_tmem_kernel(BfvDev d, KsInnerArgs a) {
    using S = NttShape<LOGN>;
    static_assert(S::T == 256 || S::T == 128, "TMEM layout assumes 4 or 8 warps");
    // 4 columns (acc0, acc1 as 32-bit word pairs) per element; warps beyond
    // the four lane quadrants take the next column block
    constexpr uint32_t kColsPerThread = 4 * kE;
    __shared__ __align__(16) uint64_t sm[S::M];
    __shared__ uint32_t tmem_base_sh;
    const uint32_t warp = threadIdx.x / 32;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base_sh)),
                     "n"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tbase = tmem_base_sh + ((32u * (warp & 3u)) << 16) + (warp >> 2) * kColsPerThread;

    const uint32_t LK = d.L + d.K;
    const uint32_t rank = S::CL > 1 ? cluster_rank() : 0;
    const uint32_t id = blockIdx.x / S::CL;
    const uint32_t c = id / LK, r = id % LK;
    const PrimeView<uint64_t> P = prime_view<uint64_t>(d.primes[r]);
    const uint64_t q = P.q, two_q = 2 * q;
    const uint32_t cta_base = rank * S::M;
    const uint64_t n = 1ull << LOGN;

    // acc_h[e] += v_e * key_j[h][r][x_e] for the thread's 16 elements, two
    // at a time: columns [4e, 4e+4) of the thread's block = (acc0, acc1) words
    auto mac_all = [&](uint32_t j, bool first, auto&& value_of) {
        const ulonglong2* k0 = static_cast<const ulonglong2*>(a.key) + ((uint64_t(j) * 2 * LK + r) << LOGN);
        const ulonglong2* k1 = k0 + (uint64_t(LK) << LOGN);
#pragma unroll 2
        for (int pair = 0; pair < kE / 2; ++pair) {
            ulonglong2 w0[2], w1[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const uint32_t x = cta_base + threadIdx.x + (pair * 2 + e) * S::T;
                w0[e] = __ldg(&k0[x]);
                w1[e] = __ldg(&k1[x]);
            }
            uint32_t acc[8];
            if (!first) tmem_ld8(tbase + pair * 8, acc);
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const uint32_t y = threadIdx.x + (pair * 2 + e) * S::T;
                const uint64_t v = value_of(y, cta_base + y);
                uint64_t t0 = mul_shoup_lazy(v, w0[e].x, w0[e].y, q);
                uint64_t t1 = mul_shoup_lazy(v, w1[e].x, w1[e].y, q);
                if (!first) {
                    t0 = add_lazy2((uint64_t(acc[4 * e + 1]) << 32) | acc[4 * e], t0, two_q);
                    t1 = add_lazy2((uint64_t(acc[4 * e + 3]) << 32) | acc[4 * e + 2], t1, two_q);
                }
                acc[4 * e] = static_cast<uint32_t>(t0);
                acc[4 * e + 1] = static_cast<uint32_t>(t0 >> 32);
                acc[4 * e + 2] = static_cast<uint32_t>(t1);
                acc[4 * e + 3] = static_cast<uint32_t>(t1 >> 32);
            }
            tmem_st8(tbase + pair * 8, acc);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    };
    __shared__ uint64_t mbar;
    Xchg xc = xchg_init<S::CL>(&mbar, 1);
    for (uint32_t j = 0; j < d.dnum; ++j) {
        const uint32_t lo = j * d.alpha, hi = min(d.L, lo + d.alpha);
        const bool first = j == 0;
        if (r >= lo && r < hi) {
            const uint64_t* dn = static_cast<const uint64_t*>(a.dn) + c * a.d_stride + (uint64_t(r) << LOGN);
            mac_all(j, first, [&](uint32_t, uint32_t x) {
                return __ldg(&dn[a.d_galois ? galois_src(x, a.d_galois, LOGN) : x]);
            });
            continue;
        }
        const uint64_t* src = static_cast<const uint64_t*>(a.dc) + (uint64_t(c) * d.L + lo) * n;
        fwd_conv<LOGN, uint64_t>(sm, P, rank, src, hi - lo, d.dhat_mod_sh + lo * LK + r, LK, true, xc);
        xc.parity ^= 1;
        mac_all(j, first, [&](uint32_t y, uint32_t) { return reduce_4q<uint64_t>(sm[swz(y)], q, two_q); });
    }
    uint64_t* out0 = static_cast<uint64_t*>(a.acc) + (uint64_t(c) * 2 * LK + r) * n + cta_base;
    uint64_t* out1 = out0 + uint64_t(LK) * n;
#pragma unroll
    for (int quarter = 0; quarter < kE / 4; ++quarter) {
        uint32_t acc[16];
        tmem_ld16(tbase + quarter * 16, acc);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const uint32_t y = threadIdx.x + (quarter * 4 + e) * S::T;
            const uint64_t v0 = (uint64_t(acc[4 * e + 1]) << 32) | acc[4 * e];
            const uint64_t v1 = (uint64_t(acc[4 * e + 3]) << 32) | acc[4 * e + 2];
            out0[y] = v0 >= q ? v0 - q : v0;
            out1[y] = v1 >= q ? v1 - q : v1;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base_sh), "n"(kTmemCols));
}

struct ModDownArgs {
    const void* acc;          // [count][2][L+K][n]: Q limbs evaluations, P limbs coefficients (word-sized)
    // residue operands below are in the kernel word W (the context's residue word)
    const void* add0;         // optional, poly stride add_stride
    const void* add1;
    uint64_t add_stride;
    uint64_t add_galois;      // automorphism applied to add reads (0 = none)
    const void* sum0;         // optional second addend (no automorphism), poly stride sum_stride
    const void* sum1;
    uint64_t sum_stride;
    void* out0;
    void* out1;
    uint64_t out_stride;
    const void* p_inv;        // [L] (P^-1 mod q_r, Shoup): PairT<W>
    uint32_t count;
};

#ifndef LB_MODDOWN_DIRECT
#define LB_MODDOWN_DIRECT 1
#endif
#ifndef LB_MODDOWN32_MINB
#define LB_MODDOWN32_MINB LB_NTT32_MINB
#endif
template <class W> constexpr int moddown_min_blocks() { return sizeof(W) == 8 ? kMinBlocks : LB_MODDOWN32_MINB; }

#ifndef LB_MD_PREFETCH
#define LB_MD_PREFETCH 0  // 1: measured no gain (156.0 vs 156.4 images/s; 48 registers spill 60 bytes)
#endif

// ModDown's epilogue on one last-pass group of C consecutive evaluations:
// out = (acc_q - conv) P^-1 + sigma_g(add) + sum.
template <int LOGN, class W>
struct MdEpilogue {
    static constexpr int C = 1 << fwd_last_radix<LOGN>();
    const W* accq;
    const W* add;
    const W* sum;
    W* out;
    uint32_t cta_base;
    uint64_t galois;
    PairT<W> pinv;
    W q;
    struct Ops {
        W va[C], vb[C], vs[C];
    };
    __device__ __forceinline__ Ops prefetch(uint32_t base) const {
        Ops o;
        const uint32_t x0 = cta_base + base;
        if constexpr (sizeof(W) == 4 && C == 4) {
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(accq + x0));
            o.va[0] = v.x; o.va[1] = v.y; o.va[2] = v.z; o.va[3] = v.w;
            const uint4 t = sum ? __ldg(reinterpret_cast<const uint4*>(sum + x0)) : make_uint4(0, 0, 0, 0);
            o.vs[0] = t.x; o.vs[1] = t.y; o.vs[2] = t.z; o.vs[3] = t.w;
        } else if constexpr (sizeof(W) == 8 && C % 2 == 0) {  // u64 pairs as 16-byte loads
#pragma unroll
            for (int k = 0; k < C; k += 2) {
                const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(accq + x0 + k));
                o.va[k] = v.x;
                o.va[k + 1] = v.y;
                const ulonglong2 t = sum ? __ldg(reinterpret_cast<const ulonglong2*>(sum + x0 + k)) : make_ulonglong2(0, 0);
                o.vs[k] = t.x;
                o.vs[k + 1] = t.y;
            }
        } else {
#pragma unroll
            for (int k = 0; k < C; ++k) {
                o.va[k] = __ldg(&accq[x0 + k]);
                o.vs[k] = sum ? __ldg(&sum[x0 + k]) : 0;
            }
        }
#pragma unroll
        for (int k = 0; k < C; ++k)
            o.vb[k] = add ? __ldg(&add[galois ? galois_src(x0 + k, galois, LOGN) : x0 + k]) : 0;
        return o;
    }
    __device__ __forceinline__ void finish(uint32_t base, const W (&rr)[C], const Ops& o) const {
        const uint32_t x0 = cta_base + base;
        const W two_q = 2 * q;
        W u[C];
#pragma unroll
        for (int k = 0; k < C; ++k) {
            const W conv = reduce_4q<W>(rr[k], q, two_q);
            W v = shoup_full<W>(o.va[k] + q - conv, pinv.x, pinv.y, q);
            v = csub<W>(v + o.vb[k], q);
            u[k] = csub<W>(v + o.vs[k], q);
        }
        if constexpr (sizeof(W) == 4 && C == 4) {
            *reinterpret_cast<uint4*>(out + x0) = make_uint4(u[0], u[1], u[2], u[3]);
        } else if constexpr (sizeof(W) == 8 && C % 2 == 0) {
#pragma unroll
            for (int k = 0; k < C; k += 2) *reinterpret_cast<ulonglong2*>(out + x0 + k) = make_ulonglong2(u[k], u[k + 1]);
        } else {
#pragma unroll
            for (int k = 0; k < C; ++k) out[x0 + k] = u[k];
        }
    }
};

// Paired instance (32-bit words): one cluster runs both accumulator
// components of (ciphertext, q_r) side by side — same prime, twiddles,
// conversion weights, P^-1 and automorphism positions (fwd_core NT = 2).
#ifndef LB_MD_PAIR_MINB
#define LB_MD_PAIR_MINB 4
#endif

template <int LOGN>
__global__ void __launch_bounds__(NttShape<LOGN>::T, LB_MD_PAIR_MINB) moddown_pair_kernel(BfvDev d, ModDownArgs a) {
    using S = NttShape<LOGN>;
    using W = uint32_t;
    __shared__ __align__(16) W sm[2 * plane_words<LOGN, W>()];
    const uint32_t LK = d.L + d.K;
    const uint32_t rank = S::CL > 1 ? cluster_rank() : 0;
    const uint32_t r = blockIdx.x / S::CL, c = block_yz();
    if (c >= a.count) return;  // whole cluster
    const PrimeView<W> P = prime_view<W, LOGN>(d.tab32, d.primes, r);
    const W q = P.q;
    const uint64_t n = 1ull << LOGN;
    const W* accp = static_cast<const W*>(a.acc) + (uint64_t(c) * 2 * LK + d.L) * n;  // component h at + h LK n
    __shared__ uint64_t mbar;
    const Xchg xc = xchg_init<S::CL>(&mbar, 1);
    const uint32_t cta_base = rank * S::M;
    const W* accq = static_cast<const W*>(a.acc) + (uint64_t(c) * 2 * LK + r) * n;
    const uint64_t lo = c * a.add_stride + (uint64_t(r) << LOGN), ls = c * a.sum_stride + (uint64_t(r) << LOGN);
    const W* add0 = a.add0 ? static_cast<const W*>(a.add0) + lo : nullptr;
    const W* add1 = a.add1 ? static_cast<const W*>(a.add1) + lo : nullptr;
    const W* sum0 = a.sum0 ? static_cast<const W*>(a.sum0) + ls : nullptr;
    const W* sum1 = a.sum1 ? static_cast<const W*>(a.sum1) + ls : nullptr;
    const uint64_t oo = c * a.out_stride + (uint64_t(r) << LOGN);
    const PairT<W> pinv = static_cast<const PairT<W>*>(a.p_inv)[r];
    const uint32_t mu = d.mu60[r];
#if LB_MD_L2PF
    // the epilogue's operands come from HBM (the accumulators and the addends
    // were written a kernel or more ago): one bulk L2 prefetch per operand
    // chunk at entry, so the last pass finds them in L2. The automorphism maps
    // this CTA's chunk of positions into ONE chunk of the addend.
    if (threadIdx.x == 0) {
        constexpr uint32_t kBytes = S::M * sizeof(W);
        prefetch_l2(accq + cta_base, kBytes);
        prefetch_l2(accq + uint64_t(LK) * n + cta_base, kBytes);
        if (sum0) prefetch_l2(sum0 + cta_base, kBytes);
        if (sum1) prefetch_l2(sum1 + cta_base, kBytes);
        const uint32_t gb = a.add_galois ? (galois_src(cta_base, a.add_galois, LOGN) & ~uint32_t(S::M - 1)) : cta_base;
        if (add0) prefetch_l2(add0 + gb, kBytes);
        if (add1) prefetch_l2(add1 + gb, kBytes);
    }
#endif
    const MdEpilogue<LOGN, W> ep0{accq, add0, sum0, static_cast<W*>(a.out0) + oo, cta_base, a.add_galois, pinv, q};
    const MdEpilogue<LOGN, W> ep1{accq + uint64_t(LK) * n, add1, sum1, static_cast<W*>(a.out1) + oo, cta_base, a.add_galois, pinv, q};
    fwd_conv<LOGN, W, true, 2>(sm, P, rank, accp, d.K, KsTables<W>::phat(d) + r, d.L, true, xc, mu,
                               [&](uint32_t u, uint32_t base, W(&rr)[1 << fwd_last_radix<LOGN>()]) {
                                   if (u)
                                       ep1.finish(base, rr, ep1.prefetch(base));
                                   else
                                       ep0.finish(base, rr, ep0.prefetch(base));
                               },
                               uint64_t(LK) * n);
}

// Quad instance: both components AND two target primes q_r, q_{r+1} per
// cluster. The P -> Q conversion reads every P-limb coefficient once for both
// targets (the loader forms both sums from the same K loads; the second
// target's values wait in a per-thread smem stash), which halves the kernel's
// dominant L2 traffic (each coefficient of [acc]_P was read L times, once per
// target prime); the second transform then loads from the stash.
#ifndef LB_MD_QUAD_MINB
#define LB_MD_QUAD_MINB 3
#endif
#ifndef LB_MD_RPAIR_MINB
#define LB_MD_RPAIR_MINB 5
#endif
// NT = 2: both components (the quad); NT = 1: one component, two targets
template <int LOGN, int NT> constexpr size_t moddown_quad_smem() {
    return NT * (plane_words<LOGN, uint32_t>() + NttShape<LOGN>::M) * sizeof(uint32_t);
}

template <int A, int LOGN, int NT, class Last>
__device__ __forceinline__ void md_quad_first(uint32_t* planes, uint32_t* stash, const PrimeView<uint32_t>& P1,
                                              uint32_t q2, uint32_t mu1, uint32_t mu2, uint32_t rank,
                                              const uint32_t* __restrict__ accp, uint64_t comp_stride,
                                              const uint2* __restrict__ w, uint32_t w_stride, Xchg xc, Last&& last) {
    using S = NttShape<LOGN>;
    constexpr uint64_t n = 1ull << LOGN;
    uint32_t w1[A], w2[A];
#pragma unroll
    for (int i = 0; i < A; ++i) {
        w1[i] = w[i * w_stride].x;
        w2[i] = w[i * w_stride + 1].x;
    }
    const uint32_t q1 = P1.q;
    fwd_core<LOGN, NT>(planes, P1, rank, [&](uint32_t u, uint32_t rho, uint32_t off) {
        const uint32_t* s0 = accp + u * comp_stride + rho;
        uint32_t v[A];
#pragma unroll
        for (int i = 0; i < A; ++i) v[i] = __ldg(&s0[i * n + off]);
        uint64_t a1 = static_cast<uint64_t>(v[0]) * w1[0], a2 = static_cast<uint64_t>(v[0]) * w2[0];
#pragma unroll
        for (int i = 1; i < A; ++i) {
            a1 += static_cast<uint64_t>(v[i]) * w1[i];
            a2 += static_cast<uint64_t>(v[i]) * w2[i];
        }
        stash[(u * kE + off / S::NE) * S::T + threadIdx.x] = barrett61_lazy(a2, mu2, 2 * q2);
        return csub<uint32_t>(barrett61_lazy(a1, mu1, 2 * q1), 4 * q1);
    }, true, xc, last);
}

// NT = 2: grid.y/z = ciphertexts (both components per cluster);
// NT = 1: grid.y/z = ciphertext x component.
template <int LOGN, int NT>
__global__ void __launch_bounds__(NttShape<LOGN>::T, NT == 2 ? LB_MD_QUAD_MINB : LB_MD_RPAIR_MINB)
    moddown_quad_kernel(BfvDev d, ModDownArgs a) {
    using S = NttShape<LOGN>;
    using W = uint32_t;
    extern __shared__ __align__(16) uint8_t smem_raw[];
    W* planes = reinterpret_cast<W*>(smem_raw);
    W* stash = planes + NT * plane_words<LOGN, W>();  // [NT][kE][T], thread-private columns
    const uint32_t LK = d.L + d.K;
    const uint32_t rank = S::CL > 1 ? cluster_rank() : 0;
    const uint32_t r1 = 2 * (blockIdx.x / S::CL), yz = block_yz();
    const uint32_t c = NT == 2 ? yz : yz >> 1, h0 = NT == 2 ? 0u : (yz & 1u);
    if (c >= a.count) return;  // whole cluster
    const bool two = r1 + 1 < d.L;
    const uint32_t r2 = two ? r1 + 1 : r1;
    const PrimeView<W> P1 = prime_view<W, LOGN>(d.tab32, d.primes, r1);
    const PrimeView<W> P2 = prime_view<W, LOGN>(d.tab32, d.primes, r2);
    const uint64_t n = 1ull << LOGN, comp = uint64_t(LK) * n;
    const W* accp = static_cast<const W*>(a.acc) + ((uint64_t(c) * 2 + h0) * LK + d.L) * n;
    __shared__ uint64_t mbar;
    Xchg xc = xchg_init<S::CL>(&mbar, 1);
    const uint32_t cta_base = rank * S::M;
    const W* accq = static_cast<const W*>(a.acc) + (uint64_t(c) * 2 + h0) * LK * n;
    const uint64_t lo = c * a.add_stride, ls = c * a.sum_stride, oo = c * a.out_stride;
    const PairT<W>* pinvs = static_cast<const PairT<W>*>(a.p_inv);
    // epilogue of component h0 + u at prime r
    auto finish = [&](uint32_t u, uint32_t r, W q, uint32_t base, W(&rr)[1 << fwd_last_radix<LOGN>()]) {
        const uint64_t ro = uint64_t(r) << LOGN;
        const bool h = (h0 + u) != 0;
        const W* add = static_cast<const W*>(h ? a.add1 : a.add0);
        const W* sum = static_cast<const W*>(h ? a.sum1 : a.sum0);
        const MdEpilogue<LOGN, W> ep{accq + u * comp + ro,
                                     add ? add + lo + ro : nullptr,
                                     sum ? sum + ls + ro : nullptr,
                                     static_cast<W*>(h ? a.out1 : a.out0) + oo + ro,
                                     cta_base, a.add_galois, pinvs[r], q};
        ep.finish(base, rr, ep.prefetch(base));
    };
    const uint2* w = KsTables<W>::phat(d) + r1;
    const uint32_t mu1 = d.mu60[r1], mu2 = d.mu60[r2];
    auto last1 = [&](uint32_t u, uint32_t base, W(&rr)[1 << fwd_last_radix<LOGN>()]) { finish(u, r1, P1.q, base, rr); };
    switch (d.K) {
        case 2: md_quad_first<2, LOGN, NT>(planes, stash, P1, P2.q, mu1, mu2, rank, accp, comp, w, d.L, xc, last1); break;
        case 3: md_quad_first<3, LOGN, NT>(planes, stash, P1, P2.q, mu1, mu2, rank, accp, comp, w, d.L, xc, last1); break;
        case 4: md_quad_first<4, LOGN, NT>(planes, stash, P1, P2.q, mu1, mu2, rank, accp, comp, w, d.L, xc, last1); break;
        default: md_quad_first<5, LOGN, NT>(planes, stash, P1, P2.q, mu1, mu2, rank, accp, comp, w, d.L, xc, last1); break;
    }
    if (!two) return;  // whole cluster
    xc.parity ^= 1;
    const W four_q2 = 4 * P2.q;
    fwd_core<LOGN, NT>(planes, P2, rank, [&](uint32_t u, uint32_t, uint32_t off) {
        return csub<W>(stash[(u * kE + off / S::NE) * S::T + threadIdx.x], four_q2);
    }, true, xc, [&](uint32_t u, uint32_t base, W(&rr)[1 << fwd_last_radix<LOGN>()]) { finish(u, r2, P2.q, base, rr); });
}

template <int LOGN, class W, bool K29 = false>
__global__ void __launch_bounds__(NttShape<LOGN>::T, moddown_min_blocks<W>()) moddown_kernel(BfvDev d, ModDownArgs a) {
    using S = NttShape<LOGN>;
    __shared__ __align__(16) W sm[plane_words<LOGN, W>()];
    const uint32_t LK = d.L + d.K;
    const uint32_t rank = S::CL > 1 ? cluster_rank() : 0;
    const uint32_t r = blockIdx.x / S::CL, ch = block_yz();
    const uint32_t h = ch & 1, c = ch >> 1;
    if (c >= a.count) return;  // whole cluster
    const PrimeView<W> P = prime_view<W, LOGN>(d.tab32, d.primes, r);
    const W q = P.q, two_q = 2 * q;
    const uint64_t n = 1ull << LOGN;
    const W* accp = static_cast<const W*>(a.acc) + ((uint64_t(c) * 2 + h) * LK + d.L) * n;
    // K == 1: [acc]_p (< p < 4 q_r) feeds the lazy transform unreduced;
    // else the P limbs already hold y_l = [acc_l (P/p_l)^-1]_{p_l} (folded
    // into the inverse transform) and the loader forms sum_l y_l [P/p_l]_{q_r}
    __shared__ uint64_t mbar;
    const Xchg xc = xchg_init<S::CL>(&mbar, 1);
    const uint32_t cta_base = rank * S::M;
    const W* accq = static_cast<const W*>(a.acc) + ((uint64_t(c) * 2 + h) * LK + r) * n;
    const W* add = static_cast<const W*>(h ? a.add1 : a.add0);
    if (add) add += c * a.add_stride + (uint64_t(r) << LOGN);
    const W* sum = static_cast<const W*>(h ? a.sum1 : a.sum0);
    if (sum) sum += c * a.sum_stride + (uint64_t(r) << LOGN);
    W* out = static_cast<W*>(h ? a.out1 : a.out0) + c * a.out_stride + (uint64_t(r) << LOGN);
    const PairT<W> pinv = static_cast<const PairT<W>*>(a.p_inv)[r];
    constexpr bool kWide = K29 && LB_WIDE_CONV && sizeof(W) == 4;
    const uint32_t mu = kWide ? d.mu60[r] : 0u;
#if LB_MODDOWN_DIRECT
    // epilogue on the transform's last-pass groups (consecutive evaluations,
    // in registers): 16-byte loads of the Q accumulator and the second
    // addend and 16-byte stores of the result for radix-4 groups of u32;
    // with LB_MD_PREFETCH the next group's operands are in flight during the
    // current group's butterflies
    MdEpilogue<LOGN, W> ep{accq, add, sum, out, cta_base, a.add_galois, pinv, q};
#if LB_MD_PREFETCH
    fwd_conv<LOGN, W, kWide>(sm, P, rank, accp, d.K, KsTables<W>::phat(d) + r, d.L, true, xc, mu, ep);
#else
    fwd_conv<LOGN, W, kWide>(sm, P, rank, accp, d.K, KsTables<W>::phat(d) + r, d.L, true, xc, mu,
                             [&](uint32_t, uint32_t base, W(&rr)[1 << fwd_last_radix<LOGN>()]) { ep.finish(base, rr, ep.prefetch(base)); });
#endif
#else
    fwd_conv<LOGN, W, kWide>(sm, P, rank, accp, d.K, KsTables<W>::phat(d) + r, d.L, true, xc, mu);
    const uint32_t sbt = swb<W, LOGN>(threadIdx.x);
    // Epilogue in two halves: issue every global load of a half (including
    // the automorphism gather, which hits scattered sectors) before using
    // any of them, so their latencies overlap.
    constexpr int kHalf = 8;
#pragma unroll
    for (int part = 0; part < kE / kHalf; ++part) {
        W va[kHalf], vb[kHalf], vs[kHalf];
#pragma unroll
        for (int jj = 0; jj < kHalf; ++jj) {
            const uint32_t x = cta_base + threadIdx.x + (part * kHalf + jj) * S::T;
            va[jj] = static_cast<W>(__ldg(&accq[x]));
            vb[jj] = add ? __ldg(&add[a.add_galois ? galois_src(x, a.add_galois, LOGN) : x]) : 0;
            vs[jj] = sum ? __ldg(&sum[x]) : 0;
        }
#pragma unroll
        for (int jj = 0; jj < kHalf; ++jj) {
            const uint32_t y = threadIdx.x + (part * kHalf + jj) * S::T;
            const W conv = reduce_4q<W>(sm_at<LOGN>(sm, sbt, (part * kHalf + jj) * S::T), q, two_q);
            W u = shoup_full<W>(va[jj] + q - conv, pinv.x, pinv.y, q);
            u += vb[jj];
            u = csub<W>(u, q);
            u += vs[jj];
            u = csub<W>(u, q);
            out[cta_base + y] = u;
        }
    }
#endif
}

}  // namespace lb
