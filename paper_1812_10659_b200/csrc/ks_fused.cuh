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
    const uint64_t* dc;      // [count][L][n] coefficients of the input
    const uint64_t* dn;      // input evaluations, poly stride d_stride
    uint64_t d_stride;
    uint64_t d_galois;       // automorphism applied to dn reads (0 = none)
    const ulonglong2* key;   // [dnum][2][L+K][n] (value, Shoup companion)
    uint64_t* acc;           // [count][2][L+K][n] evaluations
    uint32_t count;
};

// a + b for a, b in [0, 2q) -> [0, 2q)
__device__ __forceinline__ uint64_t add_lazy2(uint64_t a, uint64_t b, uint64_t two_q) {
    const uint64_t s = a + b;
    return s >= two_q ? s - two_q : s;
}

template <int LOGN>
__global__ void __launch_bounds__(NttShape<LOGN>::T, 2) ks_inner_kernel(BfvDev d, KsInnerArgs a) {
    using S = NttShape<LOGN>;
    extern __shared__ __align__(16) uint64_t smem[];
    uint64_t* sm = smem;
    uint64_t* acc0 = smem + S::M;
    uint64_t* acc1 = smem + 2 * S::M;
    const uint32_t LK = d.L + d.K;
    const uint32_t rank = S::CL > 1 ? cluster_rank() : 0;
    const uint32_t id = blockIdx.x / S::CL;
    const uint32_t c = id / LK, r = id % LK;
    const PrimeDev& P = d.primes[r];
    const uint64_t q = P.q, two_q = 2 * q;
    const uint32_t cta_base = rank * S::M;
    const uint64_t n = 1ull << LOGN;
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
        const ulonglong2* k0 = a.key + ((uint64_t(j) * 2 * LK + r) << LOGN);
        const ulonglong2* k1 = k0 + (uint64_t(LK) << LOGN);
        constexpr int kHalf = kE / 2;
#pragma unroll
        for (int part = 0; part < 2; ++part) {
            ulonglong2 w0[kHalf], w1[kHalf];
#pragma unroll
            for (int jj = 0; jj < kHalf; ++jj) {
                const uint32_t x = cta_base + threadIdx.x + (part * kHalf + jj) * S::T;
                w0[jj] = __ldg(&k0[x]);
                w1[jj] = __ldg(&k1[x]);
            }
#pragma unroll
            for (int jj = 0; jj < kHalf; ++jj) {
                const uint32_t y = threadIdx.x + (part * kHalf + jj) * S::T;
                const uint64_t v = value_of(y, cta_base + y);
                acc0[y] = add_lazy2(acc0[y], mul_shoup_lazy(v, w0[jj].x, w0[jj].y, q), two_q);
                acc1[y] = add_lazy2(acc1[y], mul_shoup_lazy(v, w1[jj].x, w1[jj].y, q), two_q);
            }
        }
    };
    for (uint32_t j = 0; j < d.dnum; ++j) {
        const uint32_t lo = j * d.alpha, hi = min(d.L, lo + d.alpha);
        if (r >= lo && r < hi) {
            // the digit already lives in this prime: use the input's evaluations
            const uint64_t* dn = a.dn + c * a.d_stride + (uint64_t(r) << LOGN);
            mac_all(j, [&](uint32_t, uint32_t x) {
                return __ldg(&dn[a.d_galois ? galois_src(x, a.d_galois, LOGN) : x]);
            });
            continue;
        }
        const uint64_t* src = a.dc + (uint64_t(c) * d.L + lo) * n;
        if (hi - lo == 1) {
            // single-prime digit: the coefficient (< q_lo < 4 q_r) feeds the
            // lazy transform unreduced
            fwd_core<LOGN>(sm, P, rank, [&](uint32_t x) { return __ldg(&src[x]); });
        } else {
            // src limbs already hold y_i = [d_i (D_j/q_i)^-1]_{q_i}; fast base
            // conversion sum_i y_i [D_j/q_i]_r, kept lazily in [0, 2r)
            fwd_core<LOGN>(sm, P, rank, [&](uint32_t x) {
                uint64_t v = 0;
                for (uint32_t i = lo; i < hi; ++i) {
                    const ulonglong2 w = d.dhat_mod_sh[i * LK + r];
                    v = add_lazy2(v, mul_shoup_lazy(__ldg(&src[(uint64_t(i - lo) << LOGN) + x]), w.x, w.y, q), two_q);
                }
                return v;
            });
        }
        mac_all(j, [&](uint32_t y, uint32_t) { return reduce_4q(sm[swz(y)], q, two_q); });
    }
    uint64_t* out0 = a.acc + (uint64_t(c) * 2 * LK + r) * n + cta_base;
    uint64_t* out1 = out0 + uint64_t(LK) * n;
#pragma unroll
    for (int jj = 0; jj < kE; ++jj) {
        const uint32_t y = threadIdx.x + jj * S::T;
        const uint64_t v0 = acc0[y], v1 = acc1[y];
        out0[y] = v0 >= q ? v0 - q : v0;
        out1[y] = v1 >= q ? v1 - q : v1;
    }
    // no trailing cluster barrier: the last remote access to this CTA's smem
    // (a scatter) is ordered before the cluster sync inside fwd_core
}

struct ModDownArgs {
    const uint64_t* acc;      // [count][2][L+K][n]: Q limbs evaluations, P limbs coefficients
    const uint64_t* add0;     // optional, poly stride add_stride
    const uint64_t* add1;
    uint64_t add_stride;
    uint64_t add_galois;      // automorphism applied to add reads (0 = none)
    const uint64_t* sum0;     // optional second addend (no automorphism), poly stride sum_stride
    const uint64_t* sum1;
    uint64_t sum_stride;
    uint64_t* out0;
    uint64_t* out1;
    uint64_t out_stride;
    const ulonglong2* p_inv;  // [L] (P^-1 mod q_r, Shoup)
    uint32_t count;
};

template <int LOGN>
__global__ void __launch_bounds__(NttShape<LOGN>::T, kMinBlocks) moddown_kernel(BfvDev d, ModDownArgs a) {
    using S = NttShape<LOGN>;
    __shared__ __align__(16) uint64_t sm[S::M];
    const uint32_t LK = d.L + d.K;
    const uint32_t rank = S::CL > 1 ? cluster_rank() : 0;
    const uint32_t id = blockIdx.x / S::CL;
    const uint32_t r = id % d.L, h = (id / d.L) & 1, c = id / (2 * d.L);
    const PrimeDev& P = d.primes[r];
    const uint64_t q = P.q, two_q = 2 * q;
    const uint64_t n = 1ull << LOGN;
    const uint64_t* accp = a.acc + ((uint64_t(c) * 2 + h) * LK + d.L) * n;
    if (d.K == 1) {
        // [acc]_p (< p < 4 q_r) feeds the lazy transform unreduced
        fwd_core<LOGN>(sm, P, rank, [&](uint32_t x) { return __ldg(&accp[x]); });
    } else {
        // P limbs already hold y_l = [acc_l (P/p_l)^-1]_{p_l} (folded into the
        // inverse transform); sum_l y_l [P/p_l]_{q_r}, lazily in [0, 2q)
        fwd_core<LOGN>(sm, P, rank, [&](uint32_t x) {
            uint64_t v = 0;
            for (uint32_t l = 0; l < d.K; ++l) {
                const ulonglong2 w = d.phat_mod_sh[l * d.L + r];
                v = add_lazy2(v, mul_shoup_lazy(__ldg(&accp[(uint64_t(l) << LOGN) + x]), w.x, w.y, q), two_q);
            }
            return v;
        });
    }
    const uint32_t cta_base = rank * S::M;
    const uint64_t* accq = a.acc + ((uint64_t(c) * 2 + h) * LK + r) * n;
    const uint64_t* add = h ? a.add1 : a.add0;
    if (add) add += c * a.add_stride + (uint64_t(r) << LOGN);
    const uint64_t* sum = h ? a.sum1 : a.sum0;
    if (sum) sum += c * a.sum_stride + (uint64_t(r) << LOGN);
    uint64_t* out = (h ? a.out1 : a.out0) + c * a.out_stride + (uint64_t(r) << LOGN);
    const ulonglong2 pinv = a.p_inv[r];
    // Epilogue in two halves: issue every global load of a half (including
    // the automorphism gather, which hits scattered sectors) before using
    // any of them, so their latencies overlap.
    constexpr int kHalf = kE / 2;
#pragma unroll
    for (int part = 0; part < 2; ++part) {
        uint64_t va[kHalf], vb[kHalf], vs[kHalf];
#pragma unroll
        for (int jj = 0; jj < kHalf; ++jj) {
            const uint32_t x = cta_base + threadIdx.x + (part * kHalf + jj) * S::T;
            va[jj] = __ldg(&accq[x]);
            vb[jj] = add ? __ldg(&add[a.add_galois ? galois_src(x, a.add_galois, LOGN) : x]) : 0;
            vs[jj] = sum ? __ldg(&sum[x]) : 0;
        }
#pragma unroll
        for (int jj = 0; jj < kHalf; ++jj) {
            const uint32_t y = threadIdx.x + (part * kHalf + jj) * S::T;
            const uint64_t conv = reduce_4q(sm[swz(y)], q, two_q);
            uint64_t u = mul_shoup(va[jj] + q - conv, pinv.x, pinv.y, q);
            u = add_mod(u, vb[jj], q);
            u = add_mod(u, vs[jj], q);
            out[cta_base + y] = u;
        }
    }
}

}  // namespace lb
