// Batched negacyclic NTT / INTT over RNS limbs, sm_100a.
//
// Replaces NttTables::forward / inverse (proj/src/ring.cpp:73-115): same
// primitive 2N-th root psi (smallest-base search, proj/src/modular.cpp:44-56),
// same evaluation points psi^(2k+1). The device transform leaves evaluations
// in BIT-REVERSED order: out[bitrev(k)] = a(psi^(2k+1)); the C-ABI documents
// the mapping and every NTT-domain permutation (slots, automorphisms) is
// expressed in it.
//
// Work decomposition (one limb = N u64 = 128 KiB at N=16384):
//   * a thread-block CLUSTER of CL = max(1, N/4096) CTAs owns one limb; each
//     CTA keeps N/CL contiguous coefficients (32 KiB) in shared memory, so
//     several limbs are resident per SM and loads of one overlap the
//     butterflies of another;
//   * every thread holds 16 coefficients in registers and runs 4 radix-2
//     stages per shared-memory round trip (radix-16 passes);
//   * the one pass whose butterflies span CTAs goes through distributed
//     shared memory (st/ld.shared::cluster) — forward: stages 0-3 read
//     straight from HBM and scatter into the owners' smem; inverse: stages
//     3-0 gather from the owners' smem and write straight to HBM;
//   * shared memory is padded (32-bit words: conflict-free, accesses as base
//     + immediate) or XOR-swizzled (64-bit words), see Lay below;
//   * on 32-bit words a cluster runs TWO limbs of the same prime side by
//     side (NT = 2): twiddles, addresses and the exchange are shared;
//   * butterflies are Harvey lazy Cooley-Tukey / Gentleman-Sande with Shoup
//     twiddles, values kept in [0, 4q) and reduced once at the end.
#pragma once

#include <cooperative_groups.h>
#include <cstdint>
#include <type_traits>

#include "modarith.cuh"

namespace lb {

// Per-prime device tables. fwd[i] = (psi^bitrev(i), shoup), inv[i] =
// (psi^-bitrev(i), shoup) with bitrev over log2 N bits; inv_last = twiddles
// of stage 0 premultiplied by n^-1 (index 0: n^-1 itself, index 1:
// psi^-bitrev(1) * n^-1).
struct PrimeDev {
    uint64_t q;
    uint64_t ratio_lo, ratio_hi;
    const ulonglong2* fwd;
    const ulonglong2* inv;
    uint64_t ninv, ninv_shoup;
    uint64_t inv1n, inv1n_shoup;  // psi^-bitrev(1) * n^-1
    // 32-bit copies for primes below 2^30 (NULL otherwise): Shoup companions
    // floor(w * 2^32 / q), used by the 32-bit word kernels
    const uint2* fwd32;
    const uint2* inv32;
    uint2 ninv32, inv1n32;
};

// Arithmetic word of a kernel instance. A batch whose primes are all below
// 2^30 is transformed with 32-bit words (values < 4q < 2^32, one IMAD.HI +
// two IMADs per Shoup product instead of the ~14-instruction 64-bit
// emulation); its storage word St is u32 (ciphertexts of such a context,
// key-switch intermediates) or u64 (the generic limb-batch API).
template <class W> struct WordT;
template <> struct WordT<uint64_t> { using Pair = ulonglong2; };
template <> struct WordT<uint32_t> { using Pair = uint2; };
template <class W> using PairT = typename WordT<W>::Pair;

__device__ __forceinline__ uint32_t mulhi_w(uint32_t a, uint32_t b) { return __umulhi(a, b); }
__device__ __forceinline__ uint64_t mulhi_w(uint64_t a, uint64_t b) { return __umul64hi(a, b); }

// x * w mod q in [0, 2q) for any word x (Shoup, companion wp).
template <class W>
__device__ __forceinline__ W shoup_lazy(W x, W w, W wp, W q) { return x * w - mulhi_w(x, wp) * q; }

// x >= m ? x - m : x for x < 2m: x - m wraps above x exactly when x < m, so
// the unsigned minimum picks the right value. Compiles to one VIADDMNMX.U32
// for 32-bit words (vs ISETP + SEL + IADD).
template <class W>
__device__ __forceinline__ W csub(W x, W m) { return min(x, static_cast<W>(x - m)); }

template <class W>
__device__ __forceinline__ W shoup_full(W x, W w, W wp, W q) { return csub<W>(shoup_lazy(x, w, wp, q), q); }

template <class W> __device__ __forceinline__ const PairT<W>* fwd_table(const PrimeDev& P);
template <> __device__ __forceinline__ const ulonglong2* fwd_table<uint64_t>(const PrimeDev& P) { return P.fwd; }
template <> __device__ __forceinline__ const uint2* fwd_table<uint32_t>(const PrimeDev& P) { return P.fwd32; }
template <class W> __device__ __forceinline__ const PairT<W>* inv_table(const PrimeDev& P);
template <> __device__ __forceinline__ const ulonglong2* inv_table<uint64_t>(const PrimeDev& P) { return P.inv; }
template <> __device__ __forceinline__ const uint2* inv_table<uint32_t>(const PrimeDev& P) { return P.inv32; }
template <class W> __device__ __forceinline__ PairT<W> ninv_pair(const PrimeDev& P);
template <> __device__ __forceinline__ ulonglong2 ninv_pair<uint64_t>(const PrimeDev& P) {
    return make_ulonglong2(P.ninv, P.ninv_shoup);
}
template <> __device__ __forceinline__ uint2 ninv_pair<uint32_t>(const PrimeDev& P) { return P.ninv32; }
template <class W> __device__ __forceinline__ PairT<W> inv1n_pair(const PrimeDev& P);
template <> __device__ __forceinline__ ulonglong2 inv1n_pair<uint64_t>(const PrimeDev& P) {
    return make_ulonglong2(P.inv1n, P.inv1n_shoup);
}
template <> __device__ __forceinline__ uint2 inv1n_pair<uint32_t>(const PrimeDev& P) { return P.inv1n32; }

// Descriptor of a batch of RNS polynomials laid out [poly][limb][N]:
// limb l of every poly uses prime first_prime + l.
// Optional prime_map: limb_id -> prime index = prime_map[limb_id % map_period]
// (negative = leave that limb untouched), for batches whose limbs do not map
// to one contiguous prime range (Q then B, or the per-digit key-switch
// extensions that skip the digit's own primes).
struct LimbBatch {
    uint64_t* data;
    uint32_t polys;
    uint32_t limbs;        // limbs per poly
    uint32_t first_prime;  // index into the context prime table
    uint64_t poly_stride;  // elements between consecutive polys (>= limbs*N)
    const int16_t* prime_map = nullptr;
    uint32_t map_period = 0;
    // inverse transform only: read the input from `src` (same [poly][limb]
    // shape and word as `data`, poly stride src_stride) instead of in place, optionally through
    // the automorphism x -> x^galois on the evaluations (galois 0 = none).
    const uint64_t* src = nullptr;
    uint64_t src_stride = 0;
    uint64_t galois = 0;
    // inverse transform only: per limb position l (< limbs), the final-stage
    // constants {n^-1 * s_l, psi^-bitrev(1) * n^-1 * s_l} as (value, Shoup)
    // pairs, which scale the output by s_l for free (NULL = s_l = 1);
    // last_stage32 is the same for the 32-bit word path.
    const ulonglong2* last_stage = nullptr;
    const uint2* last_stage32 = nullptr;
    // prime_map batches only: every mapped prime is below 2^30 (the caller
    // knows; contiguous batches are checked on the host)
    bool map_small = false;
    // `data` holds u32 residues (32-bit word batches only; strides in
    // elements): the key switch keeps its intermediates packed
    bool packed32 = false;
};

// Kernel-parameter copy of what a 32-bit word transform needs before its
// first butterfly: q and the twiddle-table slot of every prime of the
// context. Read from the constant bank by prime index, so the twiddle and
// data loads of a CTA issue at once instead of behind a dependent global
// load of the PrimeDev entry. Contexts with more than kTabPrimes primes run
// on 64-bit words (Context::word32_enabled).
constexpr int kTabPrimes = 64;
struct PrimeTab32 {
    const uint2* tw = nullptr;  // slot s: fwd32[n] then inv32[n] at tw + s * 2n
    uint32_t count = 0;
    uint32_t q[kTabPrimes] = {};
    uint8_t slot[kTabPrimes] = {};
};

// What the transform cores read of a prime.
template <class W>
struct PrimeView {
    W q;
    const PairT<W>* fwd;
    const PairT<W>* inv;
};

template <class W>
__device__ __forceinline__ PrimeView<W> prime_view(const PrimeDev& P) {
    if constexpr (sizeof(W) == 8)
        return PrimeView<W>{P.q, P.fwd, P.inv};
    else
        return PrimeView<W>{static_cast<W>(P.q), P.fwd32, P.inv32};
}

template <class W, int LOGN>
__device__ __forceinline__ PrimeView<W> prime_view(const PrimeTab32& tab, const PrimeDev* __restrict__ primes, int pidx) {
    if constexpr (sizeof(W) == 4) {
        // 32-bit word kernels only run on contexts that filled the table
        const uint2* base = tab.tw + (static_cast<size_t>(tab.slot[pidx]) << (LOGN + 1));
        return PrimeView<W>{tab.q[pidx], base, base + (1u << LOGN)};
    } else {
        return prime_view<W>(primes[pidx]);
    }
}

// Linear block index over grid.y/z (work items beyond 65535 spill into z).
__device__ __forceinline__ uint32_t block_yz() { return blockIdx.z * gridDim.y + blockIdx.y; }

// Evaluation-domain source position of x under x -> x^g (bit-reversed order).
// g < 2n <= 2^16 and 2k + 1 < 2n, so the product fits 32 bits.
__device__ __forceinline__ uint32_t galois_src(uint32_t x, uint64_t g, int logn) {
    const uint32_t n = 1u << logn;
    const uint32_t k = __brev(x) >> (32 - logn);
    const uint32_t e = (static_cast<uint32_t>(g) * (2u * k + 1u)) & (2u * n - 1u);
    return __brev((e - 1u) >> 1) >> (32 - logn);
}

#ifndef LB_NTT_LOGE
#define LB_NTT_LOGE 4  // radix 32 (LOGE 5, 128 threads) measured slower on B200: 481 vs 512 Gbfly/s
#endif
constexpr int kLogE = LB_NTT_LOGE;     // 2^kLogE coefficients per thread (radix of a register pass)
constexpr int kE = 1 << kLogE;
#ifndef LB_CTA_COEFFS
#define LB_CTA_COEFFS 4096
#endif
constexpr int kCtaCoeffs = LB_CTA_COEFFS;  // coefficients owned by one CTA
constexpr int kThreads = kCtaCoeffs / kE;  // 128 (radix 32) or 256 (radix 16)
constexpr int kMinBlocks = kThreads <= 128 ? 4 : kThreads == 256 ? 3 : 1;  // resident CTAs per SM the register budget must allow

// Shared-memory layouts of a CTA chunk.
//   u64 words (two banks each, 16 per 128-byte row): XOR swizzle
//     y ^ ((y >> 4) & 15), one LOP3 per access.
//   u32 words: PADDING, y + A * (y >> S) with (A, S) = (4, 6) — 4 pad words
//     after every 64 — or (2, 5) for n = 8192. By enumeration of every pass's
//     warp access pattern this is conflict-free for n = 8192 and 16384 (1.2
//     wavefronts per access at n = 32768, 1.25 at n = 4096; the XOR swizzle
//     y ^ ((y >> 5) & 31) used before averaged 1.38). Padding is affine: for
//     y = base + c with base and c bit-disjoint (every access below: a
//     thread-dependent base plus a compile-time multiple of a power-of-two
//     stride larger than the base's set bits) pad(y) = pad(base) + pad(c), so
//     an access is [base register + immediate] with no address instruction,
//     and a last-pass group of 2^C consecutive words stays contiguous and
//     aligned (one 8/16-byte access).
__device__ __forceinline__ uint32_t swz(uint32_t y) { return y ^ ((y >> 4) & 15u); }

template <class W, int LOGN>
struct Lay {
    static constexpr bool kPad = sizeof(W) == 4;
    static constexpr uint32_t A = LOGN == 13 ? 2 : 4, S = LOGN == 13 ? 5 : 6;
    __host__ __device__ static constexpr uint32_t idx(uint32_t y) {
        return kPad ? y + A * (y >> S) : (y ^ ((y >> 4) & 15u));
    }
    // words of a plane holding m logical words (m a multiple of 2^S)
    __host__ __device__ static constexpr uint32_t plane(uint32_t m) { return kPad ? m + A * (m >> S) : m; }
};

// Words of the smem plane of one CTA chunk.
template <int LOGN, class W>
constexpr uint32_t plane_words() {
    return Lay<W, LOGN>::plane(kCtaCoeffs < (1 << LOGN) ? kCtaCoeffs : (1 << LOGN));
}

// swb(): byte offset of a base, computed once per thread and pass;
// lay_add(sb, c): byte offset of base + c; sm_at<LOGN>(): the element.
template <class W, int LOGN>
__device__ __forceinline__ uint32_t swb(uint32_t base) {
    return Lay<W, LOGN>::idx(base) * static_cast<uint32_t>(sizeof(W));
}
template <class W, int LOGN>
__device__ __forceinline__ uint32_t lay_add(uint32_t sb, uint32_t c) {
    if constexpr (Lay<W, LOGN>::kPad)
        return sb + swb<W, LOGN>(c);
    else
        return sb ^ swb<W, LOGN>(c);
}
template <int LOGN, class W>
__device__ __forceinline__ W& sm_at(W* sm, uint32_t sb, uint32_t c) {
    return *reinterpret_cast<W*>(reinterpret_cast<char*>(sm) + lay_add<W, LOGN>(sb, c));
}

// A group of 2^C consecutive logical words at a 2^C-aligned base (byte
// offset sb): contiguous and aligned in the padded layout, so it moves as
// 8/16-byte accesses; element by element in the XOR layout.
template <int LOGN, int C, class W>
__device__ __forceinline__ void lds_group(const W* sm, uint32_t sb, W (&r)[1 << C]) {
    if constexpr (Lay<W, LOGN>::kPad && C >= 2) {
#pragma unroll
        for (int k = 0; k < (1 << C); k += 4) {
            const uint4 v = *reinterpret_cast<const uint4*>(reinterpret_cast<const char*>(sm) + sb + k * 4);
            r[k] = v.x;
            r[k + 1] = v.y;
            r[k + 2] = v.z;
            r[k + 3] = v.w;
        }
    } else if constexpr (Lay<W, LOGN>::kPad && C == 1) {
        const uint2 v = *reinterpret_cast<const uint2*>(reinterpret_cast<const char*>(sm) + sb);
        r[0] = v.x;
        r[1] = v.y;
    } else {
#pragma unroll
        for (int k = 0; k < (1 << C); ++k) r[k] = sm_at<LOGN>(const_cast<W*>(sm), sb, k);
    }
}
template <int LOGN, int C, class W>
__device__ __forceinline__ void sts_group(W* sm, uint32_t sb, const W (&r)[1 << C]) {
    if constexpr (Lay<W, LOGN>::kPad && C >= 2) {
#pragma unroll
        for (int k = 0; k < (1 << C); k += 4)
            *reinterpret_cast<uint4*>(reinterpret_cast<char*>(sm) + sb + k * 4) = make_uint4(r[k], r[k + 1], r[k + 2], r[k + 3]);
    } else if constexpr (Lay<W, LOGN>::kPad && C == 1) {
        *reinterpret_cast<uint2*>(reinterpret_cast<char*>(sm) + sb) = make_uint2(r[0], r[1]);
    } else {
#pragma unroll
        for (int k = 0; k < (1 << C); ++k) sm_at<LOGN>(sm, sb, k) = r[k];
    }
}

// a + b kept on the ALU pipe. The 32-bit butterflies are bound by the FMA
// pipe (IMAD.HI issues at half the IMAD rate on B200: 32 vs 64 lanes/clk/SM,
// tools/pipes.py), but ptxas balances pipes as if it were full rate and turns
// 2-input adds into IMAD.IADD. A third addend it cannot see through (a zero
// in constant memory) makes the add a 3-input IADD3, which IMAD cannot do.
#ifndef LB_ADD_ALU
#define LB_ADD_ALU 1
#endif
static __constant__ uint32_t kZero32 = 0;
template <class W>
__device__ __forceinline__ W add_alu(W a, W b) {
    if constexpr (sizeof(W) == 4 && LB_ADD_ALU)
        return a + b + kZero32;
    else
        return a + b;
}

// Harvey lazy CT butterfly: X, Y in [0, 4q) -> X + WY, X - WY in [0, 4q).
template <class W, class Pr>
__device__ __forceinline__ void ct_bfly(W& x, W& y, Pr w, W q, W two_q) {
    W xx = csub<W>(x, two_q);
    W t = shoup_lazy<W>(y, w.x, w.y, q);
    x = add_alu<W>(xx, t);
    y = xx - t + two_q;
}

// Harvey lazy GS butterfly: X, Y in [0, 2q) -> X + Y, (X - Y) W in [0, 2q).
template <class W, class Pr>
__device__ __forceinline__ void gs_bfly(W& x, W& y, Pr w, W q, W two_q) {
    W s = add_alu<W>(x, y);
    s = csub<W>(s, two_q);
    W d = x - y + two_q;
    x = s;
    y = shoup_lazy<W>(d, w.x, w.y, q);
}

template <class W>
__device__ __forceinline__ W reduce_4q(W v, W q, W two_q) {
    return csub<W>(csub<W>(v, two_q), q);
}

// Forward radix-2^C pass over one group held in r[0..2^C): global stages
// s0 .. s0+C-1, B = global block index at stage s0.
// The 2^l twiddles of stage l of a group are consecutive table entries at a
// 2^l-aligned index, so 32-bit (w, w') pairs load two per 16-byte LDG.128.
template <class W, int COUNT>
__device__ __forceinline__ void load_twiddles(const PairT<W>* __restrict__ p, PairT<W> (&t)[COUNT]) {
    if constexpr (sizeof(W) == 4 && COUNT >= 2) {
        const uint4* v = reinterpret_cast<const uint4*>(p);
#pragma unroll
        for (int i = 0; i < COUNT / 2; ++i) {
            const uint4 x = __ldg(&v[i]);
            t[2 * i] = make_uint2(x.x, x.y);
            t[2 * i + 1] = make_uint2(x.z, x.w);
        }
    } else {
#pragma unroll
        for (int i = 0; i < COUNT; ++i) t[i] = __ldg(&p[i]);
    }
}

// stage Lv of a radix-2^C group (compile-time Lv so the twiddle array is
// sized) over NT transforms of the SAME prime held side by side in registers:
// every twiddle is loaded once and applied to all NT (r[u] = transform u).
template <int C, int Lv, bool INVERSE, class W, int NT>
__device__ __forceinline__ void group_stage(W (&r)[NT][1 << C], const PairT<W>* __restrict__ tw, uint32_t s0,
                                            uint32_t B, W q, W two_q) {
    constexpr int half = 1 << (C - 1 - Lv);
    PairT<W> t[1 << Lv];
    load_twiddles<W>(tw + (1u << (s0 + Lv)) + (B << Lv), t);
#pragma unroll
    for (int k = 0; k < (1 << C); ++k) {
        if (k & half) continue;
#pragma unroll
        for (int u = 0; u < NT; ++u) {
            if constexpr (INVERSE)
                gs_bfly(r[u][k], r[u][k + half], t[k >> (C - Lv)], q, two_q);
            else
                ct_bfly(r[u][k], r[u][k + half], t[k >> (C - Lv)], q, two_q);
        }
    }
}

template <int C, int Lv, class W, int NT>
__device__ __forceinline__ void fwd_stages(W (&r)[NT][1 << C], const PairT<W>* __restrict__ tw, uint32_t s0,
                                           uint32_t B, W q, W two_q) {
    group_stage<C, Lv, false, W, NT>(r, tw, s0, B, q, two_q);
    if constexpr (Lv + 1 < C) fwd_stages<C, Lv + 1, W, NT>(r, tw, s0, B, q, two_q);
}

// stages Lv down to LAST (inclusive)
template <int C, int Lv, int LAST, class W, int NT>
__device__ __forceinline__ void inv_stages(W (&r)[NT][1 << C], const PairT<W>* __restrict__ tw, uint32_t s0,
                                           uint32_t B, W q, W two_q) {
    group_stage<C, Lv, true, W, NT>(r, tw, s0, B, q, two_q);
    if constexpr (Lv > LAST) inv_stages<C, Lv - 1, LAST, W, NT>(r, tw, s0, B, q, two_q);
}

template <int C, class W, int NT>
__device__ __forceinline__ void fwd_group(W (&r)[NT][1 << C], const PairT<W>* __restrict__ tw, uint32_t s0,
                                          uint32_t B, W q, W two_q) {
    fwd_stages<C, 0, W, NT>(r, tw, s0, B, q, two_q);
}
template <int C, class W, int NT>
__device__ __forceinline__ void inv_group(W (&r)[NT][1 << C], const PairT<W>* __restrict__ tw, uint32_t s0,
                                          uint32_t B, W q, W two_q) {
    inv_stages<C, C - 1, 0, W, NT>(r, tw, s0, B, q, two_q);
}

// One local radix-2^C pass over the CTA's smem chunk (global stages
// s0..s0+C-1; every block at stage s0 lies inside one CTA).
// NT > 1: transform u lives in the plane at sm + u * (chunk words).
template <int LOGN, int C, bool INVERSE, class W, int NT = 1>
__device__ __forceinline__ void local_pass(W* sm, const PairT<W>* __restrict__ tw, uint32_t s0, uint32_t cta_base,
                                           W q, W two_q) {
    constexpr int G = kE >> C;  // groups per thread
    constexpr uint32_t kPlane = plane_words<LOGN, W>();
    const uint32_t stride = (1u << LOGN) >> (s0 + C);
    const uint32_t log_bs = LOGN - s0;
#pragma unroll
    for (int i = 0; i < G; ++i) {
        const uint32_t g = threadIdx.x + i * kThreads;
        const uint32_t b = g / stride, o = g % stride;
        const uint32_t base = (b << log_bs) + o;
        const uint32_t B = (cta_base >> log_bs) + b;
        // base has no bits in [log2 stride, log_bs), where k * stride lives
        const uint32_t sb = swb<W, LOGN>(base);
        W r[NT][1 << C];
#pragma unroll
        for (int u = 0; u < NT; ++u)
#pragma unroll
            for (int k = 0; k < (1 << C); ++k) r[u][k] = sm_at<LOGN>(sm + u * kPlane, sb, k * stride);
        if (INVERSE)
            inv_group<C>(r, tw, s0, B, q, two_q);
        else
            fwd_group<C>(r, tw, s0, B, q, two_q);
#pragma unroll
        for (int u = 0; u < NT; ++u)
#pragma unroll
            for (int k = 0; k < (1 << C); ++k) sm_at<LOGN>(sm + u * kPlane, sb, k * stride) = r[u][k];
    }
}

// local pass of C stages, C chosen at run time among 1..kLogE
template <int LOGN, bool INVERSE, int NT = 1, int C = kLogE, class W>
__device__ __forceinline__ void local_pass_n(int c, W* sm, const PairT<W>* __restrict__ tw, uint32_t s0,
                                             uint32_t cta_base, W q, W two_q) {
    if constexpr (C >= 1) {
        if (c == C)
            local_pass<LOGN, C, INVERSE, W, NT>(sm, tw, s0, cta_base, q, two_q);
        else
            local_pass_n<LOGN, INVERSE, NT, C - 1, W>(c, sm, tw, s0, cta_base, q, two_q);
    }
}

template <int LOGN>
struct NttShape {
    static constexpr int N = 1 << LOGN;
    static constexpr int CL = N > kCtaCoeffs ? N / kCtaCoeffs : 1;
    static constexpr int M = N / CL;           // coefficients per CTA
    static constexpr int T = M / kE;           // threads per CTA
    static constexpr int PER_CTA = kE / CL;    // first-pass outputs each CTA receives per thread group
    static constexpr int NE = N / kE;          // stride of the cross-CTA pass
};

// Prime-table index of limb l of a poly, or -1 when the limb is to be
// skipped (the division only on mapped batches, which are off the hot path).
template <bool MAPPED>
__device__ __forceinline__ int prime_index(const LimbBatch& b, uint32_t poly, uint32_t l) {
    if constexpr (MAPPED)
        return b.prime_map[(poly * b.limbs + l) % b.map_period];
    else
        return static_cast<int>(b.first_prime + l);  // stays a uniform value
}

template <class St = uint64_t>
__device__ __forceinline__ St* limb_ptr(const LimbBatch& b, uint32_t poly, uint32_t l, int logn) {
    return reinterpret_cast<St*>(b.data) + (uint64_t)poly * b.poly_stride + ((uint64_t)l << logn);
}

__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.aligned;\n" ::: "memory"); }
// No release fence: for barriers that only order this CTA's earlier smem
// READS (whose values are already consumed) before peers' remote writes, or
// keep this CTA resident until peers finish reading it.
__device__ __forceinline__ void cluster_arrive_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory"); }

// ---- transaction-count mbarriers for the cross-CTA pass ------------------------------
// The forward transform's first pass scatters every thread's 16 outputs over
// the cluster. Instead of a cluster-wide barrier (release fence + all-CTA
// rendezvous) after the scatter, remote values travel as st.async stores
// that complete_tx on the RECEIVER's mbarrier; each CTA waits only until its
// own chunk has arrived (its threads' local stores counted as arrivals).
#ifndef LB_NTT_MBAR
#define LB_NTT_MBAR 1
#endif
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* m, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(m)), "r"(count) : "memory");
}
// makes mbarrier inits visible to the cluster (pairs with the start barrier)
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
__device__ __forceinline__ uint32_t mapa_rank(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_async(uint32_t raddr, uint32_t v, uint32_t rmbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];\n" ::"r"(raddr), "r"(v),
                 "r"(rmbar)
                 : "memory");
}
__device__ __forceinline__ void st_async(uint32_t raddr, uint64_t v, uint32_t rmbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];\n" ::"r"(raddr), "l"(v),
                 "r"(rmbar)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t m) {
    asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(m) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint32_t m, uint32_t tx) {
    asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(m), "r"(tx)
                 : "memory");
}
#ifndef LB_MBAR_HINT
#define LB_MBAR_HINT 0  // try_wait suspend-time hint in ns (0 = the hardware default)
#endif
__device__ __forceinline__ void mbar_wait(uint32_t m, uint32_t parity) {
#if LB_MBAR_HINT
    asm volatile(
        "{\n .reg .pred p;\n LB_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        " @!p bra LB_WAIT_%=;\n}\n" ::"r"(m),
        "r"(parity), "n"(LB_MBAR_HINT)
        : "memory");
#else
    asm volatile(
        "{\n .reg .pred p;\n LB_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra LB_WAIT_%=;\n}\n" ::"r"(m),
        "r"(parity)
        : "memory");
#endif
}

// Bulk L2 prefetch by the TMA unit (one instruction for a whole range):
// kernels whose epilogue streams operands that do not feed the transform
// issue it at entry, so those reads hit L2 instead of HBM.
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}

// Exchange state of one forward transform: this CTA's mbarrier (shared
// address; 0 = use the cluster barrier instead) and the phase parity to wait
// for. Kernels init one mbarrier per concurrently live smem plane with
// count = threads per CTA before their first transform.
struct Xchg {
    uint32_t mbar = 0;
    uint32_t parity = 0;
};

// Thread 0 inits `count` mbarriers (expected arrivals: every thread of the
// CTA); visible to the cluster after the first transform's start barrier.
// Returns the exchange state of mbarrier 0 (none for single-CTA limbs).
template <int CL>
__device__ __forceinline__ Xchg xchg_init(uint64_t* mbar, int count) {
    if constexpr (CL > 1 && LB_NTT_MBAR) {
        if (threadIdx.x == 0) {
            for (int i = 0; i < count; ++i) mbar_init(&mbar[i], blockDim.x);
            mbar_fence_init();
        }
        return Xchg{smem_addr(mbar), 0};
    } else {
        return Xchg{};
    }
}

// Forward transform core, shared by the plain and the fused kernels. The
// cluster's CTAs cooperatively transform one limb: `load(rho, off)` supplies
// input coefficient rho + off (any value < 4q, so loaders may skip their
// final reduction); off is a compile-time multiple of n/16 and rho the
// thread's fixed lane, so loaders address from `base + rho` with immediate
// offsets,
// and on return the CTA's chunk [rank*M, (rank+1)*M) of the bit-reversed
// evaluations sits in `sm` (swizzled, values in [0, 4q)).
// Callers looping over several transforms must cluster-sync between them
// (peers scatter into this CTA's smem).
// start_sync = false skips the barrier that protects `sm` from being
// overwritten while still being read: for callers whose transforms each write
// a fresh smem plane after a first synchronised one.
// The forward transform's last local pass: stages LOGN-kLast .. LOGN-1 over
// groups of 2^kLast consecutive evaluations (stride 1), handed to
// last(base, r) in registers (chunk-local base, r[k] < 4q at base + k)
// instead of going back to smem: epilogues that stream the result out skip a
// store, a barrier and a reload.
template <int LOGN>
constexpr int fwd_last_radix() { return (LOGN % kLogE) == 0 ? kLogE : LOGN % kLogE; }

// An epilogue object with prefetch(base) -> Ops and finish(base, r, ops)
// gets its global operands for group i + 1 issued before group i's
// butterflies (one group of software pipelining), so their latency overlaps
// compute instead of stalling the epilogue; a plain callable last(base, r)
// loads on use.
template <class T, class = void>
struct has_prefetch : std::false_type {};
template <class T>
struct has_prefetch<T, std::void_t<decltype(&std::decay_t<T>::prefetch)>> : std::true_type {};

template <int LOGN, int NT, class W, class Last>
__device__ __forceinline__ void fwd_last_pass(W* sm, const PairT<W>* __restrict__ tw, uint32_t cta_base, W q,
                                              W two_q, Last&& last) {
    constexpr int C = fwd_last_radix<LOGN>();
    constexpr int G = kE >> C;
    constexpr uint32_t s0 = LOGN - C;
    constexpr uint32_t kPlane = plane_words<LOGN, W>();
    if constexpr (has_prefetch<Last>::value && NT == 1) {
        auto ops = last.prefetch(threadIdx.x << C);
#pragma unroll
        for (int i = 0; i < G; ++i) {
            const uint32_t g = threadIdx.x + i * kThreads;
            const uint32_t base = g << C;
            decltype(ops) nxt = ops;
            if (i + 1 < G) nxt = last.prefetch((g + kThreads) << C);
            const uint32_t sb = swb<W, LOGN>(base);
            W r[1][1 << C];
            lds_group<LOGN, C>(sm, sb, r[0]);
            fwd_group<C>(r, tw, s0, (cta_base >> C) + g, q, two_q);
            last.finish(base, r[0], ops);
            ops = nxt;
        }
    } else {
#pragma unroll
        for (int i = 0; i < G; ++i) {
            const uint32_t g = threadIdx.x + i * kThreads;
            const uint32_t base = g << C;
            const uint32_t sb = swb<W, LOGN>(base);
            W r[NT][1 << C];
#pragma unroll
            for (int u = 0; u < NT; ++u) lds_group<LOGN, C>(sm + u * kPlane, sb, r[u]);
            fwd_group<C>(r, tw, s0, (cta_base >> C) + g, q, two_q);
#pragma unroll
            for (int u = 0; u < NT; ++u) last(u, base, r[u]);
        }
    }
}

// NT transforms of the same prime side by side (twiddles, addresses and the
// exchange handshake shared): transform u is loaded with load(u, rho, off),
// lives in the plane at sm + u * M and ends in last(u, base, r).
template <int LOGN, int NT = 1, class W, class Load, class Last = std::nullptr_t>
__device__ __forceinline__ void fwd_core(W* sm, const PrimeView<W>& P, uint32_t rank, Load&& load,
                                         bool start_sync = true, Xchg xc = Xchg{}, Last&& last = nullptr) {
    using S = NttShape<LOGN>;
    namespace cg = cooperative_groups;
    constexpr uint32_t kPlane = plane_words<LOGN, W>();
    const W q = P.q, two_q = 2 * q;
    const PairT<W>* __restrict__ tw = P.fwd;
    // Every CTA of the cluster must be running (and done reading its smem)
    // before peers write into it: arrive now, wait before the remote stores.
    if constexpr (S::CL > 1) {
        if (start_sync) cluster_arrive_relaxed();
    }
    {
        const uint32_t rho = rank * S::T + threadIdx.x;
        W r[NT][kE];
#pragma unroll
        for (int u = 0; u < NT; ++u)
#pragma unroll
            for (int k = 0; k < kE; ++k) r[u][k] = static_cast<W>(load(u, rho, k * S::NE));
        fwd_group<kLogE>(r, tw, 0, 0, q, two_q);
        if (start_sync) {
            if constexpr (S::CL > 1) cluster_wait();
            else __syncthreads();
        }
        const uint32_t sb = swb<W, LOGN>(rho);  // rho < NE
        if constexpr (S::CL > 1 && LB_NTT_MBAR) {
            const uint32_t lbase = smem_addr(sm);
#pragma unroll
            for (int dst = 0; dst < S::CL; ++dst) {
                if (dst == static_cast<int>(rank)) {
#pragma unroll
                    for (int u = 0; u < NT; ++u)
#pragma unroll
                        for (int i = 0; i < S::PER_CTA; ++i)
                            sm_at<LOGN>(sm + u * kPlane, sb, i * S::NE) = r[u][dst * S::PER_CTA + i];
                } else {
                    const uint32_t rbase = mapa_rank(lbase, dst), rmbar = mapa_rank(xc.mbar, dst);
#pragma unroll
                    for (int u = 0; u < NT; ++u)
#pragma unroll
                        for (int i = 0; i < S::PER_CTA; ++i)
                            st_async(rbase + u * static_cast<uint32_t>(kPlane * sizeof(W)) + lay_add<W, LOGN>(sb, i * S::NE),
                                     r[u][dst * S::PER_CTA + i], rmbar);
                }
            }
        } else {
#pragma unroll
            for (int u = 0; u < NT; ++u)
#pragma unroll
                for (int k = 0; k < kE; ++k) {
                    const uint32_t dst = k / S::PER_CTA;
                    const uint32_t c = (k % S::PER_CTA) * S::NE;
                    if constexpr (S::CL > 1) {
                        W* remote = cg::this_cluster().map_shared_rank(sm + u * kPlane, dst);
                        sm_at<LOGN>(remote, sb, c) = r[u][k];
                    } else {
                        sm_at<LOGN>(sm + u * kPlane, sb, c) = r[u][k];
                    }
                }
        }
    }
    if constexpr (S::CL > 1) {
        if constexpr (LB_NTT_MBAR) {
            // remote bytes this CTA receives: PER_CTA words from every thread of
            // every peer
            constexpr uint32_t kRemoteBytes = NT * (S::CL - 1) * S::T * S::PER_CTA * sizeof(W);
            if (threadIdx.x == 0)
                mbar_arrive_tx(xc.mbar, kRemoteBytes);
            else
                mbar_arrive(xc.mbar);
            mbar_wait(xc.mbar, xc.parity);
        } else {
            cg::this_cluster().sync();
        }
    } else {
        __syncthreads();
    }
    const uint32_t cta_base = rank * S::M;
    constexpr bool kDirect = !std::is_same_v<std::decay_t<Last>, std::nullptr_t>;
    constexpr int kEnd = kDirect ? LOGN - fwd_last_radix<LOGN>() : LOGN;
#pragma unroll
    for (int s0 = kLogE; s0 < kEnd; s0 += kLogE) {
        local_pass_n<LOGN, false, NT>(LOGN - s0 < kLogE ? LOGN - s0 : kLogE, sm, tw, s0, cta_base, q, two_q);
        __syncthreads();
    }
    if constexpr (kDirect) fwd_last_pass<LOGN, NT, W>(sm, tw, cta_base, q, two_q, last);
}

__device__ __forceinline__ uint32_t cluster_rank() {
    namespace cg = cooperative_groups;
    return cg::this_cluster().block_rank();
}

// grid = (CL * limbs, polys split over y and z); cluster dims (CL, 1, 1).
#ifndef LB_NTT32_MINB
#define LB_NTT32_MINB 5  // 51 registers: 146.3 vs 145.0 img/s at 4 CTAs/SM
#endif
// Paired transforms (NT = 2, 32-bit words): a cluster runs limb l of polys
// 2p and 2p + 1 side by side, so twiddle loads, smem addresses and the
// exchange handshake are paid once for two transforms and every warp carries
// two independent butterfly chains. Registers per thread allow one CTA less
// per SM than the single-transform instance, which still means more
// transforms in flight per SM.
#ifndef LB_NTT_PAIR_MINB
#define LB_NTT_PAIR_MINB 5  // 51 registers: forward 0.63 vs 0.61 of the roof at 4 CTAs/SM
#endif
template <class W, int NT = 1> constexpr int ntt_min_blocks() {
    return sizeof(W) == 8 ? kMinBlocks : NT == 1 ? LB_NTT32_MINB : LB_NTT_PAIR_MINB;
}

template <int LOGN, class W, class St = uint64_t, bool MAPPED = false, int NT = 1>
__global__ void __launch_bounds__(NttShape<LOGN>::T, ntt_min_blocks<W, NT>()) ntt_forward_kernel(LimbBatch b, const PrimeDev* __restrict__ primes,
                                                                                                     const __grid_constant__ PrimeTab32 tab) {
    using S = NttShape<LOGN>;
    __shared__ __align__(16) W sm[NT * plane_words<LOGN, W>()];
    const uint32_t rank = S::CL > 1 ? cluster_rank() : 0;
    const uint32_t l = blockIdx.x / S::CL, poly = block_yz() * NT;
    if (poly >= b.polys) return;  // whole cluster skips together (polys is a multiple of NT)
    const int pidx = prime_index<MAPPED>(b, poly, l);
    if (pidx < 0) return;
    const PrimeView<W> P = prime_view<W, LOGN>(tab, primes, pidx);
    St* __restrict__ a = limb_ptr<St>(b, poly, l, LOGN);
    __shared__ uint64_t mbar;
    const Xchg xc = xchg_init<S::CL>(&mbar, 1);
    const W q = P.q, two_q = 2 * q;
    // the last pass's groups (consecutive evaluations) stored straight from
    // registers, fully reduced (16-byte stores for radix-4 groups of u32)
    fwd_core<LOGN, NT>(
        sm, P, rank,
        [&](uint32_t u, uint32_t rho, uint32_t off) { return static_cast<W>(__ldcs(&(a + u * b.poly_stride + rho)[off])); },
        true, xc,
        [&](uint32_t u, uint32_t base, W(&r)[1 << fwd_last_radix<LOGN>()]) {
            St* out = a + u * b.poly_stride + rank * S::M;
            constexpr int C = fwd_last_radix<LOGN>();
            if constexpr (sizeof(St) == 4 && C == 2) {
                __stcs(reinterpret_cast<uint4*>(out + base),
                       make_uint4(reduce_4q<W>(r[0], q, two_q), reduce_4q<W>(r[1], q, two_q),
                                  reduce_4q<W>(r[2], q, two_q), reduce_4q<W>(r[3], q, two_q)));
            } else if constexpr (sizeof(St) == 8 && C >= 1) {
                // pairs of u64 as 16-byte stores (scalar 8-byte stores at a
                // 2^C-element lane stride would split every warp store)
#pragma unroll
                for (int k = 0; k < (1 << C); k += 2)
                    __stcs(reinterpret_cast<ulonglong2*>(out + base + k),
                           make_ulonglong2(reduce_4q<W>(r[k], q, two_q), reduce_4q<W>(r[k + 1], q, two_q)));
            } else {
#pragma unroll
                for (int k = 0; k < (1 << C); ++k) __stcs(&out[base + k], static_cast<St>(reduce_4q<W>(r[k], q, two_q)));
            }
        });
}

// Cross-CTA pass tail: stages 3, 2, 1 as usual; stage 0 with the scaled
// n^-1 pairs merged (c0 for the first half, c1 = psi^-bitrev(1) n^-1 s).
template <class W, int NT>
__device__ __forceinline__ void inv_final(W (&r)[NT][kE], const PairT<W>* __restrict__ tw, W q, PairT<W> c0,
                                          PairT<W> c1) {
    const W two_q = 2 * q;
    inv_stages<kLogE, kLogE - 1, 1, W, NT>(r, tw, 0, 0, q, two_q);
    constexpr int half0 = kE / 2;
#pragma unroll
    for (int u = 0; u < NT; ++u)
#pragma unroll
        for (int k = 0; k < half0; ++k) {
            W x = r[u][k], y = r[u][k + half0];
            W s = add_alu<W>(x, y);  // < 4q
            W d = x - y + two_q;
            r[u][k] = shoup_full<W>(s, c0.x, c0.y, q);
            r[u][k + half0] = shoup_full<W>(d, c1.x, c1.y, q);
        }
}

// The inverse's first (tail) pass, stages LOGN-1 .. LOGN-kTail, straight from
// global memory: its butterfly groups are 2^kTail consecutive coefficients
// (stride 1), so each group is one vector load (16 bytes for kTail = 2 on
// u32), and the results go to smem once — no staging store + reload of the
// input, and the loads overlap the groups' butterflies. load_group(u, y, r)
// fills r[0 .. 2^kTail) with chunk elements y .. y + 2^kTail - 1 of
// transform u (plane sm + u * M).
template <int LOGN, class W, int NT = 1, class LoadGroup>
__device__ __forceinline__ void inv_tail_pass(W* sm, const PrimeView<W>& P, uint32_t cta_base, LoadGroup&& load_group) {
    constexpr int kTail = (LOGN - kLogE) % kLogE;
    constexpr int G = kE >> kTail;  // groups per thread
    using S = NttShape<LOGN>;
    const W q = P.q, two_q = 2 * q;
    const PairT<W>* __restrict__ tw = P.inv;
    constexpr uint32_t s0 = LOGN - kTail;
#pragma unroll
    for (int i = 0; i < G; ++i) {
        const uint32_t g = threadIdx.x + i * S::T;
        const uint32_t base = g << kTail;
        W r[NT][1 << kTail];
#pragma unroll
        for (int u = 0; u < NT; ++u) load_group(u, base, r[u]);
        inv_group<kTail>(r, tw, s0, (cta_base >> kTail) + g, q, two_q);
        const uint32_t sb = swb<W, LOGN>(base);
#pragma unroll
        for (int u = 0; u < NT; ++u) sts_group<LOGN, kTail>(sm + u * plane_words<LOGN, W>(), sb, r[u]);
    }
}

// Push-based inverse transform core (cluster limbs, LB_NTT_MBAR). On entry
// `sm` holds this CTA's chunk after the tail pass (inv_tail_pass: stages
// LOGN-1 .. LOGN-kTail, swizzled, values < 2q, visible to every thread: the
// caller synchronised); `recv` is a fresh
// receive plane of M words and `mbar` this CTA's mbarrier for it (count =
// threads, phase `parity`). Peers must have initialised their mbarriers
// (start_wait: wait here on the cluster barrier the caller arrived on).
// On return r[k] = coefficient rho + k * NE (rho = rank * T + thread), fully
// reduced, scaled by the final-stage pairs c0 (n^-1 s) and c1.
// NT transforms: planes sm + u * M and recv + u * M, one mbarrier for all.
template <int LOGN, class W, int NT>
__device__ __forceinline__ void inv_core_push(W* sm, W* recv, uint32_t mbar, uint32_t parity, const PrimeView<W>& P,
                                              uint32_t rank, PairT<W> c0, PairT<W> c1, bool start_wait,
                                              W (&r)[NT][kE]) {
    using S = NttShape<LOGN>;
    static_assert(S::CL > 1, "push exchange needs a cluster");
    const W q = P.q, two_q = 2 * q;
    const PairT<W>* __restrict__ tw = P.inv;
    const uint32_t cta_base = rank * S::M;
    constexpr int kTail = (LOGN - kLogE) % kLogE;
    static_assert(kTail > 0, "cluster limbs have a tail pass");
#pragma unroll
    for (int s0 = LOGN - kTail - kLogE; s0 >= 2 * kLogE; s0 -= kLogE) {
        local_pass<LOGN, kLogE, true, W, NT>(sm, tw, s0, cta_base, q, two_q);
        __syncthreads();
    }
    // stages 7..4 (s0 = kLogE, one radix-16 group per thread): block bb,
    // offset o; element k (chunk index bb*NE + o + k*stride) belongs to
    // CTA k / PER_CTA, thread o + (k % PER_CTA) * stride, slot
    // (rank * PER_CTA + bb) of its receive plane
    constexpr uint32_t stride = S::N >> (2 * kLogE);
    static_assert(S::T % stride == 0 && S::T / stride == S::PER_CTA, "push layout");
    const uint32_t bb = threadIdx.x / stride, o = threadIdx.x % stride;
    const uint32_t sb = swb<W, LOGN>(bb * S::NE + o);
#pragma unroll
    for (int u = 0; u < NT; ++u)
#pragma unroll
        for (int k = 0; k < kE; ++k) r[u][k] = sm_at<LOGN>(sm + u * plane_words<LOGN, W>(), sb, k * stride);
    inv_group<kLogE>(r, tw, kLogE, (cta_base >> (LOGN - kLogE)) + bb, q, two_q);
    if (start_wait) cluster_wait();
    const uint32_t slot = (rank * S::PER_CTA + bb) * S::T + o;
    const uint32_t lrecv = smem_addr(recv + slot);
#pragma unroll
    for (int dst = 0; dst < S::CL; ++dst) {
        if (dst == static_cast<int>(rank)) {
#pragma unroll
            for (int u = 0; u < NT; ++u)
#pragma unroll
                for (int i = 0; i < S::PER_CTA; ++i) recv[u * S::M + slot + i * stride] = r[u][dst * S::PER_CTA + i];
        } else {
            const uint32_t rb = mapa_rank(lrecv, dst), rm = mapa_rank(mbar, dst);
#pragma unroll
            for (int u = 0; u < NT; ++u)
#pragma unroll
                for (int i = 0; i < S::PER_CTA; ++i)
                    st_async(rb + (u * S::M + i * stride) * static_cast<uint32_t>(sizeof(W)), r[u][dst * S::PER_CTA + i],
                             rm);
        }
    }
    constexpr uint32_t kRemoteBytes = NT * (S::CL - 1) * S::T * S::PER_CTA * sizeof(W);
    if (threadIdx.x == 0)
        mbar_arrive_tx(mbar, kRemoteBytes);
    else
        mbar_arrive(mbar);
    mbar_wait(mbar, parity);
#pragma unroll
    for (int u = 0; u < NT; ++u)
#pragma unroll
        for (int k = 0; k < kE; ++k) r[u][k] = recv[u * S::M + k * S::T + threadIdx.x];
    inv_final<W, NT>(r, tw, q, c0, c1);
}

// Paired push core on THREE planes (two chunks + one receive plane, 4 CTAs
// per SM instead of 3): the second transform's receive plane aliases the
// first transform's chunk, which is dead once every thread of the cluster has
// read it in its push pass — a second cluster barrier says so (arrive after
// the reads, wait before the second push, its latency behind the second
// transform's butterflies). The tail and local passes and the final stages
// stay paired (shared twiddles); the two push passes run one after the other.
// `mbar`: two consecutive mbarriers (count = threads), phase 0.
template <int LOGN, class W>
__device__ __forceinline__ void inv_core_push_alias(W* sm, W* recv0, uint32_t mbar, const PrimeView<W>& P,
                                                    uint32_t rank, PairT<W> c0, PairT<W> c1, W (&r)[2][kE]) {
    using S = NttShape<LOGN>;
    static_assert(S::CL > 1, "push exchange needs a cluster");
    const W q = P.q, two_q = 2 * q;
    const PairT<W>* __restrict__ tw = P.inv;
    const uint32_t cta_base = rank * S::M;
    constexpr int kTail = (LOGN - kLogE) % kLogE;
    static_assert(kTail > 0, "cluster limbs have a tail pass");
    constexpr uint32_t kPlane = plane_words<LOGN, W>();
    static_assert(kPlane >= S::M, "receive plane fits a chunk plane");
#pragma unroll
    for (int s0 = LOGN - kTail - kLogE; s0 >= 2 * kLogE; s0 -= kLogE) {
        local_pass<LOGN, kLogE, true, W, 2>(sm, tw, s0, cta_base, q, two_q);
        __syncthreads();
    }
    constexpr uint32_t stride = S::N >> (2 * kLogE);
    static_assert(S::T % stride == 0 && S::T / stride == S::PER_CTA, "push layout");
    const uint32_t bb = threadIdx.x / stride, o = threadIdx.x % stride;
    const uint32_t sb = swb<W, LOGN>(bb * S::NE + o);
    const uint32_t slot = (rank * S::PER_CTA + bb) * S::T + o;
    constexpr uint32_t kRemoteBytes = (S::CL - 1) * S::T * S::PER_CTA * sizeof(W);
    W* recv1 = sm;  // transform 1 lands in transform 0's chunk plane
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        W(&x)[1][kE] = reinterpret_cast<W(&)[1][kE]>(r[u]);
#pragma unroll
        for (int k = 0; k < kE; ++k) x[0][k] = sm_at<LOGN>(sm + u * kPlane, sb, k * stride);
        inv_group<kLogE>(x, tw, kLogE, (cta_base >> (LOGN - kLogE)) + bb, q, two_q);
        cluster_wait();  // u = 0: peers' mbarriers are initialised; u = 1: every chunk-0 read of the cluster is done
        W* recv = u ? recv1 : recv0;
        const uint32_t mb = mbar + 8 * u;
        const uint32_t lrecv = smem_addr(recv + slot);
#pragma unroll
        for (int dst = 0; dst < S::CL; ++dst) {
            if (dst == static_cast<int>(rank)) {
#pragma unroll
                for (int i = 0; i < S::PER_CTA; ++i) recv[slot + i * stride] = x[0][dst * S::PER_CTA + i];
            } else {
                const uint32_t rb = mapa_rank(lrecv, dst), rm = mapa_rank(mb, dst);
#pragma unroll
                for (int i = 0; i < S::PER_CTA; ++i)
                    st_async(rb + i * stride * static_cast<uint32_t>(sizeof(W)), x[0][dst * S::PER_CTA + i], rm);
            }
        }
        if (threadIdx.x == 0)
            mbar_arrive_tx(mb, kRemoteBytes);
        else
            mbar_arrive(mb);
        if (u == 0) cluster_arrive_relaxed();
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        mbar_wait(mbar + 8 * u, 0);
        const W* recv = u ? recv1 : recv0;
#pragma unroll
        for (int k = 0; k < kE; ++k) r[u][k] = recv[k * S::T + threadIdx.x];
    }
    inv_final<W, 2>(r, tw, q, c0, c1);
}

// Inverse transform. With LB_NTT_MBAR the cross-CTA pass is push-based: the
// last local pass (stages 7..4) sends its outputs straight from registers to
// the owning CTA's receive plane (st.async + complete_tx), so the owner waits
// on its own mbarrier instead of two cluster-wide barriers around remote
// loads. Dynamic smem: M words (+ M receive words when pushing).
template <int LOGN> constexpr bool inv_push() { return NttShape<LOGN>::CL > 1 && LB_NTT_MBAR; }
// (paired: two chunk planes and ONE receive plane, inv_core_push_alias)
template <int LOGN, class W, int NT = 1> constexpr size_t ntt_inverse_smem() {
    return (NT * plane_words<LOGN, W>() + (inv_push<LOGN>() ? NttShape<LOGN>::M : 0)) * sizeof(W);
}
#ifndef LB_INV_PAIR_MINB
#define LB_INV_PAIR_MINB 4  // 51 KiB per paired CTA
#endif
template <class W, int NT> constexpr int inv_min_blocks() {
    return NT == 1 ? ntt_min_blocks<W>() : LB_INV_PAIR_MINB;
}

template <int LOGN, class W, class St = uint64_t, bool MAPPED = false, int NT = 1>
__global__ void __launch_bounds__(NttShape<LOGN>::T, inv_min_blocks<W, NT>()) ntt_inverse_kernel(LimbBatch b, const PrimeDev* __restrict__ primes,
                                                                                                     const __grid_constant__ PrimeTab32 tab) {
    using S = NttShape<LOGN>;
    namespace cg = cooperative_groups;
    constexpr bool kPush = inv_push<LOGN>();
    static_assert(NT == 1 || kPush, "paired inverse transforms use the push exchange");
    extern __shared__ __align__(16) uint8_t inv_smem_raw[];
    W* sm = reinterpret_cast<W*>(inv_smem_raw);  // planes sm + u * M
    W* recv = sm + NT * plane_words<LOGN, W>();  // receive planes [kE][T], linear (push only)
    __shared__ uint64_t mbar[NT];
    const uint32_t rank = S::CL > 1 ? cg::this_cluster().block_rank() : 0;
    const uint32_t l = blockIdx.x / S::CL, poly = block_yz() * NT;
    if (poly >= b.polys) return;  // whole cluster skips together (polys is a multiple of NT)
    const int pidx = prime_index<MAPPED>(b, poly, l);
    if (pidx < 0) return;
    if constexpr (kPush) {
        xchg_init<S::CL>(mbar, NT);
        cluster_arrive_relaxed();  // peers may push once every mbarrier is initialised
    }
    const PrimeView<W> P = prime_view<W, LOGN>(tab, primes, pidx);
    const W q = P.q, two_q = 2 * q;
    St* __restrict__ a = limb_ptr<St>(b, poly, l, LOGN);
    const PairT<W>* __restrict__ tw = P.inv;
    const uint32_t cta_base = rank * S::M;

    const uint32_t sbt = swb<W, LOGN>(threadIdx.x);
    if constexpr (kPush) {
        // tail pass straight from global memory (through the automorphism
        // when reading a key switch's input)
        constexpr int kTail = (LOGN - kLogE) % kLogE;
        if (b.src) {
            const St* in = reinterpret_cast<const St*>(b.src) + uint64_t(poly) * b.src_stride + (uint64_t(l) << LOGN);
            inv_tail_pass<LOGN, W, NT>(sm, P, cta_base, [&](uint32_t u, uint32_t y, W (&r)[1 << kTail]) {
#pragma unroll
                for (int k = 0; k < (1 << kTail); ++k) {
                    const uint32_t x = cta_base + y + k;
                    r[k] = static_cast<W>(__ldg(&(in + u * b.src_stride)[b.galois ? galois_src(x, b.galois, LOGN) : x]));
                }
            });
        } else {
            const St* in = a + cta_base;
            inv_tail_pass<LOGN, W, NT>(sm, P, cta_base, [&](uint32_t u, uint32_t y, W (&r)[1 << kTail]) {
                const St* inu = in + u * b.poly_stride;
                if constexpr (sizeof(St) == 4 && kTail == 2) {
                    const uint4 v = __ldcs(reinterpret_cast<const uint4*>(inu + y));
                    r[0] = v.x;
                    r[1] = v.y;
                    r[2] = v.z;
                    r[3] = v.w;
                } else {
#pragma unroll
                    for (int k = 0; k < (1 << kTail); ++k) r[k] = static_cast<W>(__ldcs(&inu[y + k]));
                }
            });
        }
    } else if (b.src) {
        // src holds words of the batch's storage type (the key switch reads its
        // input ciphertext, stored in the context's residue word)
        const St* in = reinterpret_cast<const St*>(b.src) + uint64_t(poly) * b.src_stride + (uint64_t(l) << LOGN);
#pragma unroll
        for (int j = 0; j < kE; ++j) {
            const uint32_t y = threadIdx.x + j * S::T;
            const uint32_t x = cta_base + y;
            sm_at<LOGN>(sm, sbt, j * S::T) = static_cast<W>(__ldg(&in[b.galois ? galois_src(x, b.galois, LOGN) : x]));
        }
    } else {
        const St* in = a + cta_base;
#pragma unroll
        for (int j = 0; j < kE; ++j) {
            const uint32_t y = threadIdx.x + j * S::T;
            sm_at<LOGN>(sm, sbt, j * S::T) = static_cast<W>(__ldcs(&in[y]));
        }
    }
    __syncthreads();
    PairT<W> c0, c1;
    {
        const PairT<W>* last = nullptr;
        if constexpr (sizeof(W) == 8)
            last = b.last_stage;
        else
            last = b.last_stage32;
        if (last) {
            c0 = last[2 * l];
            c1 = last[2 * l + 1];
        } else {
            c0 = ninv_pair<W>(primes[pidx]);
            c1 = inv1n_pair<W>(primes[pidx]);
        }
    }
    const uint32_t rho = rank * S::T + threadIdx.x;
    W r[NT][kE];
    if constexpr (kPush) {
        if constexpr (NT == 2)
            inv_core_push_alias<LOGN, W>(sm, recv, smem_addr(mbar), P, rank, c0, c1, r);
        else
            inv_core_push<LOGN, W, NT>(sm, recv, smem_addr(mbar), 0, P, rank, c0, c1, true, r);
    } else {
        // local passes in reverse: the last (possibly short) chunk first
        constexpr int kTail = (LOGN - kLogE) % kLogE;
        if constexpr (kTail > 0) {
            local_pass<LOGN, kTail, true, W>(sm, tw, LOGN - kTail, cta_base, q, two_q);
            __syncthreads();
        }
#pragma unroll
        for (int s0 = LOGN - kTail - kLogE; s0 >= kLogE; s0 -= kLogE) {
            local_pass<LOGN, kLogE, true, W>(sm, tw, s0, cta_base, q, two_q);
            __syncthreads();
        }
        // cross-CTA pass: stages 3..0 gathered from the owners
        if constexpr (S::CL > 1) cg::this_cluster().sync();
        const uint32_t sb = swb<W, LOGN>(rho);  // rho < NE
#pragma unroll
        for (int k = 0; k < kE; ++k) {
            const uint32_t src = k / S::PER_CTA;
            const uint32_t c = (k % S::PER_CTA) * S::NE;
            if constexpr (S::CL > 1) {
                W* remote = cg::this_cluster().map_shared_rank(sm, src);
                r[0][k] = sm_at<LOGN>(remote, sb, c);
            } else {
                r[0][k] = sm_at<LOGN>(sm, sb, c);
            }
        }
        inv_final<W, NT>(r, tw, q, c0, c1);
    }
#pragma unroll
    for (int u = 0; u < NT; ++u)
#pragma unroll
        for (int k = 0; k < kE; ++k) __stcs(&(a + u * b.poly_stride)[rho + k * S::NE], static_cast<St>(r[u][k]));
    if constexpr (S::CL > 1 && !kPush) {  // keep smem alive for peers' remote loads
        cluster_arrive_relaxed();
        cluster_wait();
    }
}

}  // namespace lb
