// BFV-RNS layer: constants, key generation and the batched ciphertext
// operations. The reference evaluator's ring backend does the
// same slot-level actions on plaintext polynomials (proj/src/evaluator.cpp:
// lift_big :67-91, lower :98-118, add :137-152, add_plain :154-176, mul
// :178-202, mul_plain :204-226, mul_scalar :242-258, rotations :260-332);
// here every one of them runs on BFV ciphertexts.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "bfv.hpp"
#include "bfv_kernels.cuh"
#include "host_math.hpp"
#include "ks_fused.cuh"

namespace lb {

namespace {

constexpr int kBlock = 256;

inline unsigned grid_for(uint64_t work, int per_thread = 1) {
    uint64_t g = (work + static_cast<uint64_t>(kBlock) * per_thread - 1) / (static_cast<uint64_t>(kBlock) * per_thread);
    return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(g, 1u << 30)));
}

using host::invm;
using host::mulm;

uint64_t subm(uint64_t a, uint64_t b, uint64_t p) { return a >= b ? a - b : a + (p - b); }

// product of primes[lo..hi) except index `skip`, modulo `mod`
uint64_t prod_mod(const std::vector<uint64_t>& pr, size_t lo, size_t hi, size_t skip, uint64_t mod) {
    uint64_t r = 1 % mod;
    for (size_t k = lo; k < hi; ++k)
        if (k != skip) r = mulm(r, pr[k] % mod, mod);
    return r;
}

ulonglong2 frac128(uint64_t num, uint64_t d) {
    unsigned __int128 x = static_cast<unsigned __int128>(num) << 64;
    const uint64_t hi = static_cast<uint64_t>(x / d);
    const uint64_t r = static_cast<uint64_t>(x % d);
    x = static_cast<unsigned __int128>(r) << 64;
    return make_ulonglong2(hi, static_cast<uint64_t>(x / d));
}

// ---- device kernels ------------------------------------------------------------

// v < 2^64 with v >> 32 < 2^32 -> v mod r for r < 2^30: hi * [2^32]_r and lo
// by Shoup (each [0, 2r)), two conditional subtractions.
__device__ __forceinline__ uint32_t reduce64_32(uint64_t v, uint32_t r, uint4 red) {
    const uint32_t hi = static_cast<uint32_t>(v >> 32), lo = static_cast<uint32_t>(v);
    const uint32_t t = shoup_lazy<uint32_t>(hi, red.x, red.y, r) + shoup_lazy<uint32_t>(lo, 1u, red.z, r);
    return csub<uint32_t>(csub<uint32_t>(t, 2 * r), r);
}


// secret s (ternary, §3.2) reduced into every prime of Q, P, B
__global__ void k_secret_coeffs(BfvDev d, uint64_t* out, uint32_t primes) {
    const uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (idx >= uint64_t(primes) * d.n) return;
    const uint32_t r = idx / d.n, k = idx % d.n;
    const int64_t s = sample_ternary(prng_at(stream_key(d.seed, kStreamSecret), k));
    out[idx] = reduce_signed(s, modulus_of(d.primes[r]));
}

// out[c][r][pos] = in[c][r][src(pos)]: x -> x^g on bit-reversed evaluations
template <class St>
__global__ void k_automorph(const St* __restrict__ in, St* __restrict__ out, uint64_t total, uint32_t logn, uint64_t g) {
    const uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (idx >= total) return;
    const uint32_t n = 1u << logn;
    const uint32_t pos = idx & (n - 1);
    const uint32_t k = __brev(pos) >> (32 - logn);
    const uint64_t e = (g * (2ull * k + 1)) & (2ull * n - 1);
    const uint32_t k2 = static_cast<uint32_t>((e - 1) >> 1);
    const uint32_t src = __brev(k2) >> (32 - logn);
    out[idx] = in[(idx & ~uint64_t(n - 1)) | src];
}

// ---- key generation (§3.5) ----
__global__ void k_keygen_error(BfvDev d, uint64_t key_id, uint64_t* e_out /*[dnum][L+K][n]*/) {
    const uint32_t LK = d.L + d.K;
    const uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (idx >= uint64_t(d.dnum) * LK * d.n) return;
    const uint32_t k = idx % d.n;
    const uint32_t r = (idx / d.n) % LK;
    const uint32_t j = idx / (uint64_t(d.n) * LK);
    const int64_t e = sample_cbd21(prng_at(stream_key(d.seed, stream_ksk_e(key_id, j)), k));
    e_out[idx] = reduce_signed(e, modulus_of(d.primes[r]));
}

// key[j][0][r] = -a s + e + [r in digit j] [P]_r s' ; key[j][1][r] = a
__global__ void k_keygen_finish(BfvDev d, uint64_t key_id, const uint64_t* __restrict__ e_ntt,
                                const uint64_t* __restrict__ s_target /*[L+K][n]*/, const uint64_t* __restrict__ p_mod,
                                uint64_t* __restrict__ key) {
    const uint32_t LK = d.L + d.K;
    const uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (idx >= uint64_t(d.dnum) * LK * d.n) return;
    const uint32_t pos = idx % d.n;
    const uint32_t r = (idx / d.n) % LK;
    const uint32_t j = idx / (uint64_t(d.n) * LK);
    const Modulus m = modulus_of(d.primes[r]);
    const uint64_t a = sample_uniform(m.q, prng_at(stream_key(d.seed, stream_ksk_a(key_id, j, r)), pos));
    const uint64_t as = mul_mod(a, d.s_ntt[uint64_t(r) * d.n + pos], m);
    uint64_t b = sub_mod(e_ntt[idx], as, m.q);
    const uint32_t lo = j * d.alpha, hi = min(d.L, lo + d.alpha);
    if (r >= lo && r < hi) b = add_mod(b, mul_mod(p_mod[r], s_target[uint64_t(r) * d.n + pos], m), m.q);
    const uint64_t base = (uint64_t(j) * 2 * LK + r) * d.n + pos;
    key[base] = b;
    key[base + uint64_t(LK) * d.n] = a;
}

// (k, floor(k 2^64 / q)) for every key entry; rows of n entries share a prime
__global__ void k_shoup_pairs(BfvDev d, const uint64_t* __restrict__ key, ulonglong2* __restrict__ out, uint64_t total,
                              uint32_t limbs) {
    const uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (idx >= total) return;
    const Modulus m = modulus_of(d.primes[(idx / d.n) % limbs]);
    const uint64_t k = key[idx];
    // estimate from the 128-bit ratio (never too large), then correct
    uint64_t est = k * m.ratio_hi + mulhi64(k, m.ratio_lo);
    uint64_t lo = 0 - est * m.q;
    uint64_t hi = k - mulhi64(est, m.q) - (est * m.q != 0 ? 1 : 0);
    while (hi != 0 || lo >= m.q) {
        ++est;
        hi -= (lo < m.q) ? 1 : 0;
        lo -= m.q;
    }
    out[idx] = make_ulonglong2(k, est);
}

// (k, floor(k 2^32 / q)) for the 32-bit word key switch (every q < 2^30)
__global__ void k_shoup_pairs32(BfvDev d, const uint64_t* __restrict__ key, uint2* __restrict__ out, uint64_t total,
                                uint32_t limbs) {
    const uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (idx >= total) return;
    const uint64_t q = d.primes[(idx / d.n) % limbs].q;
    const uint64_t k = key[idx];
    out[idx] = make_uint2(static_cast<uint32_t>(k), static_cast<uint32_t>((k << 32) / q));
}

// (key_j[0], key_j[1]) word pairs [dnum][limbs][n] for the 29-bit key switch
// (64-bit product sums need no Shoup companions): half the key bytes
__global__ void k_pack_key29(const uint64_t* __restrict__ key, uint2* __restrict__ out, uint32_t dnum, uint32_t limbs,
                             uint32_t n) {
    const uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    const uint64_t per_j = uint64_t(limbs) * n;
    if (idx >= dnum * per_j) return;
    const uint64_t j = idx / per_j, rx = idx % per_j;
    out[idx] = make_uint2(static_cast<uint32_t>(key[(2 * j) * per_j + rx]), static_cast<uint32_t>(key[(2 * j + 1) * per_j + rx]));
}

__global__ void k_square_limbs(const uint64_t* __restrict__ s, uint64_t* __restrict__ out, BfvDev d, uint32_t limbs) {
    const uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (idx >= uint64_t(limbs) * d.n) return;
    const Modulus m = modulus_of(d.primes[idx / d.n]);
    out[idx] = mul_mod(s[idx], s[idx], m);
}

// ---- encoding / encryption (§3.3, §3.4) ----
// dst[(b*T + j)][slot_pos[i]] = values[b][i] mod t_j
__global__ void k_scatter_slots(BfvDev d, const int64_t* __restrict__ values, uint32_t B, uint64_t* __restrict__ dst) {
    const uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (idx >= uint64_t(B) * d.T * d.n) return;
    const uint32_t i = idx % d.n;
    const uint32_t j = (idx / d.n) % d.T;
    const uint64_t b = idx / (uint64_t(d.n) * d.T);
    const Modulus m = modulus_of(d.primes[d.tbase + j]);
    dst[(b * d.T + j) * d.n + d.slot_pos[i]] = reduce_signed(values[b * d.n + i], m);
}

// round(Q m / t) mod q_i = Delta m + floor(([Q]_t m + floor(t/2)) / t)
__device__ __forceinline__ uint64_t scaled_message(const BfvDev& d, uint32_t j, uint32_t i, uint64_t mval,
                                                   const Modulus& qm) {
    const uint64_t t = d.primes[d.tbase + j].q;
    const uint64_t extra = (d.q_mod_t[j] * mval + (t >> 1)) / t;
    return add_mod(mul_mod(d.delta[j * d.L + i], mval, qm), reduce_u64(extra, qm), qm.q);
}

// c0 (coefficient domain) = e + round(Q m / t); m: [count][n] mod t_j. One
// thread per coefficient: the error sample and the rounding term
// floor(([Q]_t m + t/2) / t) (a 64-bit division) are limb-independent, so
// they are computed once and the thread walks the L limbs.
template <class St>
__global__ void k_enc_coeffs(BfvDev d, const uint64_t* __restrict__ mcoef, uint32_t count, uint64_t id_base,
                             St* __restrict__ ct) {
    const uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (idx >= uint64_t(count) * d.n) return;
    const uint32_t k = idx % d.n;
    const uint64_t c = idx / d.n;
    const uint32_t j = c % d.T;
    const int64_t e = sample_cbd21(prng_at(stream_key(d.seed, stream_enc_e(id_base + c)), k));
    const uint64_t mval = mcoef[c * d.n + k];
    const uint64_t t = d.primes[d.tbase + j].q;
    const uint64_t extra = (d.q_mod_t[j] * mval + (t >> 1)) / t;
    St* out = ct + c * 2 * d.L * d.n + k;
    if constexpr (sizeof(St) == 4) {
        // every q_i < 2^30 and t < 2^32: Shoup products in 32-bit words
        for (uint32_t i = 0; i < d.L; ++i) {
            const uint32_t q = static_cast<uint32_t>(d.primes[i].q);
            const uint2 dl = d.delta32[j * d.L + i], one = d.one32[i];
            const uint32_t a = shoup_full<uint32_t>(static_cast<uint32_t>(mval), dl.x, dl.y, q);
            const uint32_t b = shoup_full<uint32_t>(static_cast<uint32_t>(extra), 1u, one.y, q);
            const uint32_t ee = e < 0 ? q - static_cast<uint32_t>(-e) : static_cast<uint32_t>(e);  // |e| <= 21
            out[uint64_t(i) * d.n] = csub<uint32_t>(csub<uint32_t>(a + b, q) + ee, q);
        }
        return;
    }
    for (uint32_t i = 0; i < d.L; ++i) {
        const Modulus qm = modulus_of(d.primes[i]);
        const uint64_t sm = add_mod(mul_mod(d.delta[j * d.L + i], mval, qm), reduce_u64(extra, qm), qm.q);
        out[uint64_t(i) * d.n] = static_cast<St>(add_mod(reduce_signed(e, qm), sm, qm.q));
    }
}

// c1 = a (sampled in the evaluation domain), c0 = NTT(e + round(Qm/t)) - a s
// (blocks never straddle a row: n is a multiple of the block size, so the
// row's PRNG stream key is derived once per block)
template <class St>
__global__ void k_enc_finish(BfvDev d, uint32_t count, uint64_t id_base, St* __restrict__ ct) {
    __shared__ uint64_t key_sh;
    const uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    const uint32_t pos = idx % d.n;
    const uint32_t i = (idx / d.n) % d.L;
    const uint64_t c = idx / (uint64_t(d.n) * d.L);
    if (threadIdx.x == 0) key_sh = stream_key(d.seed, stream_enc_a(id_base + c, i));
    __syncthreads();
    if (idx >= uint64_t(count) * d.L * d.n) return;
    const Modulus qm = modulus_of(d.primes[i]);
    const uint64_t a = sample_uniform(qm.q, prng_at(key_sh, pos));
    St* c0 = ct + (c * 2 * d.L + i) * d.n;
    St* c1 = c0 + uint64_t(d.L) * d.n;
    c1[pos] = static_cast<St>(a);
    if constexpr (sizeof(St) == 4) {
        const uint32_t q = static_cast<uint32_t>(qm.q);
        const uint2 sp = d.s32[uint64_t(i) * d.n + pos];
        const uint32_t as = shoup_full<uint32_t>(static_cast<uint32_t>(a), sp.x, sp.y, q);
        const uint32_t v = c0[pos];
        c0[pos] = v >= as ? v - as : v + q - as;
    } else {
        c0[pos] = static_cast<St>(sub_mod(c0[pos], mul_mod(a, d.s_ntt[uint64_t(i) * d.n + pos], qm), qm.q));
    }
}

// ---- fused encryption (u32 residues) ----
// Per coefficient of every ciphertext: the limb-independent pieces of c0's
// coefficients, extra = floor(([Q]_t m + t/2) / t) and the error sample e.
__global__ void k_enc_prep32(BfvDev d, const uint64_t* __restrict__ mcoef, uint32_t count, uint64_t id_base,
                             uint32_t* __restrict__ extra, int8_t* __restrict__ err) {
    const uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (idx >= uint64_t(count) * d.n) return;
    const uint32_t k = idx % d.n;
    const uint64_t c = idx / d.n;
    const uint32_t j = c % d.T;
    const uint64_t mval = mcoef[idx];
    const uint64_t t = d.primes[d.tbase + j].q;
    extra[idx] = static_cast<uint32_t>((d.q_mod_t[j] * mval + (t >> 1)) / t);
    err[idx] = static_cast<int8_t>(sample_cbd21(prng_at(stream_key(d.seed, stream_enc_e(id_base + c)), k)));
}

// One cluster per (ciphertext, limb i): c0's coefficients (e + round(Q m/t))
// mod q_i formed in the forward transform's first-pass loads, the transform,
// then c1 = a (sampled at each evaluation position) and c0 -= a s in the
// store: k_enc_coeffs + NTT + k_enc_finish in one pass over the limb.
template <int LOGN>
__global__ void __launch_bounds__(NttShape<LOGN>::T, ntt_min_blocks<uint32_t>())
    k_encrypt32(BfvDev d, const uint64_t* __restrict__ mcoef, const uint32_t* __restrict__ extra,
                const int8_t* __restrict__ err, uint64_t id_base, uint32_t* __restrict__ ct) {
    using S = NttShape<LOGN>;
    using W = uint32_t;
    __shared__ __align__(16) W sm[plane_words<LOGN, W>()];
    __shared__ uint64_t mbar;
    const uint32_t rank = S::CL > 1 ? cluster_rank() : 0;
    const uint32_t id = blockIdx.x / S::CL;
    const uint32_t c = id / d.L, i = id % d.L, j = c % d.T;
    const uint64_t n = 1ull << LOGN;
    const PrimeView<W> P = prime_view<W, LOGN>(d.tab32, d.primes, i);
    const W q = P.q;
    const uint2 dl = d.delta32[j * d.L + i], one = d.one32[i];
    const uint64_t* m = mcoef + uint64_t(c) * n;
    const uint32_t* ex = extra + uint64_t(c) * n;
    const int8_t* er = err + uint64_t(c) * n;
    const Xchg xc = xchg_init<S::CL>(&mbar, 1);
    const uint64_t key_a = stream_key(d.seed, stream_enc_a(id_base + c, i));
    W* c0 = ct + (uint64_t(c) * 2 * d.L + i) * n;
    W* c1 = c0 + uint64_t(d.L) * n;
    const uint2* s32 = d.s32 + uint64_t(i) * n;
    constexpr int C = 1 << fwd_last_radix<LOGN>();
    fwd_core<LOGN>(
        sm, P, rank,
        [&](uint32_t, uint32_t rho, uint32_t off) {
            const uint32_t k = rho + off;
            const W a = shoup_full<W>(static_cast<W>(__ldg(&m[k])), dl.x, dl.y, q);
            const W b = shoup_full<W>(__ldg(&ex[k]), 1u, one.y, q);
            const int e = __ldg(&er[k]);
            const W ee = e < 0 ? q - static_cast<W>(-e) : static_cast<W>(e);  // |e| <= 21
            return csub<W>(csub<W>(a + b, q) + ee, q);
        },
        true, xc,
        // the last pass's groups of consecutive evaluations, in registers
        [&](uint32_t, uint32_t base, W(&rr)[C]) {
            const uint32_t p0 = rank * S::M + base;
            W u0[C], u1[C];
#pragma unroll
            for (int k = 0; k < C; ++k) {
                const W v = reduce_4q<W>(rr[k], q, 2 * q);
                const W au = static_cast<W>(sample_uniform(q, prng_at(key_a, p0 + k)));
                const uint2 sp = __ldg(&s32[p0 + k]);
                const W as = shoup_full<W>(au, sp.x, sp.y, q);
                u1[k] = au;
                u0[k] = v >= as ? v - as : v + q - as;
            }
            if constexpr (C == 4) {
                *reinterpret_cast<uint4*>(c1 + p0) = make_uint4(u1[0], u1[1], u1[2], u1[3]);
                *reinterpret_cast<uint4*>(c0 + p0) = make_uint4(u0[0], u0[1], u0[2], u0[3]);
            } else {
#pragma unroll
                for (int k = 0; k < C; ++k) {
                    c1[p0 + k] = u1[k];
                    c0[p0 + k] = u0[k];
                }
            }
        });
}

// pt_mul = centered lift of m; pt_add = round(Q m / t); m: [T][n]
template <class St>
__global__ void k_pt_lift(BfvDev d, const uint64_t* __restrict__ mcoef, St* __restrict__ pt_mul, St* __restrict__ pt_add) {
    const uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (idx >= uint64_t(d.T) * d.L * d.n) return;
    const uint32_t k = idx % d.n;
    const uint32_t i = (idx / d.n) % d.L;
    const uint32_t j = idx / (uint64_t(d.n) * d.L);
    const Modulus qm = modulus_of(d.primes[i]);
    const uint64_t t = d.primes[d.tbase + j].q;
    const uint64_t mv = mcoef[uint64_t(j) * d.n + k];
    const int64_t centered = mv > (t >> 1) ? static_cast<int64_t>(mv) - static_cast<int64_t>(t) : static_cast<int64_t>(mv);
    if (pt_mul) pt_mul[idx] = static_cast<St>(reduce_signed(centered, qm));
    if (pt_add) pt_add[idx] = static_cast<St>(scaled_message(d, j, i, mv, qm));
}

// ---- decryption (§3.7) ----
template <class St>
__global__ void k_phase(BfvDev d, const St* __restrict__ ct, uint32_t count, uint64_t* __restrict__ x) {
    const uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (idx >= uint64_t(count) * d.L * d.n) return;
    const uint32_t pos = idx % d.n;
    const uint32_t i = (idx / d.n) % d.L;
    const uint64_t c = idx / (uint64_t(d.n) * d.L);
    const Modulus qm = modulus_of(d.primes[i]);
    const St* c0 = ct + (c * 2 * d.L + i) * d.n;
    const St* c1 = c0 + uint64_t(d.L) * d.n;
    if constexpr (sizeof(St) == 4) {
        const uint32_t q = static_cast<uint32_t>(qm.q);
        const uint2 sp = d.s32[uint64_t(i) * d.n + pos];
        x[idx] = csub<uint32_t>(c0[pos] + shoup_full<uint32_t>(c1[pos], sp.x, sp.y, q), q);
    } else {
        x[idx] = add_mod(c0[pos], mul_mod(c1[pos], d.s_ntt[uint64_t(i) * d.n + pos], qm), qm.q);
    }
}

// m = round(t x / Q) mod t from coefficient residues x: [count][L][n]
__global__ void k_dec_scale(BfvDev d, const uint64_t* __restrict__ x, uint32_t count, uint64_t* __restrict__ m) {
    const uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (idx >= uint64_t(count) * d.n) return;
    const uint32_t k = idx % d.n;
    const uint64_t c = idx / d.n;
    const uint32_t j = c % d.T;
    uint64_t H = 0, Lo = 0;
    for (uint32_t i = 0; i < d.L; ++i) {
        const Modulus qm = modulus_of(d.primes[i]);
        const uint64_t y = mul_mod(x[(c * d.L + i) * d.n + k], d.qhat_inv[i], qm);
        uint64_t ip, fp;
        fixmul(y, d.phi[j * d.L + i], ip, fp);
        Lo += fp;
        H += ip + (Lo < fp ? 1 : 0) + y * d.phi_int[j * d.L + i];
    }
    const Modulus tm = modulus_of(d.primes[d.tbase + j]);
    m[idx] = reduce_u64(H + (Lo >> 63), tm);
}

__global__ void k_gather_slots(BfvDev d, const uint64_t* __restrict__ ev, uint32_t count, uint64_t* __restrict__ out) {
    const uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (idx >= uint64_t(count) * d.n) return;
    const uint32_t i = idx % d.n;
    const uint64_t c = idx / d.n;
    out[idx] = ev[c * d.n + d.slot_pos[i]];
}

// ---- elementwise (ct ops) ----
// 2D grid: blockIdx.y walks the rows (poly-limb pairs, row = (c*2 + comp)*L
// + i, so the prime is fixed per block), blockIdx.x * blockDim.x * 2 + ... the
// coefficients, two per thread through 16-byte accesses. Rows beyond the
// grid's y extent are covered by the row loop.
constexpr int kEwThreads = 256;

struct EwShape {
    uint32_t rows;
    uint32_t L;
    uint32_t T;
    uint32_t logn;
};

template <class F>
__device__ __forceinline__ void ew_rows(const EwShape& sh, F&& f) {
    const uint32_t n = 1u << sh.logn;
    const uint32_t k = (blockIdx.x * kEwThreads + threadIdx.x) * 2;
    if (k >= n) return;
    for (uint32_t row = blockIdx.y; row < sh.rows; row += gridDim.y) {
        const uint32_t i = row % sh.L;
        const uint32_t comp = (row / sh.L) & 1;
        const uint32_t c = row / (2 * sh.L);
        f(uint64_t(row) << sh.logn | k, i, comp, c, k);
    }
}

// two consecutive residues, widened to u64 (16-byte access for u64 words,
// 8-byte for u32)
template <class St> __device__ __forceinline__ ulonglong2 ld2(const St* p) {
    if constexpr (sizeof(St) == 8) {
        return *reinterpret_cast<const ulonglong2*>(p);
    } else {
        const uint2 v = *reinterpret_cast<const uint2*>(p);
        return make_ulonglong2(v.x, v.y);
    }
}
template <class St> __device__ __forceinline__ ulonglong2 ldg2(const St* p) {
    if constexpr (sizeof(St) == 8) {
        return __ldg(reinterpret_cast<const ulonglong2*>(p));
    } else {
        const uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
        return make_ulonglong2(v.x, v.y);
    }
}
template <class St> __device__ __forceinline__ void st2(St* p, uint64_t a, uint64_t b) {
    if constexpr (sizeof(St) == 8)
        *reinterpret_cast<ulonglong2*>(p) = make_ulonglong2(a, b);
    else
        *reinterpret_cast<uint2*>(p) = make_uint2(static_cast<uint32_t>(a), static_cast<uint32_t>(b));
}

inline dim3 ew_grid(const EwShape& sh) {
    const uint32_t n = 1u << sh.logn;
    return dim3((n / 2 + kEwThreads - 1) / kEwThreads, std::min<uint32_t>(sh.rows, 65535u));
}

template <class St>
__global__ void __launch_bounds__(kEwThreads) k_add(BfvDev d, EwShape sh, const St* __restrict__ a,
                                                    const St* __restrict__ b, St* __restrict__ out) {
    ew_rows(sh, [&](uint64_t off, uint32_t i, uint32_t, uint32_t, uint32_t) {
        const uint64_t q = d.primes[i].q;
        const ulonglong2 x = ld2(a + off);
        const ulonglong2 y = ld2(b + off);
        st2(out + off, add_mod(x.x, y.x, q), add_mod(x.y, y.y, q));
    });
}

struct ScalarTab {
    ulonglong2 v[32];  // per ciphertext prime: (s mod q_i, Shoup companion)
};

template <class St>
__global__ void __launch_bounds__(kEwThreads) k_mul_scalar(BfvDev d, EwShape sh, const St* __restrict__ a, ScalarTab s,
                                                           St* __restrict__ out) {
    ew_rows(sh, [&](uint64_t off, uint32_t i, uint32_t, uint32_t, uint32_t) {
        const uint64_t q = d.primes[i].q;
        const ulonglong2 w = s.v[i];
        const ulonglong2 x = ld2(a + off);
        st2(out + off, mul_shoup(x.x, w.x, w.y, q), mul_shoup(x.y, w.x, w.y, q));
    });
}

template <class St>
__global__ void __launch_bounds__(kEwThreads) k_mul_scalar_add(BfvDev d, EwShape sh, const St* __restrict__ acc,
                                                               const St* __restrict__ x, ScalarTab s,
                                                               St* __restrict__ out) {
    ew_rows(sh, [&](uint64_t off, uint32_t i, uint32_t, uint32_t, uint32_t) {
        const uint64_t q = d.primes[i].q;
        const ulonglong2 w = s.v[i];
        const ulonglong2 u = ld2(acc + off);
        const ulonglong2 v = ld2(x + off);
        st2(out + off, add_mod(u.x, mul_shoup(v.x, w.x, w.y, q), q), add_mod(u.y, mul_shoup(v.y, w.x, w.y, q), q));
    });
}

// out[c][comp][i] = a[c][comp][i] * pt[c mod T][i]
template <class St>
__global__ void __launch_bounds__(kEwThreads) k_mul_plain(BfvDev d, EwShape sh, const St* __restrict__ a,
                                                          const St* __restrict__ pt, St* __restrict__ out) {
    ew_rows(sh, [&](uint64_t off, uint32_t i, uint32_t, uint32_t c, uint32_t k) {
        const ulonglong2 x = ld2(a + off);
        const ulonglong2 w = ldg2(pt + ((uint64_t(c % sh.T) * sh.L + i) << sh.logn) + k);
        if constexpr (sizeof(St) == 4) {
            if (d.qb32) {  // 30-bit residues: 64-bit product, 64 -> 32-bit Shoup reduction
                const uint32_t q = static_cast<uint32_t>(d.primes[i].q);
                const uint4 red = d.red32[i];
                const uint64_t p0 = static_cast<uint64_t>(static_cast<uint32_t>(x.x)) * static_cast<uint32_t>(w.x);
                const uint64_t p1 = static_cast<uint64_t>(static_cast<uint32_t>(x.y)) * static_cast<uint32_t>(w.y);
                st2(out + off, reduce64_32(p0, q, red), reduce64_32(p1, q, red));
                return;
            }
        }
        const Modulus qm = modulus_of(d.primes[i]);
        st2(out + off, mul_mod(x.x, w.x, qm), mul_mod(x.y, w.y, qm));
    });
}

template <class St>
__global__ void __launch_bounds__(kEwThreads) k_add_plain(BfvDev d, EwShape sh, const St* __restrict__ a,
                                                          const St* __restrict__ pt, St* __restrict__ out) {
    ew_rows(sh, [&](uint64_t off, uint32_t i, uint32_t comp, uint32_t c, uint32_t k) {
        const uint64_t q = d.primes[i].q;
        ulonglong2 x = ld2(a + off);
        if (!comp) {
            const ulonglong2 w = ldg2(pt + ((uint64_t(c % sh.T) * sh.L + i) << sh.logn) + k);
            x = make_ulonglong2(add_mod(x.x, w.x, q), add_mod(x.y, w.y, q));
        }
        st2(out + off, x.x, x.y);
    });
}

// ---- multiplication (§3.6) ----
// exact centered extension from `F` primes (table offset fbase) to `G`
// primes (table offset gbase); src: [polys][F][n] coeff, dst: [polys][G][n]
// SMALL: every F and G prime below 2^30, so y_i [F/f_i]_g < 2^60 and up to
// 16 of them sum exactly in 64 bits (one reduction per output instead of a
// 128-bit accumulator); y stays in registers (unrolled over the 16-prime cap).

// SMALL (every F and G prime below 2^30): Shoup products in 32-bit words
// (hat_inv32, prod32) and one 64 -> 32-bit reduction per output.
template <bool SMALL, class Src, class Dst>
__global__ void k_exact_extend(BfvDev d, const Src* __restrict__ src, uint32_t polys, uint32_t F, uint32_t fbase,
                               const uint64_t* __restrict__ hat_inv, const ulonglong2* __restrict__ frac,
                               const uint64_t* __restrict__ hat_mod /*[F][G]*/, const uint64_t* __restrict__ prod_mod /*[G]*/,
                               uint32_t G, uint32_t gbase, Dst* __restrict__ dst, const uint2* __restrict__ hat_inv32,
                               const uint2* __restrict__ prod32) {
    const uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (idx >= uint64_t(polys) * d.n) return;
    const uint32_t k = idx % d.n;
    const uint64_t p = idx / d.n;
    constexpr int kMax = 16;
    uint64_t y[kMax];
    uint64_t S_hi = 0, S_lo = 0;
#pragma unroll
    for (int i = 0; i < kMax; ++i) {
        if (i >= F) break;
        if constexpr (SMALL) {
            const uint32_t f = static_cast<uint32_t>(d.primes[fbase + i].q);
            const uint2 hi = hat_inv32[i];
            y[i] = shoup_full<uint32_t>(static_cast<uint32_t>(src[(p * F + i) * d.n + k]), hi.x, hi.y, f);
        } else {
            const Modulus fm = modulus_of(d.primes[fbase + i]);
            y[i] = mul_mod(src[(p * F + i) * d.n + k], hat_inv[i], fm);
        }
        uint64_t ip, fp;
        fixmul(y[i], frac[i], ip, fp);  // ip == 0: y_i / f_i < 1
        S_lo += fp;
        S_hi += ip + (S_lo < fp ? 1 : 0);
    }
    const uint64_t v = S_hi + (S_lo >> 63);  // round(sum y_i / f_i)
    for (uint32_t m = 0; m < G; ++m) {
        if constexpr (SMALL) {
            // y_i, [F/f_i]_g < 2^30: one IMAD.WIDE.U32 per term, the F <= 16
            // products sum below 2^64
            const uint32_t g = static_cast<uint32_t>(d.primes[gbase + m].q);
            uint64_t acc = 0;
#pragma unroll
            for (int i = 0; i < kMax; ++i) {
                if (i >= F) break;
                acc += static_cast<uint64_t>(static_cast<uint32_t>(y[i])) * static_cast<uint32_t>(hat_mod[i * G + m]);
            }
            const uint32_t s = reduce64_32(acc, g, d.red32[gbase + m]);
            const uint2 pm = prod32[m];
            const uint32_t vm = shoup_full<uint32_t>(static_cast<uint32_t>(v), pm.x, pm.y, g);  // v <= F < g
            dst[(p * G + m) * d.n + k] = static_cast<Dst>(s >= vm ? s - vm : s + g - vm);
            continue;
        }
        const Modulus gm = modulus_of(d.primes[gbase + m]);
        uint64_t s;
        {
            Acc128 acc;
#pragma unroll
            for (int i = 0; i < kMax; ++i) {
                if (i >= F) break;
                acc.mac(y[i], hat_mod[i * G + m]);
            }
            s = reduce_acc(acc, gm);
        }
        dst[(p * G + m) * d.n + k] = static_cast<Dst>(sub_mod(s, mul_mod(reduce_u64(v, gm), prod_mod[m], gm), gm.q));
    }
}

// tensor over Q ∪ B in the evaluation domain: d0 = a0 b0, d1 = a0 b1 + a1 b0, d2 = a1 b1
template <class St>
__global__ void k_tensor(BfvDev d, const St* __restrict__ A, const St* __restrict__ Bc,
                         const uint64_t* __restrict__ Y /*[count][4][M][n]*/, uint32_t count,
                         uint64_t* __restrict__ D /*[count][3][L+M][n]*/) {
    const uint32_t LM = d.L + d.M;
    const uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (idx >= uint64_t(count) * LM * d.n) return;
    const uint32_t pos = idx % d.n;
    const uint32_t r = (idx / d.n) % LM;
    const uint64_t c = idx / (uint64_t(d.n) * LM);
    uint64_t a0, a1, b0, b1;
    uint32_t pidx;
    if (r < d.L) {
        pidx = r;
        const uint64_t o = (c * 2 * d.L + r) * d.n + pos;
        a0 = A[o];
        a1 = A[o + uint64_t(d.L) * d.n];
        b0 = Bc[o];
        b1 = Bc[o + uint64_t(d.L) * d.n];
    } else {
        const uint32_t m = r - d.L;
        pidx = d.bbase + m;
        const uint64_t o = (c * 4 * d.M + m) * d.n + pos;
        const uint64_t st = uint64_t(d.M) * d.n;
        a0 = Y[o];
        a1 = Y[o + st];
        b0 = Y[o + 2 * st];
        b1 = Y[o + 3 * st];
    }
    const uint64_t st = uint64_t(LM) * d.n;
    const uint64_t o = (c * 3 * LM + r) * d.n + pos;
    if (d.qb32) {  // every value < 2^30: 64-bit products, 64 -> 32-bit Shoup reductions
        const uint32_t p = static_cast<uint32_t>(d.primes[pidx].q);
        const uint4 red = d.red32[pidx];
        auto mul = [](uint64_t x, uint64_t y) {
            return static_cast<uint64_t>(static_cast<uint32_t>(x)) * static_cast<uint32_t>(y);
        };
        D[o] = reduce64_32(mul(a0, b0), p, red);
        D[o + st] = reduce64_32(mul(a0, b1) + mul(a1, b0), p, red);
        D[o + 2 * st] = reduce64_32(mul(a1, b1), p, red);
        return;
    }
    const Modulus pm = modulus_of(d.primes[pidx]);
    D[o] = mul_mod(a0, b0, pm);
    Acc128 s;
    s.mac(a0, b1);
    s.mac(a1, b0);
    D[o + st] = reduce_acc(s, pm);
    D[o + 2 * st] = mul_mod(a1, b1, pm);
}

// Z = round(t D / Q) in base B; D: [polys][L+M][n] coeff, Z: [polys][M][n]
// SMALL (Q and B below 2^30, L + 1 <= 15): the Q-limb values stay in
// registers, one IMAD.WIDE.U32 per term, one 64 -> 32-bit reduction per
// output (the rounded R < L 2^30 fits the same 64-bit sum).
template <bool SMALL>
__global__ void k_scale(BfvDev d, const uint64_t* __restrict__ D, uint32_t polys, uint32_t polys_per_ct,
                        uint64_t* __restrict__ Z) {
    const uint32_t LM = d.L + d.M;
    const uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (idx >= uint64_t(polys) * d.n) return;
    const uint32_t k = idx % d.n;
    const uint64_t p = idx / d.n;
    const uint32_t j = (p / polys_per_ct) % d.T;
    const uint64_t* src = D + p * LM * d.n + k;
    uint64_t H = 0, Lo = 0;
    for (uint32_t i = 0; i < d.L; ++i) {
        uint64_t ip, fp;
        fixmul(src[uint64_t(i) * d.n], d.theta[j * d.L + i], ip, fp);
        Lo += fp;
        H += ip + (Lo < fp ? 1 : 0);
    }
    const uint64_t R = H + (Lo >> 63);
    if constexpr (SMALL) {
        constexpr int kMax = 14;
        uint32_t x[kMax];
#pragma unroll
        for (int i = 0; i < kMax; ++i) x[i] = i < static_cast<int>(d.L) ? static_cast<uint32_t>(src[uint64_t(i) * d.n]) : 0u;
        for (uint32_t m = 0; m < d.M; ++m) {
            const uint64_t* w = d.w_mod_b + uint64_t(j) * d.L * d.M + m;
            uint64_t acc = R + static_cast<uint64_t>(static_cast<uint32_t>(src[uint64_t(d.L + m) * d.n])) *
                                   static_cast<uint32_t>(d.tqinv_b[j * d.M + m]);
#pragma unroll
            for (int i = 0; i < kMax; ++i) {
                if (i >= static_cast<int>(d.L)) break;
                acc += static_cast<uint64_t>(x[i]) * static_cast<uint32_t>(w[uint64_t(i) * d.M]);
            }
            Z[(p * d.M + m) * d.n + k] =
                reduce64_32(acc, static_cast<uint32_t>(d.primes[d.bbase + m].q), d.red32[d.bbase + m]);
        }
        return;
    }
    for (uint32_t m = 0; m < d.M; ++m) {
        const Modulus bm = modulus_of(d.primes[d.bbase + m]);
        Acc128 acc;
        for (uint32_t i = 0; i < d.L; ++i) acc.mac(src[uint64_t(i) * d.n], d.w_mod_b[(j * d.L + i) * d.M + m]);
        acc.mac(src[uint64_t(d.L + m) * d.n], d.tqinv_b[j * d.M + m]);
        acc.add(R);
        Z[(p * d.M + m) * d.n + k] = reduce_acc(acc, bm);
    }
}

}  // namespace

// ---- constants -----------------------------------------------------------------

namespace {
bool ks_use_planes();
}

// 29-bit fast path of the key switch (A/B switch LB_KS29=0)
static bool ks29_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("LB_KS29");
        return !(e && e[0] == '0');
    }();
    return on;
}

void bfv_setup(Context& cx) {
    auto st = std::make_unique<BfvState>();
    const auto& P = cx.params();
    const uint32_t n = cx.n(), L = cx.L(), K = cx.K(), M = cx.M(), T = cx.T();
    const uint32_t dnum = cx.dnum(), alpha = cx.alpha();
    if (L > 16 || K > 8 || M > 16 || T > 16) throw std::invalid_argument("prime group too large");
    BfvDev& d = st->dev;
    d.n = n;
    d.logn = cx.logn();
    d.L = L;
    d.K = K;
    d.M = M;
    d.T = T;
    d.dnum = dnum;
    d.alpha = alpha;
    d.pbase = L;
    d.bbase = L + K;
    d.tbase = L + K + M;
    d.seed = P.seed;
    d.primes = cx.dev_primes();
    d.tab32 = cx.tab32();
    const auto& q = P.q;
    const auto& p = P.p;
    const auto& b = P.b;
    const auto& t = P.t;
    const uint32_t LK = L + K;

    // host staging of every table, then one upload
    std::vector<uint8_t> blob;
    auto put = [&](const void* src, size_t bytes) {
        size_t off = (blob.size() + 15) & ~size_t(15);
        blob.resize(off + bytes);
        std::memcpy(blob.data() + off, src, bytes);
        return off;
    };
    std::vector<uint32_t> slot_pos(n), pos_slot(n);
    {
        const uint64_t two_n = 2ull * n;
        uint64_t g = 1;
        for (uint32_t jj = 0; jj < n / 2; ++jj) {
            const uint32_t e0 = static_cast<uint32_t>((g - 1) / 2);
            const uint32_t e1 = static_cast<uint32_t>((two_n - g - 1) / 2);
            slot_pos[jj] = host::bitrev(e0, cx.logn());
            slot_pos[n / 2 + jj] = host::bitrev(e1, cx.logn());
            g = g * 3 % two_n;
        }
        for (uint32_t i = 0; i < n; ++i) pos_slot[slot_pos[i]] = i;
    }
    const size_t o_slot = put(slot_pos.data(), n * 4);
    const size_t o_pslot = put(pos_slot.data(), n * 4);

    std::vector<uint64_t> delta(T * L), qmt(T);
    for (uint32_t j = 0; j < T; ++j) {
        qmt[j] = prod_mod(q, 0, L, SIZE_MAX, t[j]);
        for (uint32_t i = 0; i < L; ++i) delta[j * L + i] = mulm(subm(0, qmt[j] % q[i], q[i]), invm(t[j] % q[i], q[i]), q[i]);
    }
    const size_t o_delta = put(delta.data(), delta.size() * 8);
    const size_t o_qmt = put(qmt.data(), qmt.size() * 8);

    std::vector<uint64_t> qhat_inv(L);
    std::vector<ulonglong2> phi(T * L), q_frac(L);
    std::vector<uint64_t> phi_int(std::max<size_t>(1, size_t(T) * L));
    for (uint32_t i = 0; i < L; ++i) {
        qhat_inv[i] = invm(prod_mod(q, 0, L, i, q[i]), q[i]);
        q_frac[i] = frac128(1, q[i]);
        for (uint32_t j = 0; j < T; ++j) {
            // t_j / q_i = phi_int + phi / 2^128 (t_j > q_i for 30-bit q_i)
            phi[j * L + i] = frac128(t[j] % q[i], q[i]);
            phi_int[j * L + i] = t[j] / q[i];
        }
    }
    const size_t o_qhinv = put(qhat_inv.data(), L * 8);
    const size_t o_phi = put(phi.data(), phi.size() * 16);
    const size_t o_phint = put(phi_int.data(), phi_int.size() * 8);
    const size_t o_qfrac = put(q_frac.data(), L * 16);

    std::vector<uint64_t> qhat_mod_b(L * std::max(M, 1u)), q_mod_b(std::max(M, 1u));
    std::vector<uint64_t> bhat_inv(std::max(M, 1u)), bhat_mod_q(std::max(M, 1u) * L), b_mod_q(L);
    std::vector<ulonglong2> b_frac(std::max(M, 1u));
    for (uint32_t m = 0; m < M; ++m) {
        q_mod_b[m] = prod_mod(q, 0, L, SIZE_MAX, b[m]);
        for (uint32_t i = 0; i < L; ++i) qhat_mod_b[i * M + m] = prod_mod(q, 0, L, i, b[m]);
        bhat_inv[m] = invm(prod_mod(b, 0, M, m, b[m]), b[m]);
        b_frac[m] = frac128(1, b[m]);
        for (uint32_t i = 0; i < L; ++i) bhat_mod_q[m * L + i] = prod_mod(b, 0, M, m, q[i]);
    }
    for (uint32_t i = 0; i < L; ++i) b_mod_q[i] = prod_mod(b, 0, M, SIZE_MAX, q[i]);
    const size_t o_qhmb = put(qhat_mod_b.data(), qhat_mod_b.size() * 8);
    const size_t o_qmb = put(q_mod_b.data(), q_mod_b.size() * 8);
    const size_t o_bhinv = put(bhat_inv.data(), bhat_inv.size() * 8);
    const size_t o_bfrac = put(b_frac.data(), b_frac.size() * 16);
    const size_t o_bhmq = put(bhat_mod_q.data(), bhat_mod_q.size() * 8);
    const size_t o_bmq = put(b_mod_q.data(), b_mod_q.size() * 8);
    d.qb32 = Context::word32_enabled() && cx.primes_small(0, L) && cx.primes_small(L + K, M);
    size_t o_qhi32 = 0, o_bhi32 = 0, o_qmb32 = 0, o_bmq32 = 0, o_red32 = 0;
    if (d.qb32) {
        auto pairs = [](const std::vector<uint64_t>& v, const std::vector<uint64_t>& mods, size_t count) {
            std::vector<uint2> o(std::max<size_t>(1, count));
            for (size_t k = 0; k < count; ++k)
                o[k] = make_uint2(static_cast<uint32_t>(v[k]), shoup_companion32(v[k], mods[k]));
            return o;
        };
        const auto qhi32 = pairs(qhat_inv, q, L), bhi32 = pairs(bhat_inv, b, M);
        const auto qmb32 = pairs(q_mod_b, b, M), bmq32 = pairs(b_mod_q, q, L);
        o_qhi32 = put(qhi32.data(), qhi32.size() * 8);
        o_bhi32 = put(bhi32.data(), bhi32.size() * 8);
        o_qmb32 = put(qmb32.data(), qmb32.size() * 8);
        o_bmq32 = put(bmq32.data(), bmq32.size() * 8);
        std::vector<uint4> red(size_t(L) + K + M);
        for (uint32_t r = 0; r < L + K + M; ++r) {
            const uint64_t pr = cx.prime(r);
            if (pr >= (uint64_t{1} << 30)) continue;
            const uint64_t w = (uint64_t{1} << 32) % pr;
            red[r] = make_uint4(static_cast<uint32_t>(w), shoup_companion32(w, pr), shoup_companion32(1, pr), 0u);
        }
        o_red32 = put(red.data(), red.size() * 16);
    }

    std::vector<ulonglong2> theta(T * L);
    std::vector<uint64_t> w_mod_b(std::max<size_t>(1, size_t(T) * L * M)), tqinv_b(std::max<size_t>(1, size_t(T) * M));
    for (uint32_t j = 0; j < T && M; ++j) {
        for (uint32_t i = 0; i < L; ++i) {
            const uint64_t Bm = prod_mod(b, 0, M, SIZE_MAX, q[i]);
            const uint64_t ci = invm(mulm(prod_mod(q, 0, L, i, q[i]), Bm, q[i]), q[i]);
            const uint64_t rem = mulm(mulm(t[j] % q[i], ci, q[i]), Bm, q[i]);
            theta[j * L + i] = frac128(rem, q[i]);
            for (uint32_t m = 0; m < M; ++m)
                w_mod_b[(size_t(j) * L + i) * M + m] = mulm(subm(0, rem % b[m], b[m]), invm(q[i] % b[m], b[m]), b[m]);
        }
        for (uint32_t m = 0; m < M; ++m)
            tqinv_b[j * M + m] = mulm(t[j] % b[m], invm(prod_mod(q, 0, L, SIZE_MAX, b[m]), b[m]), b[m]);
    }
    const size_t o_theta = put(theta.data(), theta.size() * 16);
    const size_t o_wmb = put(w_mod_b.data(), w_mod_b.size() * 8);
    const size_t o_tqb = put(tqinv_b.data(), tqinv_b.size() * 8);

    std::vector<uint64_t> qp(q);
    qp.insert(qp.end(), p.begin(), p.end());
    std::vector<uint64_t> dhat_inv(L), dhat_mod(size_t(L) * LK);
    for (uint32_t i = 0; i < L; ++i) {
        const uint32_t j = i / alpha, lo = j * alpha, hi = std::min(L, lo + alpha);
        dhat_inv[i] = invm(prod_mod(q, lo, hi, i, q[i]), q[i]);
        for (uint32_t r = 0; r < LK; ++r) dhat_mod[size_t(i) * LK + r] = prod_mod(q, lo, hi, i, qp[r]);
    }
    std::vector<uint64_t> phat_inv(std::max(K, 1u)), phat_mod_q(std::max(K, 1u) * L), p_inv_q(L);
    for (uint32_t l = 0; l < K; ++l) {
        phat_inv[l] = invm(prod_mod(p, 0, K, l, p[l]), p[l]);
        for (uint32_t i = 0; i < L; ++i) phat_mod_q[l * L + i] = prod_mod(p, 0, K, l, q[i]);
    }
    for (uint32_t i = 0; i < L; ++i) p_inv_q[i] = K ? invm(prod_mod(p, 0, K, SIZE_MAX, q[i]), q[i]) : 1;
    const size_t o_dhinv = put(dhat_inv.data(), L * 8);
    const size_t o_dhmod = put(dhat_mod.data(), dhat_mod.size() * 8);
    const size_t o_phinv = put(phat_inv.data(), phat_inv.size() * 8);
    const size_t o_phmq = put(phat_mod_q.data(), phat_mod_q.size() * 8);
    const size_t o_piq = put(p_inv_q.data(), L * 8);
    std::vector<ulonglong2> p_inv_shoup(L);
    for (uint32_t i = 0; i < L; ++i) p_inv_shoup[i] = make_ulonglong2(p_inv_q[i], shoup_companion(p_inv_q[i], q[i]));
    const size_t o_pish = put(p_inv_shoup.data(), L * 16);
    {
        // the fused key switch feeds single-prime digits and [acc]_P into the
        // lazy transform unreduced: every prime of Q and P must be < 4x any other
        uint64_t lo = ~uint64_t{0}, hi = 0;
        for (uint32_t r = 0; r < LK; ++r) {
            lo = std::min(lo, qp[r]);
            hi = std::max(hi, qp[r]);
        }
        if (hi / 4 >= lo) throw std::invalid_argument("ciphertext and special primes must be within a factor 4");
    }
    std::vector<uint64_t> p_mod_qp(LK);
    for (uint32_t r = 0; r < LK; ++r) p_mod_qp[r] = prod_mod(p, 0, K, SIZE_MAX, qp[r]);
    const size_t o_pmqp = put(p_mod_qp.data(), LK * 8);
    auto pair = [](uint64_t v, uint64_t m) { return make_ulonglong2(v, shoup_companion(v, m)); };
    std::vector<ulonglong2> dhat_mod_sh(size_t(L) * LK), phat_mod_sh(std::max(K, 1u) * size_t(L));
    std::vector<ulonglong2> ks_last_q(2 * size_t(L)), ks_last_p(2 * size_t(std::max(K, 1u)));
    for (uint32_t i = 0; i < L; ++i) {
        for (uint32_t r = 0; r < LK; ++r) dhat_mod_sh[size_t(i) * LK + r] = pair(dhat_mod[size_t(i) * LK + r], qp[r]);
        const PrimeDev& hp = cx.host_prime(i);
        ks_last_q[2 * i] = pair(mulm(hp.ninv, dhat_inv[i], q[i]), q[i]);
        ks_last_q[2 * i + 1] = pair(mulm(hp.inv1n, dhat_inv[i], q[i]), q[i]);
    }
    for (uint32_t l = 0; l < K; ++l) {
        for (uint32_t r = 0; r < L; ++r) phat_mod_sh[size_t(l) * L + r] = pair(phat_mod_q[size_t(l) * L + r], q[r]);
        const PrimeDev& hp = cx.host_prime(L + l);
        ks_last_p[2 * l] = pair(mulm(hp.ninv, phat_inv[l], p[l]), p[l]);
        ks_last_p[2 * l + 1] = pair(mulm(hp.inv1n, phat_inv[l], p[l]), p[l]);
    }
    // 32-bit word key switch when Q and P are all below 2^30
    d.ks32 = Context::word32_enabled() && cx.primes_small(0, LK);
    auto to32 = [&](const std::vector<ulonglong2>& v, auto&& modulus_of_index) {
        std::vector<uint2> o(v.size());
        for (size_t k = 0; k < v.size(); ++k) {
            const uint64_t m = modulus_of_index(k);
            o[k] = make_uint2(static_cast<uint32_t>(v[k].x), m ? shoup_companion32(v[k].x, m) : 0u);
        }
        return o;
    };
    size_t o_pi32 = 0, o_dh32 = 0, o_ph32 = 0, o_klq32 = 0, o_klp32 = 0, o_de32 = 0, o_one32 = 0, o_mu60 = 0;
    d.ks29 = d.ks32 && alpha <= 8 && K <= 8 && dnum <= kMaxPlanes && ks29_enabled() && ks_use_planes();
    for (uint32_t r = 0; r < LK && d.ks29; ++r)
        d.ks29 = qp[r] > (uint64_t{1} << 28) && qp[r] < (uint64_t{1} << 29);
    if (d.ks29) {
        std::vector<uint32_t> mu(LK);
        for (uint32_t r = 0; r < LK; ++r) mu[r] = static_cast<uint32_t>((uint64_t{1} << 60) / qp[r]);
        o_mu60 = put(mu.data(), mu.size() * 4);
    }
    if (d.ks32) {
        std::vector<uint2> de32(size_t(T) * L), one32(L);
        for (uint32_t j = 0; j < T; ++j)
            for (uint32_t i = 0; i < L; ++i)
                de32[j * L + i] = make_uint2(static_cast<uint32_t>(delta[j * L + i]),
                                             shoup_companion32(delta[j * L + i], q[i]));
        for (uint32_t i = 0; i < L; ++i) one32[i] = make_uint2(1u, shoup_companion32(1, q[i]));
        o_de32 = put(de32.data(), std::max<size_t>(1, de32.size()) * 8);
        o_one32 = put(one32.data(), one32.size() * 8);
        const auto pi32 = to32(p_inv_shoup, [&](size_t k) { return q[k]; });
        const auto dh32 = to32(dhat_mod_sh, [&](size_t k) { return qp[k % LK]; });
        const auto ph32 = to32(phat_mod_sh, [&](size_t k) { return K ? q[k % L] : 0; });
        const auto klq32 = to32(ks_last_q, [&](size_t k) { return q[k / 2]; });
        const auto klp32 = to32(ks_last_p, [&](size_t k) { return K ? p[k / 2] : 0; });
        o_pi32 = put(pi32.data(), pi32.size() * 8);
        o_dh32 = put(dh32.data(), dh32.size() * 8);
        o_ph32 = put(ph32.data(), ph32.size() * 8);
        o_klq32 = put(klq32.data(), klq32.size() * 8);
        o_klp32 = put(klp32.data(), klp32.size() * 8);
    }
    const size_t o_dhsh = put(dhat_mod_sh.data(), dhat_mod_sh.size() * 16);
    const size_t o_phsh = put(phat_mod_sh.data(), phat_mod_sh.size() * 16);
    const size_t o_klq = put(ks_last_q.data(), ks_last_q.size() * 16);
    const size_t o_klp = put(ks_last_p.data(), ks_last_p.size() * 16);

    std::vector<int16_t> t_map(std::max(T, 1u)), qb_map(L + M), ks_map(size_t(dnum) * LK);
    for (uint32_t j = 0; j < T; ++j) t_map[j] = int16_t(L + K + M + j);
    for (uint32_t r = 0; r < L + M; ++r) qb_map[r] = int16_t(r < L ? r : L + K + (r - L));
    for (uint32_t j = 0; j < dnum; ++j) {
        const uint32_t lo = j * alpha, hi = std::min(L, lo + alpha);
        for (uint32_t r = 0; r < LK; ++r) ks_map[j * LK + r] = (r >= lo && r < hi) ? int16_t(-1) : int16_t(r);
    }
    const size_t o_tmap = put(t_map.data(), t_map.size() * 2);
    const size_t o_qbmap = put(qb_map.data(), qb_map.size() * 2);
    const size_t o_ksmap = put(ks_map.data(), ks_map.size() * 2);

    cudaStream_t s = cx.stream();
    st->consts = DeviceBuffer(blob.size(), s);
    uint8_t* base = st->consts.get<uint8_t>();
    LB_CUDA(cudaMemcpyAsync(base, blob.data(), blob.size(), cudaMemcpyHostToDevice, s));
    d.slot_pos = reinterpret_cast<const uint32_t*>(base + o_slot);
    d.pos_slot = reinterpret_cast<const uint32_t*>(base + o_pslot);
    d.delta = reinterpret_cast<const uint64_t*>(base + o_delta);
    d.q_mod_t = reinterpret_cast<const uint64_t*>(base + o_qmt);
    d.qhat_inv = reinterpret_cast<const uint64_t*>(base + o_qhinv);
    d.phi = reinterpret_cast<const ulonglong2*>(base + o_phi);
    d.phi_int = reinterpret_cast<const uint64_t*>(base + o_phint);
    d.q_frac = reinterpret_cast<const ulonglong2*>(base + o_qfrac);
    d.qhat_mod_b = reinterpret_cast<const uint64_t*>(base + o_qhmb);
    d.q_mod_b = reinterpret_cast<const uint64_t*>(base + o_qmb);
    d.bhat_inv = reinterpret_cast<const uint64_t*>(base + o_bhinv);
    d.b_frac = reinterpret_cast<const ulonglong2*>(base + o_bfrac);
    d.bhat_mod_q = reinterpret_cast<const uint64_t*>(base + o_bhmq);
    d.b_mod_q = reinterpret_cast<const uint64_t*>(base + o_bmq);
    if (d.qb32) {
        d.qhat_inv32 = reinterpret_cast<const uint2*>(base + o_qhi32);
        d.bhat_inv32 = reinterpret_cast<const uint2*>(base + o_bhi32);
        d.q_mod_b32 = reinterpret_cast<const uint2*>(base + o_qmb32);
        d.b_mod_q32 = reinterpret_cast<const uint2*>(base + o_bmq32);
        d.red32 = reinterpret_cast<const uint4*>(base + o_red32);
    }
    d.theta = reinterpret_cast<const ulonglong2*>(base + o_theta);
    d.w_mod_b = reinterpret_cast<const uint64_t*>(base + o_wmb);
    d.tqinv_b = reinterpret_cast<const uint64_t*>(base + o_tqb);
    d.dhat_inv = reinterpret_cast<const uint64_t*>(base + o_dhinv);
    d.dhat_mod = reinterpret_cast<const uint64_t*>(base + o_dhmod);
    d.phat_inv = reinterpret_cast<const uint64_t*>(base + o_phinv);
    d.phat_mod_q = reinterpret_cast<const uint64_t*>(base + o_phmq);
    d.p_inv_q = reinterpret_cast<const uint64_t*>(base + o_piq);
    d.p_mod_qp = reinterpret_cast<const uint64_t*>(base + o_pmqp);
    d.p_inv_shoup = reinterpret_cast<const ulonglong2*>(base + o_pish);
    d.dhat_mod_sh = reinterpret_cast<const ulonglong2*>(base + o_dhsh);
    d.phat_mod_sh = reinterpret_cast<const ulonglong2*>(base + o_phsh);
    d.ks_last_q = reinterpret_cast<const ulonglong2*>(base + o_klq);
    d.ks_last_p = reinterpret_cast<const ulonglong2*>(base + o_klp);
    if (d.ks32) {
        d.p_inv32 = reinterpret_cast<const uint2*>(base + o_pi32);
        d.dhat_mod_sh32 = reinterpret_cast<const uint2*>(base + o_dh32);
        d.phat_mod_sh32 = reinterpret_cast<const uint2*>(base + o_ph32);
        d.ks_last_q32 = reinterpret_cast<const uint2*>(base + o_klq32);
        d.ks_last_p32 = reinterpret_cast<const uint2*>(base + o_klp32);
        d.delta32 = reinterpret_cast<const uint2*>(base + o_de32);
        d.one32 = reinterpret_cast<const uint2*>(base + o_one32);
    }
    d.mu60 = d.ks29 ? reinterpret_cast<const uint32_t*>(base + o_mu60) : nullptr;
    {
        // HPS scaling computes round(t D / Q) in base B, |D| < n Q^2 / 4
        double lq = 0, lb = 0, lt = 0;
        for (uint32_t i = 0; i < L; ++i) lq += std::log2(double(q[i]));
        for (uint32_t m = 0; m < M; ++m) lb += std::log2(double(b[m]));
        for (uint32_t j = 0; j < T; ++j) lt = std::max(lt, std::log2(double(t[j])));
        st->mul_base_ok = M >= L + 1 && lb >= lq + lt + std::log2(double(n)) + 2;
    }
    st->qb_small = Context::word32_enabled() && cx.primes_small(0, L) && cx.primes_small(L + K, M);
    st->t_map = reinterpret_cast<const int16_t*>(base + o_tmap);
    st->qb_map = reinterpret_cast<const int16_t*>(base + o_qbmap);
    st->ks_map = reinterpret_cast<const int16_t*>(base + o_ksmap);

    // secret key in the evaluation domain over Q, P, B
    const uint32_t nsec = L + K + M;
    st->secret = DeviceBuffer(size_t(nsec) * n * 8, s);
    k_secret_coeffs<<<grid_for(uint64_t(nsec) * n), kBlock, 0, s>>>(d, st->secret.get(), nsec);
    LB_KERNEL_DONE();
    d.s_ntt = st->secret.get();
    cx.bfv_ = std::move(st);
    cx.ntt_forward(LimbBatch{cx.bfv_->secret.get(), 1, nsec, 0, uint64_t(nsec) * n}, s);
    if (d.ks32) {
        BfvState& bs = *cx.bfv_;
        bs.secret32 = DeviceBuffer(uint64_t(L) * n * 8, s);
        k_shoup_pairs32<<<grid_for(uint64_t(L) * n), kBlock, 0, s>>>(d, d.s_ntt, bs.secret32.get<uint2>(),
                                                                      uint64_t(L) * n, L);
        LB_KERNEL_DONE();
        d.s32 = bs.secret32.get<uint2>();
    }
    LB_CUDA(cudaStreamSynchronize(s));
}

// ---- key material ----------------------------------------------------------------

template <class St>
static void automorphism_words(Context& cx, const St* in, St* out, uint32_t polys, uint32_t limbs, uint64_t galois,
                               cudaStream_t s) {
    if (galois % 2 == 0 || galois >= 2ull * cx.n()) throw std::invalid_argument("galois element must be odd in [1, 2n)");
    const uint64_t total = uint64_t(polys) * limbs * cx.n();
    if (!total) return;
    k_automorph<St><<<grid_for(total), kBlock, 0, s>>>(in, out, total, cx.logn(), galois);
    LB_KERNEL_DONE();
}

void automorphism_ntt(Context& cx, const void* in, void* out, uint32_t polys, uint32_t limbs, uint64_t galois,
                      cudaStream_t s) {
    if (cx.bfv()->dev.ks32)
        automorphism_words(cx, static_cast<const uint32_t*>(in), static_cast<uint32_t*>(out), polys, limbs, galois, s);
    else
        automorphism_words(cx, static_cast<const uint64_t*>(in), static_cast<uint64_t*>(out), polys, limbs, galois, s);
}

void ensure_key(Context& cx, uint64_t key_id, cudaStream_t s) {
    BfvState& st = *cx.bfv();
    std::lock_guard<std::mutex> lock(st.mu);
    if (st.keys.count(key_id)) return;
    if (key_id != kRelinKeyId && (key_id % 2 == 0 || key_id >= 2ull * cx.n()))
        throw std::invalid_argument("galois element must be odd in [3, 2n)");
    const BfvDev& d = st.dev;
    const uint32_t n = cx.n(), LK = d.L + d.K;
    const uint64_t key_elems = uint64_t(d.dnum) * 2 * LK * n;
    KsKey key;
    key.buf = DeviceBuffer(key_elems * 8, s);
    DeviceBuffer target(uint64_t(LK) * n * 8, s), err(uint64_t(d.dnum) * LK * n * 8, s);
    if (key_id == kRelinKeyId) {
        k_square_limbs<<<grid_for(uint64_t(LK) * n), kBlock, 0, s>>>(d.s_ntt, target.get(), d, LK);
    } else {
        automorphism_words(cx, d.s_ntt, target.get(), 1, LK, key_id, s);  // key material stays u64
    }
    LB_KERNEL_DONE();
    k_keygen_error<<<grid_for(uint64_t(d.dnum) * LK * n), kBlock, 0, s>>>(d, key_id, err.get());
    LB_KERNEL_DONE();
    cx.ntt_forward(LimbBatch{err.get(), d.dnum, LK, 0, uint64_t(LK) * n}, s);
    k_keygen_finish<<<grid_for(uint64_t(d.dnum) * LK * n), kBlock, 0, s>>>(d, key_id, err.get(), target.get(),
                                                                             d.p_mod_qp, key.buf.get());
    LB_KERNEL_DONE();
    if (d.ks29 && LB_WIDE_MAC) {
        key.shoup = DeviceBuffer(key_elems * 4, s);
        k_pack_key29<<<grid_for(key_elems / 2), kBlock, 0, s>>>(key.buf.get(), key.shoup.get<uint2>(), d.dnum, LK, n);
    } else if (d.ks32) {
        key.shoup = DeviceBuffer(key_elems * 8, s);
        k_shoup_pairs32<<<grid_for(key_elems), kBlock, 0, s>>>(d, key.buf.get(), key.shoup.get<uint2>(), key_elems, LK);
    } else {
        key.shoup = DeviceBuffer(key_elems * 16, s);
        k_shoup_pairs<<<grid_for(key_elems), kBlock, 0, s>>>(d, key.buf.get(), key.shoup.get<ulonglong2>(), key_elems,
                                                             LK);
    }
    LB_KERNEL_DONE();
    // keys are shared by every stream and outlive the (possibly side) stream
    // they were generated on: complete them now, free them on the context's
    // own stream later
    LB_CUDA(cudaStreamSynchronize(s));
    key.buf.rebind(cx.stream());
    key.shoup.rebind(cx.stream());
    st.keys.emplace(key_id, std::move(key));
}

static const void* key_shoup_ptr(Context& cx, uint64_t key_id) {
    BfvState& st = *cx.bfv();
    std::lock_guard<std::mutex> lock(st.mu);
    auto it = st.keys.find(key_id);
    if (it == st.keys.end()) throw std::invalid_argument("key not generated");
    return it->second.shoup.get();
}

const uint64_t* key_ptr(Context& cx, uint64_t key_id) {
    BfvState& st = *cx.bfv();
    std::lock_guard<std::mutex> lock(st.mu);
    auto it = st.keys.find(key_id);
    if (it == st.keys.end()) throw std::invalid_argument("key not generated");
    return it->second.buf.get();
}

// ---- key switching -------------------------------------------------------------

namespace {

bool ks_use_tmem() {
    static const bool on = [] {
        // A/B on B200 (cfg0, B=64): smem accumulators 74.7 img/s, TMEM
        // accumulators 72.3 img/s (80-register cap spills); smem is default
        const char* e = std::getenv("LB_KS_TMEM");
        return e ? e[0] != '0' : false;
    }();
    return on;
}

// paired key-switch kernels (29-bit fast path): bit 0 ModDown (both
// components per cluster), bit 1 the inner product (two ciphertexts per
// cluster), bit 2 ModDown with two target primes per cluster on top of
// bit 0 (shared P-limb loads; off: measured slower, 1.61 vs 1.54 ms per
// 320-ciphertext key switch — the stash and the second start barrier cost
// more than the halved L2 reads save), bit 3 the mixed inner-product kernel
// (pairs for the targets in Q, single ciphertexts for the targets in P: two
// planes, 4 CTAs per SM; 1.42 vs 1.54 ms per 320-ciphertext key switch against
// bit 1's kernel, which stays as the fallback for dnum = 1); LB_KS_PAIR overrides
int ks_pairs() {
    static const int mask = [] {
        const char* e = std::getenv("LB_KS_PAIR");
        return e ? std::atoi(e) : 11;
    }();
    return mask;
}

// smallest launch (ciphertexts) that runs the mixed / paired inner product:
// with two planes and 4 CTAs per SM it wins from 8 ciphertexts on (two images:
// 11.9 vs 13.1 ms of HE steps; 80 ciphertexts 0.392 vs 0.430 ms per key
// switch); a single image (5 ciphertexts, odd) stays on the single-ciphertext
// kernel. LB_KS_PAIR_MIN overrides
uint32_t ks_pair_min() {
    static const uint32_t v = [] {
        const char* e = std::getenv("LB_KS_PAIR_MIN");
        return e ? static_cast<uint32_t>(std::max(2, std::atoi(e))) : 8u;
    }();
    return v;
}

// the same for the paired ModDown (from 32: at 40 ciphertexts per launch the
// plan is 3% faster with it, lola-cifar's 12 are 0.6% slower); LB_MD_PAIR_MIN
uint32_t md_pair_min() {
    static const uint32_t v = [] {
        const char* e = std::getenv("LB_MD_PAIR_MIN");
        return e ? static_cast<uint32_t>(std::max(2, std::atoi(e))) : 32u;
    }();
    return v;
}

bool ks_use_planes() {
    static const bool on = [] {
        const char* e = std::getenv("LB_KS_PLANES");
        return e ? e[0] != '0' : true;
    }();
    return on;
}

template <int LOGN, class W>
void launch_ks_inner(const BfvDev& d, const KsInnerArgs& a, cudaStream_t s) {
    using S = NttShape<LOGN>;
    if (sizeof(W) == 8 && ks_use_tmem()) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(static_cast<unsigned>(uint64_t(a.count) * (d.L + d.K) * S::CL));
        cfg.blockDim = dim3(S::T);
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = S::CL;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        LB_CUDA(cudaLaunchKernelEx(&cfg, ks_inner_tmem_kernel<LOGN>, d, a));
        launch_counter().fetch_add(1, std::memory_order_relaxed);
        return;
    }
    if constexpr (sizeof(W) == 4) {
        if (d.ks29 && LB_WIDE_MAC && (ks_pairs() & 8) && a.count >= ks_pair_min() && d.dnum == 2 &&
            d.L == 2 * d.alpha && S::CL > 1) {
            // mixed kernel: pairs for the targets in Q, single ciphertexts for the
            // targets in P, two planes and 4 CTAs per SM everywhere
            KsInnerArgs ap = a;
            ap.count = a.count & ~1u;
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = grid_xyz((d.L + 2 * d.K) * S::CL, ap.count / 2);
            cfg.blockDim = dim3(S::T);
            cfg.stream = s;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = S::CL;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            LB_CUDA(cudaLaunchKernelEx(&cfg, ks_inner_mix_kernel<LOGN>, d, ap));
            launch_counter().fetch_add(1, std::memory_order_relaxed);
            if (!(a.count & 1u)) return;
            KsInnerArgs al = a;
            const uint32_t c = a.count - 1;
            const size_t wb = sizeof(W);
            al.dc = static_cast<const uint8_t*>(a.dc) + uint64_t(c) * d.L * d.n * wb;
            al.dn = static_cast<const uint8_t*>(a.dn) + uint64_t(c) * a.d_stride * wb;
            al.acc = static_cast<uint8_t*>(a.acc) + uint64_t(c) * 2 * (d.L + d.K) * d.n * wb;
            al.count = 1;
            launch_ks_inner<LOGN, W>(d, al, s);
            return;
        }
        if (d.ks29 && LB_WIDE_MAC && (ks_pairs() & 2) && a.count >= ks_pair_min() && d.dnum <= 2 &&
            d.L % d.alpha == 0 && S::CL > 1) {
            // two ciphertexts per cluster; targets in Q have dnum - 1 foreign
            // digits, targets in P dnum: separate launches sized for each
            static bool configured_pair = false;
            if (!configured_pair) {
                LB_CUDA(cudaFuncSetAttribute(ks_inner_pair_kernel<LOGN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(2 * 2 * plane_words<LOGN, W>() * sizeof(W))));
                configured_pair = true;
            }
            KsInnerArgs ap = a;
            ap.count = a.count & ~1u;
            {
                // one launch over every target of Q ∪ P (planes sized for the
                // targets in P: dnum foreign digits x 2 ciphertexts)
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = grid_xyz((d.L + d.K) * S::CL, ap.count / 2);
                cfg.blockDim = dim3(S::T);
                cfg.dynamicSmemBytes = size_t(d.dnum) * 2 * plane_words<LOGN, W>() * sizeof(W);
                cfg.stream = s;
                cudaLaunchAttribute attr[1];
                attr[0].id = cudaLaunchAttributeClusterDimension;
                attr[0].val.clusterDim.x = S::CL;
                attr[0].val.clusterDim.y = 1;
                attr[0].val.clusterDim.z = 1;
                cfg.attrs = attr;
                cfg.numAttrs = 1;
                LB_CUDA(cudaLaunchKernelEx(&cfg, ks_inner_pair_kernel<LOGN>, d, ap, 0u));
                launch_counter().fetch_add(1, std::memory_order_relaxed);
            }
            if (!(a.count & 1u)) return;
            // the odd ciphertext goes through the single-ciphertext kernel below
            KsInnerArgs al = a;
            const uint32_t c = a.count - 1;
            const size_t wb = sizeof(W);
            al.dc = static_cast<const uint8_t*>(a.dc) + uint64_t(c) * d.L * d.n * wb;
            al.dn = static_cast<const uint8_t*>(a.dn) + uint64_t(c) * a.d_stride * wb;
            al.acc = static_cast<uint8_t*>(a.acc) + uint64_t(c) * 2 * (d.L + d.K) * d.n * wb;
            al.count = 1;
            launch_ks_inner<LOGN, W>(d, al, s);
            return;
        }
        if (d.dnum <= kMaxPlanes && ks_use_planes()) {
            const size_t smem = size_t(d.dnum) * plane_words<LOGN, W>() * sizeof(W);
            static bool configured32 = false;
            if (!configured32) {
                LB_CUDA(cudaFuncSetAttribute(ks_inner_planes_kernel<LOGN, false>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(kMaxPlanes * plane_words<LOGN, W>() * sizeof(W))));
                LB_CUDA(cudaFuncSetAttribute(ks_inner_planes_kernel<LOGN, true>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(kMaxPlanes * plane_words<LOGN, W>() * sizeof(W))));
                configured32 = true;
            }
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = grid_xyz((d.L + d.K) * S::CL, a.count);
            cfg.blockDim = dim3(S::T);
            cfg.dynamicSmemBytes = smem;
            cfg.stream = s;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = S::CL;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            if (d.ks29)
                LB_CUDA(cudaLaunchKernelEx(&cfg, ks_inner_planes_kernel<LOGN, true>, d, a));
            else
                LB_CUDA(cudaLaunchKernelEx(&cfg, ks_inner_planes_kernel<LOGN, false>, d, a));
            launch_counter().fetch_add(1, std::memory_order_relaxed);
            return;
        }
    }
    const size_t smem = (plane_words<LOGN, W>() + 2ull * S::M) * sizeof(W);
    static bool configured = false;
    if (!configured) {
        LB_CUDA(cudaFuncSetAttribute(ks_inner_kernel<LOGN, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        configured = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(uint64_t(a.count) * (d.L + d.K) * S::CL));
    cfg.blockDim = dim3(S::T);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = S::CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    LB_CUDA(cudaLaunchKernelEx(&cfg, ks_inner_kernel<LOGN, W>, d, a));
    launch_counter().fetch_add(1, std::memory_order_relaxed);
}

template <int LOGN, class W>
void launch_moddown(const BfvDev& d, const ModDownArgs& a, cudaStream_t s) {
    using S = NttShape<LOGN>;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid_xyz(d.L * S::CL, uint64_t(a.count) * 2);
    cfg.blockDim = dim3(S::T);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = S::CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if constexpr (sizeof(W) == 4) {
        if (d.ks29 && (ks_pairs() & (4 | 16)) && d.K >= 2 && d.K <= 5 && d.L >= 2) {
            // two target primes per cluster (bit 2: with both components; bit 4: one component)
            if (ks_pairs() & 16) {
                static const bool configured = [] {
                    LB_CUDA(cudaFuncSetAttribute(moddown_quad_kernel<LOGN, 1>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 int(moddown_quad_smem<LOGN, 1>())));
                    return true;
                }();
                (void)configured;
                cfg.gridDim = grid_xyz(((d.L + 1) / 2) * S::CL, uint64_t(a.count) * 2);
                cfg.dynamicSmemBytes = moddown_quad_smem<LOGN, 1>();
                LB_CUDA(cudaLaunchKernelEx(&cfg, moddown_quad_kernel<LOGN, 1>, d, a));
            } else {
                static const bool configured = [] {
                    LB_CUDA(cudaFuncSetAttribute(moddown_quad_kernel<LOGN, 2>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 int(moddown_quad_smem<LOGN, 2>())));
                    return true;
                }();
                (void)configured;
                cfg.gridDim = grid_xyz(((d.L + 1) / 2) * S::CL, a.count);
                cfg.dynamicSmemBytes = moddown_quad_smem<LOGN, 2>();
                LB_CUDA(cudaLaunchKernelEx(&cfg, moddown_quad_kernel<LOGN, 2>, d, a));
            }
            launch_counter().fetch_add(1, std::memory_order_relaxed);
            return;
        }
        if (d.ks29 && (ks_pairs() & 1) && a.count >= md_pair_min()) {
            cfg.gridDim = grid_xyz(d.L * S::CL, a.count);
            LB_CUDA(cudaLaunchKernelEx(&cfg, moddown_pair_kernel<LOGN>, d, a));
            launch_counter().fetch_add(1, std::memory_order_relaxed);
            return;
        }
        if (d.ks29) {
            LB_CUDA(cudaLaunchKernelEx(&cfg, moddown_kernel<LOGN, W, true>, d, a));
            launch_counter().fetch_add(1, std::memory_order_relaxed);
            return;
        }
    }
    LB_CUDA(cudaLaunchKernelEx(&cfg, moddown_kernel<LOGN, W, false>, d, a));
    launch_counter().fetch_add(1, std::memory_order_relaxed);
}

template <class W>
void dispatch_ks_w(int logn, const BfvDev& d, const KsInnerArgs& ka, const ModDownArgs* ma, cudaStream_t s) {
    switch (logn) {
        case 12: ma ? launch_moddown<12, W>(d, *ma, s) : launch_ks_inner<12, W>(d, ka, s); break;
        case 13: ma ? launch_moddown<13, W>(d, *ma, s) : launch_ks_inner<13, W>(d, ka, s); break;
        case 14: ma ? launch_moddown<14, W>(d, *ma, s) : launch_ks_inner<14, W>(d, ka, s); break;
        case 15: ma ? launch_moddown<15, W>(d, *ma, s) : launch_ks_inner<15, W>(d, ka, s); break;
        default: throw std::invalid_argument("unsupported ring degree");
    }
}

void dispatch_ks(int logn, const BfvDev& d, const KsInnerArgs& ka, const ModDownArgs* ma, cudaStream_t s) {
    if (d.ks32)
        dispatch_ks_w<uint32_t>(logn, d, ka, ma, s);
    else
        dispatch_ks_w<uint64_t>(logn, d, ka, ma, s);
}

// Key switch `count` polys d (evaluations over Q, stride d_stride, read
// through x -> x^d_galois when nonzero) and write out_h = add_h + u_h
// (stride out_stride; add_h optional, read through add_galois).
//   1. inverse NTT of d (automorphism folded into the load)
//   2. fused ModUp + NTT + key inner product over Q ∪ P   (ks_inner_kernel)
//   3. inverse NTT of the P limbs of both accumulators
//   4. fused P->Q conversion + NTT + ModDown epilogue     (moddown_kernel)
// All residue operands in the context's residue word St (== the kernels'
// arithmetic word: u32 exactly when ks32); strides in elements.
template <class St>
void key_switch_impl(Context& cx, const St* d_ntt, uint64_t d_stride, uint64_t d_galois, uint64_t key_id,
                     uint32_t count, const St* add0, const St* add1, uint64_t add_stride, uint64_t add_galois,
                     St* out0, St* out1, uint64_t out_stride, cudaStream_t s, const St* sum0 = nullptr,
                     const St* sum1 = nullptr, uint64_t sum_stride = 0) {
    if (!count) return;
    BfvState& st = *cx.bfv();
    const BfvDev& d = st.dev;
    if (d.K == 0) throw std::invalid_argument("key switching needs special primes");
    ensure_key(cx, key_id, s);
    const void* key = key_shoup_ptr(cx, key_id);
    const uint32_t n = d.n, L = d.L, K = d.K, LK = L + K;
    // intermediates in the kernels' word size (u32 when ks32)
    const size_t wb = d.ks32 ? 4 : 8;
    if (wb != sizeof(St)) throw std::logic_error("key switch: residue word does not match the context");
    DeviceBuffer dc(uint64_t(count) * L * n * wb, s);
    {
        // coefficients of d, pre-multiplied by [(D_j/q_i)^-1]_{q_i} for
        // multi-prime digits (folded into the transform's n^-1)
        LimbBatch lb{dc.get(), count, L, 0, uint64_t(L) * n};
        lb.src = reinterpret_cast<const uint64_t*>(d_ntt);  // read as St words
        lb.src_stride = d_stride;
        lb.galois = d_galois;
        lb.packed32 = d.ks32;
        if (d.alpha > 1) {
            lb.last_stage = d.ks_last_q;
            lb.last_stage32 = d.ks_last_q32;
        }
        cx.ntt_inverse(lb, s);
    }
    DeviceBuffer acc(uint64_t(count) * 2 * LK * n * wb, s);
    KsInnerArgs ka{dc.get(), d_ntt, d_stride, d_galois, key, acc.get(), count};
    dispatch_ks(cx.logn(), d, ka, nullptr, s);
    {
        uint8_t* p_limbs = acc.get<uint8_t>() + uint64_t(L) * n * wb;
        LimbBatch pb{reinterpret_cast<uint64_t*>(p_limbs), count * 2, K, L, uint64_t(LK) * n};
        pb.packed32 = d.ks32;
        if (K > 1) {  // times [(P/p_l)^-1]_{p_l}
            pb.last_stage = d.ks_last_p;
            pb.last_stage32 = d.ks_last_p32;
        }
        cx.ntt_inverse(pb, s);
    }
    ModDownArgs ma{acc.get(), add0,  add1,  add_stride, add_galois, sum0,        sum1,
                   sum_stride, out0, out1,  out_stride,
                   d.ks32 ? static_cast<const void*>(d.p_inv32) : static_cast<const void*>(d.p_inv_shoup), count};
    dispatch_ks(cx.logn(), d, ka, &ma, s);
}

// Runs f(St{}) with the context's residue word (uint32_t when ks32).
template <class F>
void with_residue(const Context& cx, F&& f) {
    if (cx.bfv()->dev.ks32)
        f(uint32_t{});
    else
        f(uint64_t{});
}

// A limb batch over residue words: packed32 when the words are u32.
template <class St>
LimbBatch res_batch(St* data, uint32_t polys, uint32_t limbs, uint32_t first_prime, uint64_t stride) {
    LimbBatch b{reinterpret_cast<uint64_t*>(data), polys, limbs, first_prime, stride};
    b.packed32 = sizeof(St) == 4;
    return b;
}

}  // namespace

void key_switch(Context& cx, const void* d, uint64_t key_id, void* u0, void* u1, uint32_t count, cudaStream_t s) {
    const uint64_t LN = uint64_t(cx.L()) * cx.n();
    with_residue(cx, [&](auto w) {
        using St = decltype(w);
        key_switch_impl<St>(cx, static_cast<const St*>(d), LN, 0, key_id, count, nullptr, nullptr, 0, 0,
                            static_cast<St*>(u0), static_cast<St*>(u1), LN, s);
    });
}

// ---- public ciphertext operations ----------------------------------------------

namespace {

// fused encryption for u32 contexts (A/B switch LB_ENC_FUSED=0)
bool enc_fused() {
    static const bool on = [] {
        const char* e = std::getenv("LB_ENC_FUSED");
        return e ? e[0] != '0' : true;
    }();
    return on;
}

template <int LOGN>
void launch_encrypt32(const BfvDev& d, const uint64_t* m, const uint32_t* extra, const int8_t* err, uint32_t count,
                      uint64_t id_base, void* out, cudaStream_t s) {
    using S = NttShape<LOGN>;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(uint64_t(count) * d.L * S::CL));
    cfg.blockDim = dim3(S::T);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = S::CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    LB_CUDA(cudaLaunchKernelEx(&cfg, k_encrypt32<LOGN>, d, m, extra, err, id_base, static_cast<uint32_t*>(out)));
    launch_counter().fetch_add(1, std::memory_order_relaxed);
}

}  // namespace

void encrypt_slots(Context& cx, const int64_t* values, uint32_t B, uint64_t id_base, void* out, cudaStream_t s) {
    const BfvDev& d = cx.bfv()->dev;
    if (!B) return;
    const uint32_t n = d.n, T = d.T, L = d.L;
    if (T == 0) throw std::invalid_argument("context has no plaintext primes");
    const uint32_t count = B * T;
    DeviceBuffer m(uint64_t(count) * n * 8, s);
    k_scatter_slots<<<grid_for(uint64_t(count) * n), kBlock, 0, s>>>(d, values, B, m.get());
    LB_KERNEL_DONE();
    LimbBatch tb{m.get(), count, 1, 0, n};
    tb.prime_map = cx.bfv()->t_map;
    tb.map_period = T;
    cx.ntt_inverse(tb, s);
    if (d.ks32 && enc_fused()) {
        DeviceBuffer extra(uint64_t(count) * n * 4, s), err(uint64_t(count) * n, s);
        k_enc_prep32<<<grid_for(uint64_t(count) * n), kBlock, 0, s>>>(d, m.get(), count, id_base, extra.get<uint32_t>(),
                                                                      err.get<int8_t>());
        LB_KERNEL_DONE();
        switch (cx.logn()) {
            case 12: launch_encrypt32<12>(d, m.get(), extra.get<uint32_t>(), err.get<int8_t>(), count, id_base, out, s); break;
            case 13: launch_encrypt32<13>(d, m.get(), extra.get<uint32_t>(), err.get<int8_t>(), count, id_base, out, s); break;
            case 14: launch_encrypt32<14>(d, m.get(), extra.get<uint32_t>(), err.get<int8_t>(), count, id_base, out, s); break;
            case 15: launch_encrypt32<15>(d, m.get(), extra.get<uint32_t>(), err.get<int8_t>(), count, id_base, out, s); break;
            default: throw std::invalid_argument("unsupported ring degree");
        }
        return;
    }
    with_residue(cx, [&](auto w) {
        using St = decltype(w);
        St* ct = static_cast<St*>(out);
        k_enc_coeffs<St><<<grid_for(uint64_t(count) * n), kBlock, 0, s>>>(d, m.get(), count, id_base, ct);
        LB_KERNEL_DONE();
        cx.ntt_forward(res_batch(ct, count, L, 0, 2ull * L * n), s);
        k_enc_finish<St><<<grid_for(uint64_t(count) * L * n), kBlock, 0, s>>>(d, count, id_base, ct);
        LB_KERNEL_DONE();
    });
}

void decrypt_coeffs(Context& cx, const void* ct, uint32_t B, uint64_t* out, cudaStream_t s) {
    const BfvDev& d = cx.bfv()->dev;
    if (!B) return;
    const uint32_t n = d.n, L = d.L, count = B * d.T;
    DeviceBuffer x(uint64_t(count) * L * n * 8, s);
    with_residue(cx, [&](auto w) {
        using St = decltype(w);
        k_phase<St><<<grid_for(uint64_t(count) * L * n), kBlock, 0, s>>>(d, static_cast<const St*>(ct), count, x.get());
    });
    LB_KERNEL_DONE();
    cx.ntt_inverse(LimbBatch{x.get(), count, L, 0, uint64_t(L) * n}, s);
    k_dec_scale<<<grid_for(uint64_t(count) * n), kBlock, 0, s>>>(d, x.get(), count, out);
    LB_KERNEL_DONE();
}

void decrypt_slots(Context& cx, const void* ct, uint32_t B, uint64_t* out, cudaStream_t s) {
    const BfvDev& d = cx.bfv()->dev;
    if (!B) return;
    const uint32_t n = d.n, T = d.T, count = B * T;
    DeviceBuffer m(uint64_t(count) * n * 8, s);
    decrypt_coeffs(cx, ct, B, m.get(), s);
    LimbBatch tb{m.get(), count, 1, 0, n};
    tb.prime_map = cx.bfv()->t_map;
    tb.map_period = T;
    cx.ntt_forward(tb, s);
    k_gather_slots<<<grid_for(uint64_t(count) * n), kBlock, 0, s>>>(d, m.get(), count, out);
    LB_KERNEL_DONE();
}

void encode_plain(Context& cx, const int64_t* values, void* pt_mul, void* pt_add, cudaStream_t s) {
    const BfvDev& d = cx.bfv()->dev;
    const uint32_t n = d.n, T = d.T, L = d.L;
    DeviceBuffer m(uint64_t(T) * n * 8, s);
    k_scatter_slots<<<grid_for(uint64_t(T) * n), kBlock, 0, s>>>(d, values, 1, m.get());
    LB_KERNEL_DONE();
    LimbBatch tb{m.get(), T, 1, 0, n};
    tb.prime_map = cx.bfv()->t_map;
    tb.map_period = T;
    cx.ntt_inverse(tb, s);
    with_residue(cx, [&](auto w) {
        using St = decltype(w);
        St* pm = static_cast<St*>(pt_mul);
        St* pa = static_cast<St*>(pt_add);
        k_pt_lift<St><<<grid_for(uint64_t(T) * L * n), kBlock, 0, s>>>(d, m.get(), pm, pa);
        LB_KERNEL_DONE();
        if (pm) cx.ntt_forward(res_batch(pm, T, L, 0, uint64_t(L) * n), s);
        if (pa) cx.ntt_forward(res_batch(pa, T, L, 0, uint64_t(L) * n), s);
    });
}

static EwShape ew_shape(const BfvDev& d, uint32_t count) { return EwShape{count * 2 * d.L, d.L, d.T, d.logn}; }

void ct_add(Context& cx, const void* a, const void* b, void* out, uint32_t count, cudaStream_t s) {
    const BfvDev& d = cx.bfv()->dev;
    if (!count) return;
    const EwShape sh = ew_shape(d, count);
    with_residue(cx, [&](auto w) {
        using St = decltype(w);
        k_add<St><<<ew_grid(sh), kEwThreads, 0, s>>>(d, sh, static_cast<const St*>(a), static_cast<const St*>(b),
                                                     static_cast<St*>(out));
    });
    LB_KERNEL_DONE();
}

static ScalarTab scalar_table(Context& cx, int64_t scalar) {
    ScalarTab tab{};
    for (uint32_t i = 0; i < cx.L(); ++i) {
        const uint64_t q = cx.prime(i);
        int64_t r = scalar % static_cast<int64_t>(q);
        const uint64_t v = r < 0 ? static_cast<uint64_t>(r + static_cast<int64_t>(q)) : static_cast<uint64_t>(r);
        tab.v[i] = make_ulonglong2(v, shoup_companion(v, q));
    }
    return tab;
}

void ct_mul_scalar(Context& cx, const void* a, int64_t scalar, void* out, uint32_t count, cudaStream_t s) {
    const BfvDev& d = cx.bfv()->dev;
    if (!count) return;
    const EwShape sh = ew_shape(d, count);
    with_residue(cx, [&](auto w) {
        using St = decltype(w);
        k_mul_scalar<St><<<ew_grid(sh), kEwThreads, 0, s>>>(d, sh, static_cast<const St*>(a), scalar_table(cx, scalar),
                                                            static_cast<St*>(out));
    });
    LB_KERNEL_DONE();
}

void ct_mul_scalar_add(Context& cx, const void* acc, const void* x, int64_t scalar, void* out, uint32_t count,
                       cudaStream_t s) {
    const BfvDev& d = cx.bfv()->dev;
    if (!count) return;
    const EwShape sh = ew_shape(d, count);
    with_residue(cx, [&](auto w) {
        using St = decltype(w);
        k_mul_scalar_add<St><<<ew_grid(sh), kEwThreads, 0, s>>>(d, sh, static_cast<const St*>(acc),
                                                                static_cast<const St*>(x), scalar_table(cx, scalar),
                                                                static_cast<St*>(out));
    });
    LB_KERNEL_DONE();
}

void ct_mul_plain(Context& cx, const void* a, const void* pt, void* out, uint32_t count, cudaStream_t s) {
    const BfvDev& d = cx.bfv()->dev;
    if (!count) return;
    const EwShape sh = ew_shape(d, count);
    with_residue(cx, [&](auto w) {
        using St = decltype(w);
        k_mul_plain<St><<<ew_grid(sh), kEwThreads, 0, s>>>(d, sh, static_cast<const St*>(a), static_cast<const St*>(pt),
                                                           static_cast<St*>(out));
    });
    LB_KERNEL_DONE();
}

void ct_add_plain(Context& cx, const void* a, const void* pt, void* out, uint32_t count, cudaStream_t s) {
    const BfvDev& d = cx.bfv()->dev;
    if (!count) return;
    const EwShape sh = ew_shape(d, count);
    with_residue(cx, [&](auto w) {
        using St = decltype(w);
        k_add_plain<St><<<ew_grid(sh), kEwThreads, 0, s>>>(d, sh, static_cast<const St*>(a), static_cast<const St*>(pt),
                                                           static_cast<St*>(out));
    });
    LB_KERNEL_DONE();
}

void ct_rotate(Context& cx, const void* a_in, uint64_t galois, void* out_v, uint32_t count, cudaStream_t s) {
    const BfvDev& d = cx.bfv()->dev;
    if (!count) return;
    if (galois % 2 == 0 || galois >= 2ull * d.n) throw std::invalid_argument("galois element must be odd in [1, 2n)");
    const uint64_t LN = uint64_t(d.L) * d.n;
    with_residue(cx, [&](auto w) {
        using St = decltype(w);
        const St* a = static_cast<const St*>(a_in);
        St* out = static_cast<St*>(out_v);
        // the automorphism is folded into the key switch's loads; an in-place
        // call needs a private copy of the input (outputs scatter by permutation)
        DeviceBuffer copy;
        if (out == a) {
            const uint64_t bytes = uint64_t(count) * 2 * LN * sizeof(St);
            copy = DeviceBuffer(bytes, s);
            LB_CUDA(cudaMemcpyAsync(copy.get(), a, bytes, cudaMemcpyDeviceToDevice, s));
            a = copy.get<St>();
        }
        key_switch_impl<St>(cx, a + LN, 2 * LN, galois, galois, count, a, nullptr, 2 * LN, galois, out, out + LN,
                            2 * LN, s);
    });
}

void ct_rotate_add(Context& cx, const void* base_in, const void* x_in, uint64_t galois, void* out_v, uint32_t count,
                   cudaStream_t s) {
    const BfvDev& d = cx.bfv()->dev;
    if (!count) return;
    if (galois % 2 == 0 || galois >= 2ull * d.n) throw std::invalid_argument("galois element must be odd in [1, 2n)");
    const uint64_t LN = uint64_t(d.L) * d.n;
    with_residue(cx, [&](auto w) {
        using St = decltype(w);
        const St* x = static_cast<const St*>(x_in);
        const St* base = static_cast<const St*>(base_in);
        St* out = static_cast<St*>(out_v);
        DeviceBuffer copy;
        if (out == x || out == base) {  // outputs are written while inputs are gathered
            const uint64_t bytes = uint64_t(count) * 2 * LN * sizeof(St);
            copy = DeviceBuffer(2 * bytes, s);
            LB_CUDA(cudaMemcpyAsync(copy.get(), x, bytes, cudaMemcpyDeviceToDevice, s));
            LB_CUDA(cudaMemcpyAsync(copy.get<uint8_t>() + bytes, base, bytes, cudaMemcpyDeviceToDevice, s));
            x = copy.get<St>();
            base = copy.get<St>() + uint64_t(count) * 2 * LN;
        }
        key_switch_impl<St>(cx, x + LN, 2 * LN, galois, galois, count, x, nullptr, 2 * LN, galois, out, out + LN,
                            2 * LN, s, base, base + LN, 2 * LN);
    });
}

void ct_mul(Context& cx, const void* a_in, const void* b_in, void* out_v, uint32_t count, cudaStream_t s) {
    const BfvDev& d = cx.bfv()->dev;
    if (!count) return;
    if (!cx.bfv()->mul_base_ok)
        throw std::invalid_argument("multiplication needs an auxiliary base B with log2 B >= log2 Q + log2 t + log2 n + 2");
    const uint32_t n = d.n, L = d.L, M = d.M, LM = L + M;
    const uint64_t LN = uint64_t(L) * n;
    with_residue(cx, [&](auto w) {
        using St = decltype(w);
        const St* a = static_cast<const St*>(a_in);
        const St* b = static_cast<const St*>(b_in);
        St* out = static_cast<St*>(out_v);
        constexpr size_t W = sizeof(St);
        // (a) inputs to coefficients: X[c] = [a0 a1 b0 b1]
        DeviceBuffer X(uint64_t(count) * 4 * LN * W, s);
        St* x = X.get<St>();
        LB_CUDA(cudaMemcpy2DAsync(x, 4 * LN * W, a, 2 * LN * W, 2 * LN * W, count, cudaMemcpyDeviceToDevice, s));
        LB_CUDA(cudaMemcpy2DAsync(x + 2 * LN, 4 * LN * W, b, 2 * LN * W, 2 * LN * W, count, cudaMemcpyDeviceToDevice,
                                  s));
        cx.ntt_inverse(res_batch(x, count * 4, L, 0, LN), s);
        // (b) exact Q -> B, (c) to evaluations
        DeviceBuffer Y(uint64_t(count) * 4 * M * n * 8, s);
        const bool small = cx.bfv()->qb_small && d.qb32;
        (small ? k_exact_extend<true, St, uint64_t> : k_exact_extend<false, St, uint64_t>)<<<
            grid_for(uint64_t(count) * 4 * n), kBlock, 0, s>>>(d, x, count * 4, L, 0, d.qhat_inv, d.q_frac,
                                                              d.qhat_mod_b, d.q_mod_b, M, d.bbase, Y.get(),
                                                              d.qhat_inv32, d.q_mod_b32);
        LB_KERNEL_DONE();
        cx.ntt_forward(LimbBatch{Y.get(), count * 4, M, d.bbase, uint64_t(M) * n}, s);
        // (d) tensor over Q ∪ B
        DeviceBuffer D(uint64_t(count) * 3 * LM * n * 8, s);
        k_tensor<St><<<grid_for(uint64_t(count) * LM * n), kBlock, 0, s>>>(d, a, b, Y.get(), count, D.get());
        LB_KERNEL_DONE();
        // (e) back to coefficients over Q ∪ B
        LimbBatch db{D.get(), count * 3, LM, 0, uint64_t(LM) * n};
        db.prime_map = cx.bfv()->qb_map;
        db.map_period = LM;
        db.map_small = cx.bfv()->qb_small;
        cx.ntt_inverse(db, s);
        // (f) scale by t/Q into B, (g) exact B -> Q (in residue words), (h) to evaluations
        DeviceBuffer Z(uint64_t(count) * 3 * M * n * 8, s);
        (small && L + 1 <= 15 ? k_scale<true> : k_scale<false>)<<<grid_for(uint64_t(count) * 3 * n), kBlock, 0, s>>>(
            d, D.get(), count * 3, 3, Z.get());
        LB_KERNEL_DONE();
        DeviceBuffer E(uint64_t(count) * 3 * LN * W, s);
        St* e = E.get<St>();
        (small ? k_exact_extend<true, uint64_t, St> : k_exact_extend<false, uint64_t, St>)<<<
            grid_for(uint64_t(count) * 3 * n), kBlock, 0, s>>>(d, Z.get(), count * 3, M, d.bbase, d.bhat_inv,
                                                              d.b_frac, d.bhat_mod_q, d.b_mod_q, L, 0, e,
                                                              d.bhat_inv32, d.b_mod_q32);
        LB_KERNEL_DONE();
        cx.ntt_forward(res_batch(e, count * 3, L, 0, LN), s);
        // (i) relinearize e2 and add into (e0, e1)
        key_switch_impl<St>(cx, e + 2 * LN, 3 * LN, 0, kRelinKeyId, count, e, e + LN, 3 * LN, 0, out, out + LN,
                            2 * LN, s);
    });
}

}  // namespace lb
