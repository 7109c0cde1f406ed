// Device kernels of the BFV-RNS layer. Elementwise kernels
// are HBM-bound: one thread per coefficient, limb-major coalesced access,
// 128-bit Barrett for variable x variable products, 128-bit accumulation of
// up to 16 products before a single reduction.
#pragma once

#include <cstdint>

#include "bfv.hpp"
#include "modarith.cuh"

namespace lb {

// ---- §3.1 counter-based PRNG (shared with oracle/bfv_oracle.cpp) ------------
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t stream_key(uint64_t seed, uint64_t stream) {
    return mix64(seed ^ mix64(stream));
}
__host__ __device__ __forceinline__ uint64_t prng_at(uint64_t key, uint64_t idx) {
    return mix64(key + idx * 0xD1B54A32D192ED03ull);
}
__host__ __device__ __forceinline__ uint64_t stream_enc_a(uint64_t id, uint32_t r) {
    return (2ull << 56) | ((id & 0xFFFFFFFFFFFFull) << 8) | r;
}
__host__ __device__ __forceinline__ uint64_t stream_enc_e(uint64_t id) {
    return (3ull << 56) | ((id & 0xFFFFFFFFFFFFull) << 8);
}
__host__ __device__ __forceinline__ uint64_t stream_ksk_a(uint64_t key, uint32_t j, uint32_t r) {
    return (4ull << 56) | ((key & 0xFFFFFFFFFFull) << 16) | (uint64_t(j) << 8) | r;
}
__host__ __device__ __forceinline__ uint64_t stream_ksk_e(uint64_t key, uint32_t j) {
    return (5ull << 56) | ((key & 0xFFFFFFFFFFull) << 16) | (uint64_t(j) << 8);
}
constexpr uint64_t kStreamSecret = 1ull << 56;

__device__ __forceinline__ uint64_t sample_uniform(uint64_t q, uint64_t r) { return mulhi64(r, q); }
__device__ __forceinline__ int64_t sample_ternary(uint64_t r) {
    const uint64_t v = mulhi64(r, 3);
    return v == 2 ? -1 : static_cast<int64_t>(v);
}
__device__ __forceinline__ int64_t sample_cbd21(uint64_t r) {
    return __popcll(r & 0x1FFFFFull) - __popcll((r >> 21) & 0x1FFFFFull);
}

__device__ __forceinline__ Modulus modulus_of(const PrimeDev& P) { return Modulus{P.q, P.ratio_lo, P.ratio_hi}; }

// signed integer -> [0, q)
__device__ __forceinline__ uint64_t reduce_signed(int64_t v, const Modulus& m) {
    const bool neg = v < 0;
    const uint64_t u = neg ? static_cast<uint64_t>(-(v + 1)) + 1 : static_cast<uint64_t>(v);
    const uint64_t r = reduce_u64(u, m);
    return (neg && r) ? m.q - r : r;
}

// 128-bit accumulator for sums of up to 2^6 products of 62-bit values.
struct Acc128 {
    uint64_t hi = 0, lo = 0;
    __device__ __forceinline__ void mac(uint64_t a, uint64_t b) {
        uint64_t h, l;
        mul_wide(a, b, h, l);
        lo += l;
        hi += h + (lo < l ? 1 : 0);
    }
    __device__ __forceinline__ void add(uint64_t a) {
        lo += a;
        hi += (lo < a ? 1 : 0);
    }
};

// Reduction of an Acc128 (value < 2^126) into [0, q): the Barrett estimate
// can be low by up to two multiples for such wide inputs.
__device__ __forceinline__ uint64_t reduce_acc(const Acc128& a, const Modulus& m) {
    uint64_t carry = mulhi64(a.lo, m.ratio_lo);
    uint64_t t2hi, t2lo;
    mul_wide(a.lo, m.ratio_hi, t2hi, t2lo);
    uint64_t t1 = t2lo + carry;
    uint64_t t3 = t2hi + (t1 < t2lo ? 1 : 0);
    mul_wide(a.hi, m.ratio_lo, t2hi, t2lo);
    uint64_t s = t1 + t2lo;
    carry = t2hi + (s < t1 ? 1 : 0);
    uint64_t qest = a.hi * m.ratio_hi + t3 + carry;
    uint64_t r = a.lo - qest * m.q;
    r = r >= m.q ? r - m.q : r;
    return r >= m.q ? r - m.q : r;
}

// 64.64 fixed-point product y * F / 2^64 where F = (hi, lo) is a 128-bit
// fraction: returns (integer part, 64 fractional bits) of y*hi + mulhi(y, lo)
// read as a 128-bit value.
__device__ __forceinline__ void fixmul(uint64_t y, ulonglong2 F, uint64_t& ip, uint64_t& fp) {
    uint64_t h, l;
    mul_wide(y, F.x, h, l);
    const uint64_t add = mulhi64(y, F.y);
    l += add;
    h += (l < add ? 1 : 0);
    ip = h;
    fp = l;
}

}  // namespace lb
