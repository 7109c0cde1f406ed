// 64-bit modular arithmetic for RNS limbs on the sm_100a integer pipes.
//
// Every modulus is an odd prime q < 2^62, so values in [0, 4q) fit a u64 and
// the Harvey lazy butterflies below never overflow. Two reduction flavours:
//   * Shoup (constant operand w with companion w' = floor(w * 2^64 / q)):
//       x * w mod q in [0, 2q) with one mul.hi and two mul.lo; used for NTT
//       twiddles and every per-prime constant.
//   * Barrett-128 (both operands variable): 128-bit product reduced with the
//       two-word ratio floor(2^128 / q); used for ct x pt, tensor products and
//       key inner products.
// The reference does the same arithmetic with `unsigned __int128 % p`
// (proj/include/packnn/modular.hpp:8-23); results are identical in [0, q).
#pragma once

#include <cstdint>

#if defined(__CUDACC__)
#define LB_HD __host__ __device__ __forceinline__
#else
#define LB_HD inline
#endif

namespace lb {

struct Modulus {
    uint64_t q;
    uint64_t ratio_lo;  // floor(2^128 / q), low word
    uint64_t ratio_hi;  // high word
};

LB_HD uint64_t mulhi64(uint64_t a, uint64_t b) {
#if defined(__CUDA_ARCH__)
    return __umul64hi(a, b);
#else
    return static_cast<uint64_t>((static_cast<unsigned __int128>(a) * b) >> 64);
#endif
}

// (hi, lo) = a * b
LB_HD void mul_wide(uint64_t a, uint64_t b, uint64_t& hi, uint64_t& lo) {
    lo = a * b;
    hi = mulhi64(a, b);
}

LB_HD uint64_t add_mod(uint64_t a, uint64_t b, uint64_t q) {
    uint64_t s = a + b;
    return s >= q ? s - q : s;
}

LB_HD uint64_t sub_mod(uint64_t a, uint64_t b, uint64_t q) {
    return a >= b ? a - b : a + q - b;
}

LB_HD uint64_t neg_mod(uint64_t a, uint64_t q) { return a == 0 ? 0 : q - a; }

// Shoup companion floor(w * 2^64 / q) for w < q (host side only).
inline uint64_t shoup_companion(uint64_t w, uint64_t q) {
    return static_cast<uint64_t>((static_cast<unsigned __int128>(w) << 64) / q);
}

// 32-bit Shoup companion floor(w * 2^32 / q) for w < q < 2^30 (host side).
inline uint32_t shoup_companion32(uint64_t w, uint64_t q) { return static_cast<uint32_t>((w << 32) / q); }

// Primes below this bound are transformed with 32-bit words (4q < 2^32).
constexpr uint64_t kWord32Bound = uint64_t{1} << 30;

// x * w mod q, result in [0, 2q); any 64-bit x.
LB_HD uint64_t mul_shoup_lazy(uint64_t x, uint64_t w, uint64_t wp, uint64_t q) {
    uint64_t hi = mulhi64(x, wp);
    return x * w - hi * q;
}

LB_HD uint64_t mul_shoup(uint64_t x, uint64_t w, uint64_t wp, uint64_t q) {
    uint64_t r = mul_shoup_lazy(x, w, wp, q);
    return r >= q ? r - q : r;
}

// Barrett reduction of a 128-bit value (hi, lo) with hi < q (true for any
// product of two values below q). Result in [0, q).
LB_HD uint64_t barrett_reduce_128(uint64_t hi, uint64_t lo, const Modulus& m) {
    // floor(x * ratio / 2^128) estimated from the three significant partial
    // products; the estimate is low by at most one multiple of q.
    uint64_t carry = mulhi64(lo, m.ratio_lo);
    uint64_t t2hi, t2lo;
    mul_wide(lo, m.ratio_hi, t2hi, t2lo);
    uint64_t t1 = t2lo + carry;
    uint64_t t3 = t2hi + (t1 < t2lo ? 1 : 0);
    mul_wide(hi, m.ratio_lo, t2hi, t2lo);
    uint64_t s = t1 + t2lo;
    carry = t2hi + (s < t1 ? 1 : 0);
    uint64_t qest = hi * m.ratio_hi + t3 + carry;
    uint64_t r = lo - qest * m.q;
    return r >= m.q ? r - m.q : r;
}

LB_HD uint64_t mul_mod(uint64_t a, uint64_t b, const Modulus& m) {
    uint64_t hi, lo;
    mul_wide(a, b, hi, lo);
    return barrett_reduce_128(hi, lo, m);
}

// Reduce any 64-bit value into [0, q).
LB_HD uint64_t reduce_u64(uint64_t a, const Modulus& m) { return barrett_reduce_128(0, a, m); }

}  // namespace lb
