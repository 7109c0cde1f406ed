// Host-side number theory for table generation (setup only, never per op).
//
// Restates the reference's scalar routines (proj/src/modular.cpp:5-56) that
// FIX the transform: deterministic Miller-Rabin for u64 and the
// smallest-base primitive root search. Reproducing the latter exactly is what
// makes device NTT evaluations line up with NttTables (ring.cpp:29-35).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace lb::host {

inline uint64_t mulm(uint64_t a, uint64_t b, uint64_t p) {
    return static_cast<uint64_t>(static_cast<unsigned __int128>(a) * b % p);
}

inline uint64_t powm(uint64_t b, uint64_t e, uint64_t p) {
    uint64_t r = 1 % p;
    b %= p;
    for (; e; e >>= 1) {
        if (e & 1) r = mulm(r, b, p);
        b = mulm(b, b, p);
    }
    return r;
}

inline uint64_t invm(uint64_t a, uint64_t p) {
    if (a % p == 0) throw std::invalid_argument("inverse of zero");
    return powm(a, p - 2, p);
}

inline bool is_prime(uint64_t v) {
    if (v < 2) return false;
    static const uint64_t small[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    for (uint64_t s : small)
        if (v % s == 0) return v == s;
    uint64_t d = v - 1;
    int r = 0;
    while ((d & 1) == 0) {
        d >>= 1;
        ++r;
    }
    for (uint64_t a : small) {
        uint64_t x = powm(a, d, v);
        if (x == 1 || x == v - 1) continue;
        bool witness = true;
        for (int i = 1; i < r && witness; ++i) {
            x = mulm(x, x, v);
            if (x == v - 1) witness = false;
        }
        if (witness) return false;
    }
    return true;
}

// Primitive root of unity of power-of-two `order` chosen as in the reference:
// the first base b = 2, 3, ... whose cofactor power c = b^((p-1)/order)
// satisfies c^(order/2) == -1.
inline uint64_t root_of_unity(uint64_t p, uint64_t order) {
    if (!is_prime(p)) throw std::invalid_argument("modulus is not prime");
    if (order == 0 || (order & (order - 1))) throw std::invalid_argument("order must be a power of two");
    if ((p - 1) % order) throw std::invalid_argument("order does not divide p - 1");
    if (order == 1) return 1;
    const uint64_t cof = (p - 1) / order;
    for (uint64_t b = 2; b < p; ++b) {
        uint64_t c = powm(b, cof, p);
        if (powm(c, order / 2, p) == p - 1) return c;
    }
    throw std::invalid_argument("no primitive root found");
}

inline uint32_t bitrev(uint32_t x, int bits) {
    uint32_t r = 0;
    for (int i = 0; i < bits; ++i) r |= ((x >> i) & 1u) << (bits - 1 - i);
    return r;
}

inline int ilog2(uint64_t v) {
    int r = 0;
    while ((uint64_t{1} << r) < v) ++r;
    return r;
}

// Deterministic NTT-friendly prime search: the `count` largest primes
// p < 2^bits with p == 1 (mod 2^log_mod), skipping `exclude`.
inline std::vector<uint64_t> find_primes(int bits, int log_mod, uint32_t count,
                                         const std::vector<uint64_t>& exclude = {}) {
    if (bits < log_mod + 2 || bits > 62) throw std::invalid_argument("bad prime size");
    std::vector<uint64_t> out;
    const uint64_t step = uint64_t{1} << log_mod;
    uint64_t c = ((uint64_t{1} << bits) - 1) / step * step + 1;
    if (c >= (uint64_t{1} << bits)) c -= step;
    for (; c > step && out.size() < count; c -= step) {
        bool skip = false;
        for (uint64_t e : exclude) skip |= (e == c);
        if (!skip && is_prime(c)) out.push_back(c);
    }
    if (out.size() < count) throw std::invalid_argument("not enough primes of that shape");
    return out;
}

}  // namespace lb::host
