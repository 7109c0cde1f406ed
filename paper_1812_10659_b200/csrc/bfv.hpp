// BFV-RNS state attached to a Context: precomputed RNS constants, the secret
// key and the key-switching keys, plus the batched ciphertext operations.
//
// Algorithm specification: DESIGN.md §3 (restated independently by the CPU
// oracle in oracle/bfv_oracle.cpp). Device layout:
//   ciphertext  [2][L][n]       NTT domain (bit-reversed), limb-major
//   message     [T][2][L][n]    one ciphertext per plaintext prime t_j
//   batch       [B][T][2][L][n] B independent messages (images)
//   ks key      [dnum][2][L+K][n] NTT domain (b_j, a_j)
// Ciphertext c of a batch uses plaintext prime t_{c mod T}.
#pragma once

#include <map>
#include <mutex>

#include "context.hpp"

namespace lb {

struct BfvDev {
    uint32_t n, logn, L, K, M, T, dnum, alpha;
    uint32_t pbase, bbase, tbase;  // prime-table offsets of P, B, T (Q starts at 0)
    uint64_t seed;
    const PrimeDev* primes;
    PrimeTab32 tab32;            // the context's kernel-parameter prime table (ntt.cuh)
    const uint64_t* s_ntt;       // [L+K+M][n] secret, NTT domain, table order
    const uint32_t* slot_pos;    // [n] device NTT position of slot i
    const uint32_t* pos_slot;    // [n] inverse map
    // encryption / plaintext addition
    const uint64_t* delta;       // [T][L] floor(Q/t_j) mod q_i
    const uint64_t* q_mod_t;     // [T] [Q]_{t_j}
    // decryption
    const uint64_t* qhat_inv;    // [L] [(Q/q_i)^-1]_{q_i}
    const ulonglong2* phi;       // [T][L] floor([t_j]_{q_i} 2^128 / q_i)
    const uint64_t* phi_int;     // [T][L] floor(t_j / q_i)
    // exact extension Q -> B
    const ulonglong2* q_frac;    // [L] floor(2^128 / q_i)
    const uint64_t* qhat_mod_b;  // [L][M]
    const uint64_t* q_mod_b;     // [M]
    // exact extension B -> Q
    const uint64_t* bhat_inv;    // [M]
    const ulonglong2* b_frac;    // [M]
    const uint64_t* bhat_mod_q;  // [M][L]
    const uint64_t* b_mod_q;     // [L]
    // scaling t/Q (per plaintext prime)
    const ulonglong2* theta;     // [T][L]
    const uint64_t* w_mod_b;     // [T][L][M]
    const uint64_t* tqinv_b;     // [T][M]
    // key switching
    const uint64_t* dhat_inv;    // [L] [(D_j/q_i)^-1]_{q_i}, i in digit j
    const uint64_t* dhat_mod;    // [L][L+K] [D_j/q_i]_r
    const uint64_t* phat_inv;    // [K]
    const uint64_t* phat_mod_q;  // [K][L]
    const uint64_t* p_inv_q;     // [L]
    const uint64_t* p_mod_qp;    // [L+K] [P]_r (key generation)
    const ulonglong2* p_inv_shoup;  // [L] (P^-1 mod q_r, Shoup companion)
    // fused key switch (Shoup pairs): ModUp constants [D_j/q_i]_r per
    // (i, r in Q∪P), ModDown constants [P/p_l]_{q_r} per (l, r in Q), and the
    // inverse-transform final-stage constants that fold [(D_j/q_i)^-1]_{q_i}
    // (per q limb) and [(P/p_l)^-1]_{p_l} (per p limb) into n^-1
    const ulonglong2* dhat_mod_sh;   // [L][L+K]
    const ulonglong2* phat_mod_sh;   // [K][L]
    const ulonglong2* ks_last_q;     // [L][2]
    const ulonglong2* ks_last_p;     // [K][2]
    // 32-bit copies of the five tables above (companions floor(w 2^32 / r)),
    // present when every prime of Q and P is below 2^30: the key switch then
    // runs on 32-bit words (ks32) and keys are stored as uint2 pairs
    bool ks32;
    const uint2* p_inv32;            // [L]
    const uint2* dhat_mod_sh32;      // [L][L+K]
    const uint2* phat_mod_sh32;      // [K][L]
    const uint2* ks_last_q32;        // [L][2]
    const uint2* ks_last_p32;        // [K][2]
    // ks32 with every prime of Q and P in (2^28, 2^29): base conversions and
    // the key inner product sum plain 32x32 -> 64-bit products (< 2^61 for
    // up to 8 terms) and reduce once with mu60[r] = floor(2^60 / r)
    bool ks29;
    const uint32_t* mu60;            // [L+K]
    // 32-bit encryption / decryption constants (ks32): floor(Q/t_j) mod q_i
    // and 1 with their companions, and the secret's evaluations over Q
    const uint2* delta32;            // [T][L]
    const uint2* one32;              // [L] (1, floor(2^32 / q_i))
    const uint2* s32;                // [L][n]
    // 32-bit exact base extension (every prime of Q and B below 2^30):
    // Shoup pairs of [(Q/q_i)^-1]_{q_i}, [(B/b_m)^-1]_{b_m}, [Q]_{b_m},
    // [B]_{q_i}, and per table prime (2^32 mod r, companion, floor(2^32/r))
    bool qb32;
    const uint2* qhat_inv32;         // [L]
    const uint2* bhat_inv32;         // [M]
    const uint2* q_mod_b32;          // [M]
    const uint2* b_mod_q32;          // [L]
    const uint4* red32;              // [L+K+M] (zero entries for primes >= 2^30)
};

// Residue word of a context's ciphertexts and plaintext operands in HBM:
// uint32_t when every ciphertext and special prime is below 2^30 (ks32: the
// key switch computes in 32-bit words too), else uint64_t. Key material and
// internal extended-basis buffers stay uint64_t.
inline size_t residue_bytes(const BfvDev& d) { return d.ks32 ? 4 : 8; }

// Opaque device handle of a key-switching key.
struct KsKey {
    DeviceBuffer buf;    // [dnum][2][L+K][n]
    DeviceBuffer shoup;  // same entries as (value, Shoup companion) pairs:
                         // ulonglong2, or uint2 with 32-bit companions (ks32)
};

struct BfvState {
    BfvDev dev{};
    DeviceBuffer consts;
    // prime maps for LimbBatch (device int16 arrays inside `consts`)
    const int16_t* t_map = nullptr;   // [T]          t_j
    const int16_t* qb_map = nullptr;  // [L+M]        Q then B
    bool qb_small = false;            // every prime of Q and B is below 2^30
    bool mul_base_ok = false;         // B large enough for the exact tensor product
    const int16_t* ks_map = nullptr;  // [dnum][L+K]  Q∪P minus digit j's primes
    DeviceBuffer secret;
    DeviceBuffer secret32;  // ks32: (s mod q_i, companion) over Q, uint2 [L][n]
    std::map<uint64_t, KsKey> keys;  // key id -> key (0 = relinearization)
    std::mutex mu;
};

// Key ids: relinearization key for s^2 is id 0, Galois key
// for x -> x^g is id g (odd, >= 3).
constexpr uint64_t kRelinKeyId = 0;

// ---- batched ciphertext operations (bfv.cu) ----------------------------------
// `count` = number of ciphertexts; ciphertext c uses t_{c mod T}. Ciphertext
// and plaintext-operand buffers hold residue words (residue_bytes).

// values: device int64 [B][n] slot values (one vector per message, reduced
// mod each t_j); out: [B][T][2][L][n]; ciphertext id = id_base + c.
void encrypt_slots(Context& cx, const int64_t* values, uint32_t B, uint64_t id_base, void* out, cudaStream_t s);
// out: [B][T][n] slot residues mod t_j
void decrypt_slots(Context& cx, const void* ct, uint32_t B, uint64_t* out, cudaStream_t s);
// out: [B][T][n] plaintext coefficients mod t_j (before slot decoding)
void decrypt_coeffs(Context& cx, const void* ct, uint32_t B, uint64_t* out, cudaStream_t s);

// values: device int64 [n] (shared by every message); pt_mul / pt_add:
// [T][L][n] NTT-domain plaintext operands (centered lift; round(Q m / t)).
void encode_plain(Context& cx, const int64_t* values, void* pt_mul, void* pt_add, cudaStream_t s);

void ct_add(Context& cx, const void* a, const void* b, void* out, uint32_t count, cudaStream_t s);
void ct_mul_scalar(Context& cx, const void* a, int64_t scalar, void* out, uint32_t count, cudaStream_t s);
// pt: [T][L][n], broadcast over messages
void ct_mul_plain(Context& cx, const void* a, const void* pt_mul, void* out, uint32_t count, cudaStream_t s);
void ct_add_plain(Context& cx, const void* a, const void* pt_add, void* out, uint32_t count, cudaStream_t s);
void ct_rotate(Context& cx, const void* a, uint64_t galois, void* out, uint32_t count, cudaStream_t s);
// fused forms used by the evaluator (one counted rotation / scalar product
// plus one counted addition, one pass over memory):
//   out = base + rotate_g(x)          out = acc + scalar * x
void ct_rotate_add(Context& cx, const void* base, const void* x, uint64_t galois, void* out, uint32_t count,
                   cudaStream_t s);
void ct_mul_scalar_add(Context& cx, const void* acc, const void* x, int64_t scalar, void* out, uint32_t count,
                       cudaStream_t s);
void ct_mul(Context& cx, const void* a, const void* b, void* out, uint32_t count, cudaStream_t s);

// key material
void ensure_key(Context& cx, uint64_t key_id, cudaStream_t s);
const uint64_t* key_ptr(Context& cx, uint64_t key_id);
// raw polynomial automorphism in the NTT domain over [polys][limbs][n]
void automorphism_ntt(Context& cx, const void* in, void* out, uint32_t polys, uint32_t limbs, uint64_t galois,
                      cudaStream_t s);
// raw key switch of d ([count][L][n], NTT) -> u0, u1 ([count][L][n], NTT)
void key_switch(Context& cx, const void* d, uint64_t key_id, void* u0, void* u1, uint32_t count, cudaStream_t s);

// Record-tensor dense layer (simd.cu): outs[r] = sum_i W[r][i] * xs[i] for
// R output and F input ciphertext groups of `cts` ciphertexts each; xs, outs:
// device arrays of device pointers; W: device int64 [R][F], |W| < 2^31
// (small_weights: |W| < 2^15, enabling the 32-bit path when every q < 2^30).
void simd_weighted_sums(Context& cx, const void* const* xs, uint32_t F, void* const* outs, uint32_t R,
                        const int64_t* W, bool small_weights, uint32_t cts, cudaStream_t s);

}  // namespace lb
