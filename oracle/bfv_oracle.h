/*
 * bfv_oracle.h — CPU restatement of the BFV-RNS ciphertext arithmetic.
 *
 * TEST INFRASTRUCTURE ONLY (the checker). Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load oracle/_ref/libbfvoracle.so.
 *
 * PARITY STATUS: the reference (packnn) performs no encryption
 * (proj/README.md:10-15); the paper's library, Microsoft
 * SEAL 2.3.1, is not vendored or pinned anywhere. So the
 * ciphertext-level algorithms below are PARITY UNPINNED against the reference;
 * they are pinned (a) against the reference's ring-level semantics by
 * decrypt(op(encrypt(m))) == reference ring-backend op(m) (tests), and
 * (b) against the device implementation coefficient by coefficient.
 * The plaintext-ring conventions follow the reference: negacyclic ring
 * Z[x]/(x^n+1), psi = smallest-base primitive 2n-th root
 * (proj/src/modular.cpp:44-56), slot order by generator 3
 * (proj/src/ring.cpp:57-69), slot_encode = scatter + inverse transform
 * (ring.cpp:138-144), automorphism x -> x^g with sign fold (ring.cpp:155-171).
 *
 * Everything here works in the COEFFICIENT domain with a textbook transform;
 * the device keeps ciphertexts in the (bit-reversed) evaluation domain. The
 * two meet on coefficients: device results are inverse-transformed and
 * compared with these.
 *
 * The algorithm specification (shared with the device, restated here
 * independently) is in DESIGN.md §3; every function cites the section.
 */
#ifndef BFV_ORACLE_H
#define BFV_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bo_ctx bo_ctx;

/* prime groups: q (L ciphertext), p (K special), b (M auxiliary), t (T plaintext) */
bo_ctx* bo_create(uint32_t n, const uint64_t* q, uint32_t L, const uint64_t* p, uint32_t K,
                  const uint64_t* b, uint32_t M, const uint64_t* t, uint32_t T, uint32_t dnum,
                  uint64_t seed);
void bo_destroy(bo_ctx* c);
const char* bo_last_error(void);

/* §3.1 counter-based PRNG and samplers */
uint64_t bo_prng(uint64_t seed, uint64_t stream, uint64_t index);
int bo_secret(bo_ctx* c, int64_t* s_out);                       /* ternary secret, n coeffs */

/* plaintext ring mod t_j (reference conventions) */
int bo_slot_encode(bo_ctx* c, uint32_t tj, const uint64_t* slots, uint64_t* coeffs);
int bo_slot_decode(bo_ctx* c, uint32_t tj, const uint64_t* coeffs, uint64_t* slots);

/* §3.3 encryption: m = coefficients mod t_j; ct = [2][L][n] coefficients */
int bo_encrypt(bo_ctx* c, uint32_t tj, const uint64_t* m, uint64_t ct_id, uint64_t* ct);
/* §3.7 decryption to coefficients mod t_j */
int bo_decrypt(bo_ctx* c, uint32_t tj, const uint64_t* ct, uint64_t* m);
/* decryption phase c0 + c1 s per ciphertext prime ([L][n] coefficients);
 * tests derive the exact noise from it with Python integers */
int bo_phase(bo_ctx* c, const uint64_t* ct, uint64_t* out);

/* §3.4 plaintext operands; pt = slot values mod t_j */
int bo_mul_plain(bo_ctx* c, uint32_t tj, const uint64_t* ct, const uint64_t* slots, uint64_t* out);
int bo_add_plain(bo_ctx* c, uint32_t tj, const uint64_t* ct, const uint64_t* slots, uint64_t* out);
int bo_mul_scalar(bo_ctx* c, const uint64_t* ct, int64_t s, uint64_t* out);
int bo_add(bo_ctx* c, const uint64_t* a, const uint64_t* b, uint64_t* out);

/* §3.5 key switching and rotations */
int bo_galois_key(bo_ctx* c, uint64_t g, uint64_t* key /* [dnum][2][L+K][n] coeffs */);
int bo_rotate(bo_ctx* c, const uint64_t* ct, uint64_t g, uint64_t* out);
/* CPU-baseline timing: reps rotations with the key made once; total seconds */
int bo_time_rotate(bo_ctx* c, const uint64_t* ct, uint64_t g, uint32_t reps, uint64_t* out, double* seconds);
/* §3.6 multiplication: tensor (HPS-style exact scaling) + relinearization */
int bo_mul(bo_ctx* c, uint32_t tj, const uint64_t* a, const uint64_t* b, uint64_t* out);

#ifdef __cplusplus
}
#endif

#endif
