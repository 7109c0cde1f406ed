/*
 * lola_b200.h — C-ABI of the B200-native BFV-RNS hot path for LoLa
 * (arXiv 1812.10659). Plain pointers and sizes only; no C++ or torch types.
 *
 * The reference (packnn, /root/reference/proj) has no FFI: its backend
 * boundary is the C++ EvalContext / Evaluator / BackendKind interface
 * (proj/include/packnn/evaluator.hpp:12-91), selected by an
 * `if (cx_->kind() == BackendKind::Ring)` inside each Evaluator method
 * (proj/src/evaluator.cpp:84-85,106,166,191,214,262-270,307). Each entry
 * point below names the reference function it replaces.
 *
 * Conventions
 *   - Every function returns 0 on success; nonzero codes follow the
 *     reference CLI's exit-code map (proj/src/cli.cpp:177-192):
 *       1 internal/CUDA error, 3 invalid argument (std::invalid_argument),
 *       4 depth or magnitude budget (depth_error / magnitude_error),
 *       5 plan divergence (std::logic_error).
 *     lb_last_error() returns the message of the calling thread's last error.
 *   - `stream` is a cudaStream_t (NULL = the legacy default stream).
 *   - Device pointers are plain pointers into device memory. Limb batches of
 *     the NTT engine are `uint64_t*`. Ciphertexts and plaintext operands
 *     ("residue buffers", `void*` below) hold the context's RESIDUE WORD:
 *     uint32_t when every ciphertext and special prime is below 2^30 (the
 *     32-bit word kernels; half the HBM traffic), else uint64_t — see
 *     lb_context_residue_bytes.
 *   - RNS layout is limb-major: a polynomial is `limbs` contiguous length-n
 *     u64 arrays in [0, q_i); batches of polynomials are contiguous with a
 *     caller-given stride (in elements).
 *   - Prime table order inside a context: q_0..q_{L-1} (ciphertext),
 *     p_0..p_{K-1} (special), b_0..b_{M-1} (auxiliary), t_0..t_{T-1}
 *     (plaintext CRT primes).
 *   - NTT-domain ("evaluation") data is in BIT-REVERSED order:
 *     element bitrev(k) holds a(psi^(2k+1)), where psi is the reference's
 *     smallest-base primitive 2n-th root (proj/src/modular.cpp:44-56) and
 *     NttTables::forward returns the same values in natural order k
 *     (proj/src/ring.cpp:97-104).
 */
#ifndef LOLA_B200_H
#define LOLA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lb_context lb_context;

typedef struct {
    uint32_t n;            /* ring degree, power of two in [4096, 32768] */
    uint32_t num_q;        /* ciphertext RNS primes (L) */
    uint32_t num_p;        /* special primes for hybrid key switching (K) */
    uint32_t num_b;        /* auxiliary base of the exact tensor product (>= num_q + 1) */
    uint32_t num_t;        /* plaintext CRT primes (independent BFV instances) */
    const uint64_t* q;     /* each prime < 2^62, == 1 mod 2n, all distinct */
    const uint64_t* p;
    const uint64_t* b;
    const uint64_t* t;
    uint32_t dnum;         /* key-switch digits (0 = num_q) */
    uint64_t seed;         /* secret key / key material seed */
    int32_t device;        /* CUDA device ordinal (this library's runtime keeps its
                              own current device: callers pass torch's LOCAL_RANK) */
} lb_params;

/* ---- errors, setup ----------------------------------------------------- */

const char* lb_last_error(void);

/* Deterministic search: the `count` largest primes below 2^bits that are
 * == 1 mod 2^log_mod, skipping the `num_exclude` values in `exclude`. */
int lb_find_primes(uint32_t bits, uint32_t log_mod, uint32_t count, const uint64_t* exclude,
                   uint32_t num_exclude, uint64_t* out);

/* Replaces EvalContext::EvalContext's table build (proj/src/evaluator.cpp:36-46,
 * ring.cpp:29-71) for every prime of the chain; also generates the BFV
 * constants and the secret key from `seed`. */
int lb_context_create(const lb_params* params, lb_context** out);
int lb_context_destroy(lb_context* cx);
int lb_context_prime(const lb_context* cx, uint32_t index, uint64_t* prime, uint64_t* psi);
/* residue word of the context's ciphertexts and plaintext operands: 4
 * (uint32_t; every ciphertext and special prime below 2^30) or 8 bytes */
int lb_context_residue_bytes(const lb_context* cx, uint32_t* bytes);
/* pre-grow the device's stream-ordered allocation pool by `bytes` (kept:
 * the pool's release threshold is unbounded), so a long-running session
 * never maps fresh device memory mid-run */
int lb_pool_reserve(lb_context* cx, uint64_t bytes);
int lb_sync(lb_context* cx, void* stream);

/* ---- NTT engine (replaces NttTables::forward / inverse, ring.cpp:97-115) --
 * data: [polys][limbs][n] (poly stride `poly_stride` elements), limb l of
 * each poly uses prime table entry first_prime + l. In place. */
int lb_ntt_forward(lb_context* cx, uint64_t* data, uint32_t polys, uint32_t limbs,
                   uint32_t first_prime, uint64_t poly_stride, void* stream);
int lb_ntt_inverse(lb_context* cx, uint64_t* data, uint32_t polys, uint32_t limbs,
                   uint32_t first_prime, uint64_t poly_stride, void* stream);
/* The same on u32 residue words (the storage word of ciphertexts whose
 * primes are all below 2^30, and of the key switch's intermediates: the
 * transforms the hot path runs). Every limb's prime must be below 2^30. */
int lb_ntt_forward_u32(lb_context* cx, uint32_t* data, uint32_t polys, uint32_t limbs,
                       uint32_t first_prime, uint64_t poly_stride, void* stream);
int lb_ntt_inverse_u32(lb_context* cx, uint32_t* data, uint32_t polys, uint32_t limbs,
                       uint32_t first_prime, uint64_t poly_stride, void* stream);

/* ---- BFV ciphertext operations ---------------------------
 * A ciphertext is [2][L][n] residue words in the evaluation (NTT) domain. A message
 * is T ciphertexts, one per plaintext CRT prime: [T][2][L][n]; a batch of B
 * messages is [B][T][2][L][n]. Ops on `count` ciphertexts use plaintext prime
 * t_{c mod T} for ciphertext c. Every pointer is device memory; outputs may
 * alias inputs. */

/* Evaluator::lift (proj/src/evaluator.cpp:67-91) + encryption: values is
 * [B][n] int64 slot values (reduced mod each t_j, slot-encoded with the
 * reference's generator-3 order, ring.cpp:138-144), out [B][T][2][L][n];
 * ciphertext c gets randomness id id_base + c. id_base = LB_FRESH_IDS draws
 * B*T fresh ids from the context's single counter (the one every evaluator
 * and session uses), so no two encryptions share (a, e); an explicit id_base
 * exists for coefficient parity with the CPU oracle and must not be reused
 * outside tests. */
#define LB_FRESH_IDS UINT64_MAX
int lb_encrypt_slots(lb_context* cx, const int64_t* values, uint32_t B, uint64_t id_base, void* out, void* stream);
/* decryption + Evaluator::lower's slot decode (evaluator.cpp:98-118, before
 * the CRT join): out [B][T][n] slot residues mod t_j. */
int lb_decrypt_slots(lb_context* cx, const void* ct, uint32_t B, uint64_t* out, void* stream);
/* decryption to plaintext coefficients mod t_j, out [B][T][n]. */
int lb_decrypt_coeffs(lb_context* cx, const void* ct, uint32_t B, uint64_t* out, void* stream);
/* plaintext operand encoding (plain_limbs + slot_encode, evaluator.cpp:120-135,
 * 166-169, 214-217): values [n] int64; pt_mul, pt_add [T][L][n] (either may
 * be NULL). */
int lb_encode_plain(lb_context* cx, const int64_t* values, void* pt_mul, void* pt_add, void* stream);

int lb_ct_add(lb_context* cx, const void* a, const void* b, void* out, uint32_t count,
              void* stream);                                            /* Evaluator::add */
int lb_ct_mul_scalar(lb_context* cx, const void* a, int64_t scalar, void* out, uint32_t count,
                     void* stream);                                     /* Evaluator::mul_scalar */
int lb_ct_mul_plain(lb_context* cx, const void* a, const void* pt_mul, void* out, uint32_t count,
                    void* stream);                                      /* Evaluator::mul_plain / mask */
int lb_ct_add_plain(lb_context* cx, const void* a, const void* pt_add, void* out, uint32_t count,
                    void* stream);                                      /* Evaluator::add_plain */
/* automorphism x -> x^galois + key switch (galois_apply ring.cpp:155-171 with
 * Evaluator::rotate_columns / rotate_rows / rotate_bundle, evaluator.cpp:260-332) */
int lb_ct_rotate(lb_context* cx, const void* a, uint64_t galois, void* out, uint32_t count, void* stream);
/* tensor + relinearization (Evaluator::mul, evaluator.cpp:178-202) */
int lb_ct_mul(lb_context* cx, const void* a, const void* b, void* out, uint32_t count, void* stream);

/* key material: key_id 0 = relinearization (s^2), odd g = Galois key x->x^g.
 * lb_key_pointer returns the device key [dnum][2][L+K][n] u64 (NTT domain). */
int lb_keygen(lb_context* cx, uint64_t key_id, void* stream);
int lb_key_pointer(lb_context* cx, uint64_t key_id, const uint64_t** out);
/* raw pieces (residue buffers): NTT-domain automorphism over
 * [polys][limbs][n] (limb l uses prime l) and key switch of [count][L][n]
 * NTT-domain polys. */
int lb_automorphism(lb_context* cx, const void* in, void* out, uint32_t polys, uint32_t limbs, uint64_t galois,
                    void* stream);
int lb_key_switch(lb_context* cx, const void* d, uint64_t key_id, void* u0, void* u1, uint32_t count, void* stream);
/* Galois exponents of the reference (ring.cpp:173-184): right shift of both
 * slot rows by k columns, and the row swap. */
uint64_t lb_galois_exponent_columns(uint32_t n, uint32_t k);
uint64_t lb_galois_exponent_rows(uint32_t n);

/* ---- Evaluator boundary (proj/include/packnn/evaluator.hpp:50-91) ---------
 * The drop-in for the reference's Evaluator on a new BackendKind: every
 * method of Evaluator has one entry point with the same meaning, counting
 * rules (evaluator.cpp:137-332) and budget errors (status 4 for depth_error /
 * magnitude_error, 3 for std::invalid_argument). A message handle is one
 * BATCH of `batch` independent messages (one per image); lifted values are
 * shared by every message unless per_message is set ([batch][count]).
 * Every returned message must be released with lb_message_free. */
typedef struct lb_evaluator lb_evaluator;
typedef struct lb_message lb_message;

int lb_eval_create(lb_context* cx, uint32_t batch, uint32_t max_depth, void* stream, lb_evaluator** out);
int lb_eval_destroy(lb_evaluator* ev);
int lb_eval_fork(const lb_evaluator* ev, lb_evaluator** out);              /* Evaluator::fork */
int lb_eval_absorb(lb_evaluator* ev, const lb_evaluator* child);          /* Evaluator::absorb */
/* out[8]: ct.ct, ct.pt, scalar, mask, add, rot.col, rot.row, live peak (OpCounters) */
int lb_eval_counters(const lb_evaluator* ev, uint64_t* out);
int lb_eval_note_live(lb_evaluator* ev, uint64_t live);
int lb_eval_lift(lb_evaluator* ev, const int64_t* values, uint64_t count, int per_message, lb_message** out);
/* Evaluator::lower: out [batch][n][4] signed 256-bit words (host memory) */
int lb_eval_lower(lb_evaluator* ev, const lb_message* m, uint64_t* out);
int lb_eval_add(lb_evaluator* ev, const lb_message* a, const lb_message* b, lb_message** out);
int lb_eval_add_plain(lb_evaluator* ev, const lb_message* a, const int64_t* values, uint64_t count, lb_message** out);
int lb_eval_mul(lb_evaluator* ev, const lb_message* a, const lb_message* b, lb_message** out);
int lb_eval_mul_plain(lb_evaluator* ev, const lb_message* a, const int64_t* values, uint64_t count, lb_message** out);
int lb_eval_mask(lb_evaluator* ev, const lb_message* a, const uint8_t* bits, uint64_t count, lb_message** out);
int lb_eval_mul_scalar(lb_evaluator* ev, const lb_message* a, int64_t s, lb_message** out);
int lb_eval_rotate_columns(lb_evaluator* ev, const lb_message* a, int64_t k, lb_message** out);
int lb_eval_rotate_rows(lb_evaluator* ev, const lb_message* a, lb_message** out);
int lb_eval_rotate_bundle(lb_evaluator* ev, const lb_message* a, uint32_t amount, lb_message** out);
int lb_message_free(lb_message* m);
/* depth, plain depth, magnitude bound (decimal) of a message */
int lb_message_info(const lb_message* m, uint32_t* depth, uint32_t* plain_depth, char* magnitude, uint64_t cap);
/* device pointer of the message's ciphertexts [batch][T][2][L][n] */
int lb_message_data(const lb_message* m, const void** out);

/* ---- LoLa layer evaluator (proj/src/representation.cpp, kernels.cpp, plan.cpp) --
 * A network is the already-quantized integer network the reference's
 * QuantizedNetwork holds (proj/include/packnn/layers.hpp:100-123): linear
 * stages with a squaring after every stage but the last. */
typedef struct {
    int32_t is_conv;        /* window stage (1) or matrix (0) */
    uint32_t maps;          /* conv: output maps; dense: output rows */
    uint32_t win_h, win_w, stride_h, stride_w;
    uint32_t pad_top, pad_left, pad_bottom, pad_right;
    uint64_t cols;          /* conv: window volume; dense: input length */
    const int64_t* weights; /* maps x cols, row-major (host memory) */
    const int64_t* bias;    /* maps entries or NULL */
} lb_stage;

typedef struct {
    uint32_t channels, in_h, in_w;
    uint32_t num_stages;
    const lb_stage* stages;
    int64_t input_bound;    /* bound on |input value| (magnitude ledger) */
} lb_network;

typedef struct lb_lola_session lb_lola_session;

/* PlanOptions (proj/include/packnn/plan.hpp:35-41). The degree is the
 * context's n (lb_plan_counters takes it explicitly), so the one free
 * option is the interior window-stage matrix threshold (default 100000,
 * plan.cpp:375-380). NULL options = the reference defaults. */
typedef struct {
    uint64_t window_matrix_threshold;
} lb_plan_options;

/* build_plan (proj/src/plan.cpp:582-595) without a device: the predicted
 * per-step counters [steps][7] = (ct.ct, ct.pt, scalar, mask, add, rot.col,
 * rot.row). Strategies: lola-mnist, lola-dense-mnist, lola-cifar,
 * lola-small, linear-features. */
int lb_plan_counters(const lb_network* net, const char* strategy, uint32_t n, uint64_t* counters,
                     uint32_t max_steps, uint32_t* steps_out, uint32_t* depth_needed, uint64_t* predicted_peak);
int lb_plan_counters_ex(const lb_network* net, const char* strategy, uint32_t n, const lb_plan_options* opt,
                        uint64_t* counters, uint32_t max_steps, uint32_t* steps_out, uint32_t* depth_needed,
                        uint64_t* predicted_peak);

/* A plan bound to a device context and a batch of `batch` images; plaintext
 * weights are encoded on the device once and reused across runs. */
int lb_lola_session_create(lb_context* cx, const lb_network* net, const char* strategy, uint32_t batch,
                           uint32_t max_depth, void* stream, lb_lola_session** out);
int lb_lola_session_create_ex(lb_context* cx, const lb_network* net, const char* strategy, uint32_t batch,
                              uint32_t max_depth, const lb_plan_options* opt, void* stream, lb_lola_session** out);
int lb_lola_session_destroy(lb_lola_session* s);
int lb_lola_session_info(const lb_lola_session* s, uint32_t* steps, uint64_t* outputs, uint64_t* input_values);
/* plan.encode_input -> execute -> decode (proj/src/plan.cpp:597-633,
 * cli.cpp:68-93): images [batch][input_values] int64, scores
 * [batch][outputs][4] two's-complement 256-bit little-endian words; each may
 * live on the host or the device. counters: [steps][7] measured per step
 * (NULL ok); times: encode+encrypt, HE steps, decrypt+decode seconds (NULL
 * ok; non-NULL adds stream syncs between phases). Status 5 = a step's
 * counters diverged from the plan's prediction (std::logic_error). */
int lb_lola_session_run(lb_lola_session* s, const int64_t* images, int images_on_device, uint64_t* scores,
                        int scores_on_device, uint64_t* counters, double* times);

/* The same three phases separately: encrypt keeps the encrypted input in the
 * session (images on host or device), execute runs the HE steps on it
 * (input kept, so execute can repeat) and keeps the encrypted result,
 * decrypt decodes that result into scores. */
int lb_lola_session_encrypt(lb_lola_session* s, const int64_t* images, int images_on_device);
int lb_lola_session_execute(lb_lola_session* s, uint64_t* counters);
int lb_lola_session_decrypt(lb_lola_session* s, uint64_t* scores, int scores_on_device);
/* CUDA-graph mode (off by default). On: the next execute runs the plan once
 * (keys, plaintext encodings), captures a second run into a graph and replays
 * it; every later execute (and run) is one graph launch over the same input
 * buffers (encrypt copies new ciphertexts into them). Results, counters and
 * errors are those of the captured run. Off: frees the graph. */
int lb_lola_session_set_graph(lb_lola_session* s, int enable);
/* device pointer of encrypted output message `index` ([batch][T][2][L][n])
 * and the number of output messages (either pointer may be NULL) */
int lb_lola_session_output(const lb_lola_session* s, uint32_t index, const void** data, uint32_t* count);

/* ---- measurement ------------------------------------------------------- */

/* kernels launched by this library since load (monotonic) */
uint64_t lb_launch_count(void);

/* Integer-pipe roof: sustained register-resident Harvey/Shoup butterflies per
 * second (the same butterfly the NTT runs), grid = SMs x blocks_per_sm. */
int lb_bench_butterfly_peak(uint64_t q, int blocks_per_sm, int iters, double* bfly_per_s);

/* Pipe cross-check of that roof: sustained thread-level ops/s of IMAD
 * (mad.lo.u32), IMAD.HI (mul.hi.u32), a dependent add pair (IADD3) and the
 * min(x, x - m) conditional subtraction (VIADDMNMX), and IMAD.WIDE.U32,
 * 8 independent chains per thread; ops_per_s[5]. */
int lb_bench_int_pipes(int iters, double* ops_per_s);

#ifdef __cplusplus
}
#endif

#endif /* LOLA_B200_H */
