// CPU restatement of the BFV-RNS ciphertext arithmetic — the ciphertext
// oracle. TEST INFRASTRUCTURE ONLY; see bfv_oracle.h for scope and parity
// status, DESIGN.md §3 for the algorithm specification it restates.
//
// Deliberately plain: scalar loops, `unsigned __int128 %` for every modular
// product, a textbook natural-order transform, coefficient-domain data.
#include <chrono>
#include "bfv_oracle.h"

#include <algorithm>
#include <array>
#include <climits>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

typedef unsigned __int128 u128;
typedef std::vector<uint64_t> Poly;

thread_local std::string g_err;

uint64_t mulm(uint64_t a, uint64_t b, uint64_t p) { return static_cast<uint64_t>(static_cast<u128>(a) * b % p); }
uint64_t addm(uint64_t a, uint64_t b, uint64_t p) { return static_cast<uint64_t>((static_cast<u128>(a) + b) % p); }
uint64_t subm(uint64_t a, uint64_t b, uint64_t p) { return a >= b ? a - b : a + (p - b); }
uint64_t powm(uint64_t b, uint64_t e, uint64_t p) {
    uint64_t r = 1 % p;
    for (b %= p; e; e >>= 1, b = mulm(b, b, p))
        if (e & 1) r = mulm(r, b, p);
    return r;
}
uint64_t invm(uint64_t a, uint64_t p) { return powm(a % p, p - 2, p); }
uint64_t mulhi(uint64_t a, uint64_t b) { return static_cast<uint64_t>((static_cast<u128>(a) * b) >> 64); }
uint64_t from_signed(int64_t v, uint64_t p) {
    int64_t r = v % static_cast<int64_t>(p);
    return r < 0 ? static_cast<uint64_t>(r + static_cast<int64_t>(p)) : static_cast<uint64_t>(r);
}

// floor(num * 2^128 / d) for num < d, as (hi, lo) words.
void frac128(uint64_t num, uint64_t d, uint64_t& hi, uint64_t& lo) {
    u128 x = static_cast<u128>(num) << 64;
    hi = static_cast<uint64_t>(x / d);
    uint64_t r = static_cast<uint64_t>(x % d);
    x = static_cast<u128>(r) << 64;
    lo = static_cast<uint64_t>(x / d);
}

// ---- §3.1 PRNG ---------------------------------------------------------------
uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
uint64_t prng(uint64_t seed, uint64_t stream, uint64_t idx) {
    const uint64_t key = mix64(seed ^ mix64(stream));
    return mix64(key + idx * 0xD1B54A32D192ED03ull);
}
uint64_t stream_enc_a(uint64_t id, uint32_t r) { return (2ull << 56) | ((id & 0xFFFFFFFFFFFFull) << 8) | r; }
uint64_t stream_enc_e(uint64_t id) { return (3ull << 56) | ((id & 0xFFFFFFFFFFFFull) << 8); }
uint64_t stream_ksk_a(uint64_t key, uint32_t j, uint32_t r) { return (4ull << 56) | ((key & 0xFFFFFFFFFFull) << 16) | (uint64_t(j) << 8) | r; }
uint64_t stream_ksk_e(uint64_t key, uint32_t j) { return (5ull << 56) | ((key & 0xFFFFFFFFFFull) << 16) | (uint64_t(j) << 8); }
const uint64_t kStreamSecret = 1ull << 56;

uint64_t uniform(uint64_t q, uint64_t r) { return mulhi(r, q); }
int64_t ternary(uint64_t r) {
    uint64_t v = mulhi(r, 3);
    return v == 2 ? -1 : static_cast<int64_t>(v);
}
int64_t cbd21(uint64_t r) {
    return __builtin_popcountll(r & 0x1FFFFFull) - __builtin_popcountll((r >> 21) & 0x1FFFFFull);
}

// ---- textbook negacyclic transform (natural order) -------------------------
struct Ntt {
    uint64_t p = 0;
    uint32_t n = 0;
    uint64_t psi = 0;
    std::vector<uint64_t> psi_pow, psi_ipow;
    uint64_t ninv = 0;

    static uint64_t root(uint64_t p, uint64_t order) {
        // same selection rule as the reference: smallest base b >= 2 whose
        // cofactor power has order exactly `order`
        const uint64_t cof = (p - 1) / order;
        for (uint64_t b = 2;; ++b) {
            uint64_t c = powm(b, cof, p);
            if (powm(c, order / 2, p) == p - 1) return c;
        }
    }
    Ntt(uint64_t p_, uint32_t n_) : p(p_), n(n_) {
        if ((p - 1) % (2ull * n)) throw std::invalid_argument("prime not NTT-friendly for n");
        psi = root(p, 2ull * n);
        psi_pow.resize(n);
        psi_ipow.resize(n);
        uint64_t a = 1, b = 1, pi = invm(psi, p);
        for (uint32_t i = 0; i < n; ++i) {
            psi_pow[i] = a;
            psi_ipow[i] = b;
            a = mulm(a, psi, p);
            b = mulm(b, pi, p);
        }
        ninv = invm(n, p);
    }
    // cyclic DFT with root w, natural order in and out (recursive-free
    // decimation in time on a bit-reversed copy)
    void dft(std::vector<uint64_t>& a, uint64_t w) const {
        uint32_t bits = 0;
        while ((1u << bits) < n) ++bits;
        for (uint32_t i = 0; i < n; ++i) {
            uint32_t r = 0;
            for (uint32_t b = 0; b < bits; ++b) r |= ((i >> b) & 1u) << (bits - 1 - b);
            if (i < r) std::swap(a[i], a[r]);
        }
        for (uint32_t len = 2; len <= n; len <<= 1) {
            const uint64_t wl = powm(w, n / len, p);
            std::vector<uint64_t> tw(len / 2);
            tw[0] = 1;
            for (uint32_t k = 1; k < len / 2; ++k) tw[k] = mulm(tw[k - 1], wl, p);
            for (uint32_t s = 0; s < n; s += len)
                for (uint32_t k = 0; k < len / 2; ++k) {
                    uint64_t u = a[s + k], v = mulm(a[s + k + len / 2], tw[k], p);
                    a[s + k] = addm(u, v, p);
                    a[s + k + len / 2] = subm(u, v, p);
                }
        }
    }
    std::vector<uint64_t> forward(const std::vector<uint64_t>& c) const {
        std::vector<uint64_t> a(n);
        for (uint32_t i = 0; i < n; ++i) a[i] = mulm(c[i], psi_pow[i], p);
        dft(a, mulm(psi, psi, p));
        return a;
    }
    std::vector<uint64_t> inverse(const std::vector<uint64_t>& e) const {
        std::vector<uint64_t> a = e;
        dft(a, invm(mulm(psi, psi, p), p));
        for (uint32_t i = 0; i < n; ++i) a[i] = mulm(mulm(a[i], ninv, p), psi_ipow[i], p);
        return a;
    }
};

uint32_t bitrev(uint32_t x, uint32_t n) {
    uint32_t bits = 0, r = 0;
    while ((1u << bits) < n) ++bits;
    for (uint32_t b = 0; b < bits; ++b) r |= ((x >> b) & 1u) << (bits - 1 - b);
    return r;
}

}  // namespace

struct bo_ctx {
    uint32_t n = 0, L = 0, K = 0, M = 0, T = 0, dnum = 0, alpha = 0;
    uint64_t seed = 0;
    std::vector<uint64_t> q, p, b, t;
    std::vector<uint64_t> qp;          // q then p
    std::vector<Ntt> ntt_q, ntt_p, ntt_b, ntt_t;
    std::vector<int64_t> s;            // secret coefficients
    std::vector<uint32_t> slot_to_eval[1];

    const Ntt& ntt_qp(uint32_t r) const { return r < L ? ntt_q[r] : ntt_p[r - L]; }

    // negacyclic product modulo one prime through its transform
    Poly polymul(const Ntt& T_, const Poly& a, const Poly& bb) const {
        auto ea = T_.forward(a), eb = T_.forward(bb);
        for (uint32_t i = 0; i < n; ++i) ea[i] = mulm(ea[i], eb[i], T_.p);
        return T_.inverse(ea);
    }
    // device-convention uniform sample (bit-reversed evaluations) -> coefficients
    Poly uniform_poly(const Ntt& T_, uint64_t stream) const {
        std::vector<uint64_t> ev(n);
        for (uint32_t k = 0; k < n; ++k) ev[k] = uniform(T_.p, prng(seed, stream, bitrev(k, n)));
        return T_.inverse(ev);
    }
    std::vector<int64_t> cbd_poly(uint64_t stream) const {
        std::vector<int64_t> e(n);
        for (uint32_t k = 0; k < n; ++k) e[k] = cbd21(prng(seed, stream, k));
        return e;
    }
    Poly reduce_signed(const std::vector<int64_t>& v, uint64_t pr) const {
        Poly r(n);
        for (uint32_t k = 0; k < n; ++k) r[k] = from_signed(v[k], pr);
        return r;
    }
    // [prod_{k in set, k != skip} primes[k]]_mod
    static uint64_t prod_mod(const std::vector<uint64_t>& pr, size_t lo, size_t hi, size_t skip, uint64_t mod) {
        uint64_t r = 1 % mod;
        for (size_t k = lo; k < hi; ++k)
            if (k != skip) r = mulm(r, pr[k] % mod, mod);
        return r;
    }
};

namespace {

typedef std::vector<Poly> Rns;  // [limb][n]

// σ_g on coefficients, sign folded (reference ring.cpp:155-171 semantics)
Poly galois(const Poly& a, uint64_t g, uint64_t pr, uint32_t n) {
    Poly r(n, 0);
    const uint64_t two_n = 2ull * n;
    for (uint32_t i = 0; i < n; ++i) {
        uint64_t idx = static_cast<uint64_t>(i) * g % two_n;
        if (idx < n)
            r[idx] = a[i];
        else
            r[idx - n] = a[i] == 0 ? 0 : pr - a[i];
    }
    return r;
}

std::vector<int64_t> galois_signed(const std::vector<int64_t>& a, uint64_t g, uint32_t n) {
    std::vector<int64_t> r(n, 0);
    const uint64_t two_n = 2ull * n;
    for (uint32_t i = 0; i < n; ++i) {
        uint64_t idx = static_cast<uint64_t>(i) * g % two_n;
        if (idx < n)
            r[idx] = a[i];
        else
            r[idx - n] = -a[i];
    }
    return r;
}

// §3.5 key generation for target s' (given per prime of Q∪P as coefficients)
// key[j][0] = b_j, key[j][1] = a_j, each over Q∪P.
std::vector<std::array<Rns, 2>> make_key(const bo_ctx& c, uint64_t key_id, const Rns& s_target) {
    const uint32_t LK = c.L + c.K;
    std::vector<std::array<Rns, 2>> key(c.dnum);
    for (uint32_t j = 0; j < c.dnum; ++j) {
        const uint32_t lo = j * c.alpha, hi = std::min(c.L, lo + c.alpha);
        auto e = c.cbd_poly(stream_ksk_e(key_id, j));
        key[j][0].resize(LK);
        key[j][1].resize(LK);
        for (uint32_t r = 0; r < LK; ++r) {
            const Ntt& T_ = c.ntt_qp(r);
            const uint64_t pr = T_.p;
            Poly a = c.uniform_poly(T_, stream_ksk_a(key_id, j, r));
            Poly as = c.polymul(T_, a, c.reduce_signed(c.s, pr));
            Poly er = c.reduce_signed(e, pr);
            Poly bpoly(c.n);
            const bool in_digit = r >= lo && r < hi;
            const uint64_t pmod = bo_ctx::prod_mod(c.p, 0, c.K, SIZE_MAX, pr);
            for (uint32_t k = 0; k < c.n; ++k) {
                uint64_t v = subm(er[k], as[k], pr);
                if (in_digit) v = addm(v, mulm(pmod, s_target[r][k], pr), pr);
                bpoly[k] = v;
            }
            key[j][0][r] = std::move(bpoly);
            key[j][1][r] = std::move(a);
        }
    }
    return key;
}

// §3.5 key switch of d (coefficients over Q) -> (u0, u1) over Q
std::array<Rns, 2> key_switch(const bo_ctx& c, const Rns& d, const std::vector<std::array<Rns, 2>>& key) {
    const uint32_t L = c.L, K = c.K, LK = L + K;
    std::array<Rns, 2> acc;
    for (int k = 0; k < 2; ++k) acc[k].assign(LK, Poly(c.n, 0));
    for (uint32_t j = 0; j < c.dnum; ++j) {
        const uint32_t lo = j * c.alpha, hi = std::min(L, lo + c.alpha);
        // y_i = [d_i * Dhat_i^-1]_{q_i} for i in the digit
        std::vector<Poly> y(hi - lo, Poly(c.n));
        for (uint32_t i = lo; i < hi; ++i) {
            const uint64_t dh_inv = invm(bo_ctx::prod_mod(c.q, lo, hi, i, c.q[i]), c.q[i]);
            for (uint32_t k = 0; k < c.n; ++k) y[i - lo][k] = mulm(d[i][k], dh_inv, c.q[i]);
        }
        for (uint32_t r = 0; r < LK; ++r) {
            const Ntt& T_ = c.ntt_qp(r);
            const uint64_t pr = T_.p;
            Poly ext(c.n, 0);
            if (r >= lo && r < hi) {
                ext = d[r];
            } else {
                for (uint32_t i = lo; i < hi; ++i) {
                    const uint64_t dh = bo_ctx::prod_mod(c.q, lo, hi, i, pr);
                    for (uint32_t k = 0; k < c.n; ++k) ext[k] = addm(ext[k], mulm(y[i - lo][k] % pr, dh, pr), pr);
                }
            }
            for (int kk = 0; kk < 2; ++kk) {
                Poly prod = c.polymul(T_, ext, key[j][kk][r]);
                for (uint32_t k = 0; k < c.n; ++k) acc[kk][r][k] = addm(acc[kk][r][k], prod[k], pr);
            }
        }
    }
    // ModDown
    std::array<Rns, 2> out;
    for (int kk = 0; kk < 2; ++kk) {
        out[kk].resize(L);
        std::vector<Poly> yp(K, Poly(c.n));
        for (uint32_t l = 0; l < K; ++l) {
            const uint64_t ph_inv = invm(bo_ctx::prod_mod(c.p, 0, K, l, c.p[l]), c.p[l]);
            for (uint32_t k = 0; k < c.n; ++k) yp[l][k] = mulm(acc[kk][L + l][k], ph_inv, c.p[l]);
        }
        for (uint32_t i = 0; i < L; ++i) {
            const uint64_t qi = c.q[i];
            const uint64_t pinv = invm(bo_ctx::prod_mod(c.p, 0, K, SIZE_MAX, qi), qi);
            Poly r(c.n);
            for (uint32_t k = 0; k < c.n; ++k) {
                uint64_t conv = 0;
                for (uint32_t l = 0; l < K; ++l)
                    conv = addm(conv, mulm(yp[l][k] % qi, bo_ctx::prod_mod(c.p, 0, K, l, qi), qi), qi);
                r[k] = mulm(subm(acc[kk][i][k], conv, qi), pinv, qi);
            }
            out[kk][i] = std::move(r);
        }
    }
    return out;
}

Rns unpack(const bo_ctx& c, const uint64_t* p, uint32_t limbs) {
    Rns r(limbs, Poly(c.n));
    for (uint32_t l = 0; l < limbs; ++l) std::memcpy(r[l].data(), p + (size_t)l * c.n, c.n * 8);
    return r;
}
void pack(const bo_ctx& c, const Rns& r, uint64_t* p) {
    for (size_t l = 0; l < r.size(); ++l) std::memcpy(p + l * c.n, r[l].data(), c.n * 8);
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// Exact centered base extension (§3.6 step 1/4): x given by residues `res`
// over `from` primes -> residues over `to` primes.
Rns exact_extend(const bo_ctx& c, const Rns& res, const std::vector<uint64_t>& from, const std::vector<uint64_t>& to) {
    const size_t F = from.size();
    std::vector<uint64_t> hinv(F), fhi(F), flo(F);
    for (size_t i = 0; i < F; ++i) {
        hinv[i] = invm(bo_ctx::prod_mod(from, 0, F, i, from[i]), from[i]);
        frac128(1, from[i], fhi[i], flo[i]);  // floor(2^128 / from_i) minus nothing: 1 * 2^128 / f
    }
    Rns out(to.size(), Poly(c.n));
    std::vector<uint64_t> y(F);
    for (uint32_t k = 0; k < c.n; ++k) {
        u128 S = 0;
        for (size_t i = 0; i < F; ++i) {
            y[i] = mulm(res[i][k], hinv[i], from[i]);
            S += static_cast<u128>(y[i] * fhi[i] + mulhi(y[i], flo[i]));
        }
        const uint64_t v = static_cast<uint64_t>((S + (static_cast<u128>(1) << 63)) >> 64);
        for (size_t m = 0; m < to.size(); ++m) {
            const uint64_t tm = to[m];
            uint64_t acc = 0;
            for (size_t i = 0; i < F; ++i)
                acc = addm(acc, mulm(y[i] % tm, bo_ctx::prod_mod(from, 0, F, i, tm), tm), tm);
            const uint64_t fmod = bo_ctx::prod_mod(from, 0, F, SIZE_MAX, tm);
            out[m][k] = subm(acc, mulm(v % tm, fmod, tm), tm);
        }
    }
    return out;
}

}  // namespace

extern "C" {

const char* bo_last_error(void) { return g_err.c_str(); }

uint64_t bo_prng(uint64_t seed, uint64_t stream, uint64_t index) { return prng(seed, stream, index); }

bo_ctx* bo_create(uint32_t n, const uint64_t* q, uint32_t L, const uint64_t* p, uint32_t K, const uint64_t* b,
                  uint32_t M, const uint64_t* t, uint32_t T, uint32_t dnum, uint64_t seed) {
    bo_ctx* c = nullptr;
    int rc = guarded([&] {
        auto* x = new bo_ctx();
        x->n = n;
        x->L = L;
        x->K = K;
        x->M = M;
        x->T = T;
        x->dnum = dnum ? dnum : L;
        x->alpha = (L + x->dnum - 1) / x->dnum;
        x->seed = seed;
        x->q.assign(q, q + L);
        x->p.assign(p, p + K);
        x->b.assign(b, b + M);
        x->t.assign(t, t + T);
        for (auto v : x->q) x->ntt_q.emplace_back(v, n);
        for (auto v : x->p) x->ntt_p.emplace_back(v, n);
        for (auto v : x->b) x->ntt_b.emplace_back(v, n);
        for (auto v : x->t) x->ntt_t.emplace_back(v, n);
        x->s.resize(n);
        for (uint32_t k = 0; k < n; ++k) x->s[k] = ternary(prng(seed, kStreamSecret, k));
        c = x;
    });
    return rc ? nullptr : c;
}

void bo_destroy(bo_ctx* c) { delete c; }

int bo_secret(bo_ctx* c, int64_t* s_out) {
    return guarded([&] { std::memcpy(s_out, c->s.data(), c->n * 8); });
}

// slot (b, j) <-> evaluation at psi^e, e = (-1)^b 3^j mod 2n (ring.cpp:57-69)
static std::vector<uint32_t> slot_map(uint32_t n) {
    std::vector<uint32_t> m(n);
    const uint64_t two_n = 2ull * n;
    uint64_t g = 1;
    for (uint32_t j = 0; j < n / 2; ++j) {
        m[j] = static_cast<uint32_t>((g - 1) / 2);
        m[n / 2 + j] = static_cast<uint32_t>((two_n - g - 1) / 2);
        g = g * 3 % two_n;
    }
    return m;
}

int bo_slot_encode(bo_ctx* c, uint32_t tj, const uint64_t* slots, uint64_t* coeffs) {
    return guarded([&] {
        auto map = slot_map(c->n);
        std::vector<uint64_t> ev(c->n);
        for (uint32_t i = 0; i < c->n; ++i) ev[map[i]] = slots[i];
        auto r = c->ntt_t.at(tj).inverse(ev);
        std::memcpy(coeffs, r.data(), c->n * 8);
    });
}

int bo_slot_decode(bo_ctx* c, uint32_t tj, const uint64_t* coeffs, uint64_t* slots) {
    return guarded([&] {
        auto map = slot_map(c->n);
        auto ev = c->ntt_t.at(tj).forward(std::vector<uint64_t>(coeffs, coeffs + c->n));
        for (uint32_t i = 0; i < c->n; ++i) slots[i] = ev[map[i]];
    });
}

// §3.3: c1 = a, c0 = -a s + e + round(Q m / t)
int bo_encrypt(bo_ctx* c, uint32_t tj, const uint64_t* m, uint64_t ct_id, uint64_t* ct) {
    return guarded([&] {
        const uint64_t t = c->t.at(tj);
        auto e = c->cbd_poly(stream_enc_e(ct_id));
        uint64_t q_mod_t = 1 % t;
        for (auto qi : c->q) q_mod_t = mulm(q_mod_t, qi % t, t);
        for (uint32_t i = 0; i < c->L; ++i) {
            const Ntt& T_ = c->ntt_q[i];
            const uint64_t qi = c->q[i];
            const uint64_t delta = mulm(subm(0, q_mod_t % qi, qi), invm(t, qi), qi);  // -[Q]_t / t mod q_i
            Poly a = c->uniform_poly(T_, stream_enc_a(ct_id, i));
            Poly as = c->polymul(T_, a, c->reduce_signed(c->s, qi));
            for (uint32_t k = 0; k < c->n; ++k) {
                uint64_t v = subm(from_signed(e[k], qi), as[k], qi);
                // round(Q m / t) = Delta m + floor(([Q]_t m + floor(t/2)) / t)
                const uint64_t extra = (q_mod_t * m[k] + (t >> 1)) / t;
                v = addm(v, addm(mulm(delta, m[k] % qi, qi), extra % qi, qi), qi);
                ct[(size_t)i * c->n + k] = v;
                ct[((size_t)c->L + i) * c->n + k] = a[k];
            }
        }
    });
}

// §3.7: m = round(t x / Q) mod t with the fixed-point sum
int bo_decrypt(bo_ctx* c, uint32_t tj, const uint64_t* ct, uint64_t* m) {
    return guarded([&] {
        const uint64_t t = c->t.at(tj);
        Rns x(c->L);
        for (uint32_t i = 0; i < c->L; ++i) {
            const uint64_t qi = c->q[i];
            Poly c0(ct + (size_t)i * c->n, ct + (size_t)(i + 1) * c->n);
            Poly c1(ct + (size_t)(c->L + i) * c->n, ct + (size_t)(c->L + i + 1) * c->n);
            Poly p = c->polymul(c->ntt_q[i], c1, c->reduce_signed(c->s, qi));
            x[i].resize(c->n);
            for (uint32_t k = 0; k < c->n; ++k) x[i][k] = addm(c0[k], p[k], qi);
        }
        std::vector<uint64_t> hinv(c->L), phi_hi(c->L), phi_lo(c->L), phi_int(c->L);
        for (uint32_t i = 0; i < c->L; ++i) {
            hinv[i] = invm(bo_ctx::prod_mod(c->q, 0, c->L, i, c->q[i]), c->q[i]);
            // t / q_i = phi_int + (phi_hi, phi_lo) / 2^128 (t may exceed q_i)
            frac128(t % c->q[i], c->q[i], phi_hi[i], phi_lo[i]);
            phi_int[i] = t / c->q[i];
        }
        for (uint32_t k = 0; k < c->n; ++k) {
            uint64_t H = 0, Lo = 0;
            for (uint32_t i = 0; i < c->L; ++i) {
                const uint64_t y = mulm(x[i][k], hinv[i], c->q[i]);
                u128 pr = static_cast<u128>(y) * phi_hi[i];
                uint64_t ph = static_cast<uint64_t>(pr >> 64), pl = static_cast<uint64_t>(pr);
                const uint64_t add = mulhi(y, phi_lo[i]);
                pl += add;
                ph += (pl < add);
                Lo += pl;
                H += ph + (Lo < pl) + y * phi_int[i];
            }
            m[k] = (H + (Lo >> 63)) % t;
        }
    });
}

// c0 + c1 s per ciphertext prime (the decryption phase), coefficients
int bo_phase(bo_ctx* c, const uint64_t* ct, uint64_t* out) {
    return guarded([&] {
        for (uint32_t i = 0; i < c->L; ++i) {
            const uint64_t qi = c->q[i];
            Poly c0(ct + (size_t)i * c->n, ct + (size_t)(i + 1) * c->n);
            Poly c1(ct + (size_t)(c->L + i) * c->n, ct + (size_t)(c->L + i + 1) * c->n);
            Poly p = c->polymul(c->ntt_q[i], c1, c->reduce_signed(c->s, qi));
            for (uint32_t k = 0; k < c->n; ++k) out[(size_t)i * c->n + k] = addm(c0[k], p[k], qi);
        }
    });
}

int bo_add(bo_ctx* c, const uint64_t* a, const uint64_t* b, uint64_t* out) {
    return guarded([&] {
        for (uint32_t comp = 0; comp < 2; ++comp)
            for (uint32_t i = 0; i < c->L; ++i)
                for (uint32_t k = 0; k < c->n; ++k) {
                    const size_t o = ((size_t)comp * c->L + i) * c->n + k;
                    out[o] = addm(a[o], b[o], c->q[i]);
                }
    });
}

int bo_mul_scalar(bo_ctx* c, const uint64_t* a, int64_t s, uint64_t* out) {
    return guarded([&] {
        for (uint32_t comp = 0; comp < 2; ++comp)
            for (uint32_t i = 0; i < c->L; ++i) {
                const uint64_t sv = from_signed(s, c->q[i]);
                for (uint32_t k = 0; k < c->n; ++k) {
                    const size_t o = ((size_t)comp * c->L + i) * c->n + k;
                    out[o] = mulm(a[o], sv, c->q[i]);
                }
            }
    });
}

// §3.4: multiply by the centered lift of the encoded plaintext
int bo_mul_plain(bo_ctx* c, uint32_t tj, const uint64_t* ct, const uint64_t* slots, uint64_t* out) {
    return guarded([&] {
        const uint64_t t = c->t.at(tj);
        std::vector<uint64_t> m(c->n);
        if (bo_slot_encode(c, tj, slots, m.data())) throw std::runtime_error(g_err);
        std::vector<int64_t> mc(c->n);
        for (uint32_t k = 0; k < c->n; ++k)
            mc[k] = m[k] > t / 2 ? static_cast<int64_t>(m[k]) - static_cast<int64_t>(t) : static_cast<int64_t>(m[k]);
        for (uint32_t comp = 0; comp < 2; ++comp)
            for (uint32_t i = 0; i < c->L; ++i) {
                Poly a(ct + ((size_t)comp * c->L + i) * c->n, ct + ((size_t)comp * c->L + i + 1) * c->n);
                Poly r = c->polymul(c->ntt_q[i], a, c->reduce_signed(mc, c->q[i]));
                std::memcpy(out + ((size_t)comp * c->L + i) * c->n, r.data(), c->n * 8);
            }
    });
}

// §3.4: c0 += round(Q m / t) with m in [0, t)
int bo_add_plain(bo_ctx* c, uint32_t tj, const uint64_t* ct, const uint64_t* slots, uint64_t* out) {
    return guarded([&] {
        const uint64_t t = c->t.at(tj);
        std::vector<uint64_t> m(c->n);
        if (bo_slot_encode(c, tj, slots, m.data())) throw std::runtime_error(g_err);
        uint64_t q_mod_t = 1 % t;
        for (auto qi : c->q) q_mod_t = mulm(q_mod_t, qi % t, t);
        std::memcpy(out, ct, sizeof(uint64_t) * 2 * c->L * c->n);
        for (uint32_t i = 0; i < c->L; ++i) {
            const uint64_t qi = c->q[i];
            const uint64_t delta = mulm(subm(0, q_mod_t % qi, qi), invm(t, qi), qi);
            for (uint32_t k = 0; k < c->n; ++k) {
                const size_t o = (size_t)i * c->n + k;
                const uint64_t extra = (q_mod_t * m[k] + (t >> 1)) / t;
                out[o] = addm(out[o], addm(mulm(delta, m[k] % qi, qi), extra % qi, qi), qi);
            }
        }
    });
}

int bo_galois_key(bo_ctx* c, uint64_t g, uint64_t* key) {
    return guarded([&] {
        const uint32_t LK = c->L + c->K;
        auto sg = galois_signed(c->s, g, c->n);
        Rns target(LK);
        for (uint32_t r = 0; r < LK; ++r) target[r] = c->reduce_signed(sg, c->ntt_qp(r).p);
        auto k = make_key(*c, g, target);
        for (uint32_t j = 0; j < c->dnum; ++j)
            for (int h = 0; h < 2; ++h)
                for (uint32_t r = 0; r < LK; ++r)
                    std::memcpy(key + (((size_t)j * 2 + h) * LK + r) * c->n, k[j][h][r].data(), c->n * 8);
    });
}

int bo_rotate(bo_ctx* c, const uint64_t* ct, uint64_t g, uint64_t* out) {
    return guarded([&] {
        const uint32_t L = c->L, LK = L + c->K;
        auto sg = galois_signed(c->s, g, c->n);
        Rns target(LK);
        for (uint32_t r = 0; r < LK; ++r) target[r] = c->reduce_signed(sg, c->ntt_qp(r).p);
        auto key = make_key(*c, g, target);
        Rns c0 = unpack(*c, ct, L), c1 = unpack(*c, ct + (size_t)L * c->n, L);
        for (uint32_t i = 0; i < L; ++i) {
            c0[i] = galois(c0[i], g, c->q[i], c->n);
            c1[i] = galois(c1[i], g, c->q[i], c->n);
        }
        auto u = key_switch(*c, c1, key);
        for (uint32_t i = 0; i < L; ++i)
            for (uint32_t k = 0; k < c->n; ++k) c0[i][k] = addm(c0[i][k], u[0][i][k], c->q[i]);
        pack(*c, c0, out);
        pack(*c, u[1], out + (size_t)L * c->n);
    });
}

// CPU-baseline timing: `reps` rotations of one ciphertext by g with the key
// generated once (outside the timed region): automorphism + hybrid key
// switch + add, the same work as bo_rotate. seconds = total wall time.
int bo_time_rotate(bo_ctx* c, const uint64_t* ct, uint64_t g, uint32_t reps, uint64_t* out, double* seconds) {
    return guarded([&] {
        const uint32_t L = c->L, LK = L + c->K;
        auto sg = galois_signed(c->s, g, c->n);
        Rns target(LK);
        for (uint32_t r = 0; r < LK; ++r) target[r] = c->reduce_signed(sg, c->ntt_qp(r).p);
        auto key = make_key(*c, g, target);
        const auto t0 = std::chrono::steady_clock::now();
        for (uint32_t rep = 0; rep < reps; ++rep) {
            Rns c0 = unpack(*c, ct, L), c1 = unpack(*c, ct + (size_t)L * c->n, L);
            for (uint32_t i = 0; i < L; ++i) {
                c0[i] = galois(c0[i], g, c->q[i], c->n);
                c1[i] = galois(c1[i], g, c->q[i], c->n);
            }
            auto u = key_switch(*c, c1, key);
            for (uint32_t i = 0; i < L; ++i)
                for (uint32_t k = 0; k < c->n; ++k) c0[i][k] = addm(c0[i][k], u[0][i][k], c->q[i]);
            pack(*c, c0, out);
            pack(*c, u[1], out + (size_t)L * c->n);
        }
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
}

// §3.6 multiplication
int bo_mul(bo_ctx* c, uint32_t tj, const uint64_t* A, const uint64_t* B, uint64_t* out) {
    return guarded([&] {
        const uint32_t L = c->L, M = c->M;
        const uint64_t t = c->t.at(tj);
        std::vector<uint64_t> QB(c->q);
        QB.insert(QB.end(), c->b.begin(), c->b.end());
        // 1. extend the four input polys Q -> B, keep Q residues
        Rns x[4];
        const uint64_t* src[4] = {A, A + (size_t)L * c->n, B, B + (size_t)L * c->n};
        for (int p = 0; p < 4; ++p) {
            Rns rq = unpack(*c, src[p], L);
            Rns rb = exact_extend(*c, rq, c->q, c->b);
            x[p] = rq;
            x[p].insert(x[p].end(), rb.begin(), rb.end());
        }
        // 2. tensor over Q ∪ B
        Rns d[3];
        for (int h = 0; h < 3; ++h) d[h].resize(L + M);
        for (uint32_t r = 0; r < L + M; ++r) {
            const Ntt& T_ = r < L ? c->ntt_q[r] : c->ntt_b[r - L];
            const uint64_t pr = T_.p;
            d[0][r] = c->polymul(T_, x[0][r], x[2][r]);
            d[2][r] = c->polymul(T_, x[1][r], x[3][r]);
            Poly u = c->polymul(T_, x[0][r], x[3][r]), v = c->polymul(T_, x[1][r], x[2][r]);
            d[1][r].resize(c->n);
            for (uint32_t k = 0; k < c->n; ++k) d[1][r][k] = addm(u[k], v[k], pr);
        }
        // 3. scale by t/Q into B (rational constants per q_i)
        uint64_t Bmod;
        std::vector<uint64_t> th_hi(L), th_lo(L);
        std::vector<std::vector<uint64_t>> Wmod(L, std::vector<uint64_t>(M));
        for (uint32_t i = 0; i < L; ++i) {
            const uint64_t qi = c->q[i];
            Bmod = bo_ctx::prod_mod(c->b, 0, M, SIZE_MAX, qi);
            const uint64_t qhat = bo_ctx::prod_mod(c->q, 0, L, i, qi);
            const uint64_t ci = invm(mulm(qhat, Bmod, qi), qi);             // [(QB/q_i)^-1]_{q_i}
            const uint64_t rem = mulm(mulm(t % qi, ci, qi), Bmod, qi);        // [t c_i B]_{q_i}
            frac128(rem, qi, th_hi[i], th_lo[i]);
            for (uint32_t m = 0; m < M; ++m) {
                const uint64_t bm = c->b[m];
                Wmod[i][m] = mulm(subm(0, rem % bm, bm), invm(qi % bm, bm), bm);  // (t c_i B - rem)/q_i mod b_m
            }
        }
        std::vector<uint64_t> tQinv(M);
        for (uint32_t m = 0; m < M; ++m) {
            const uint64_t bm = c->b[m];
            tQinv[m] = mulm(t % bm, invm(bo_ctx::prod_mod(c->q, 0, L, SIZE_MAX, bm), bm), bm);
        }
        Rns e[3];
        for (int h = 0; h < 3; ++h) {
            Rns z(M, Poly(c->n));
            for (uint32_t k = 0; k < c->n; ++k) {
                uint64_t H = 0, Lo = 0;
                for (uint32_t i = 0; i < L; ++i) {
                    const uint64_t Di = d[h][i][k];
                    u128 pr = static_cast<u128>(Di) * th_hi[i];
                    uint64_t ph = static_cast<uint64_t>(pr >> 64), pl = static_cast<uint64_t>(pr);
                    const uint64_t add = mulhi(Di, th_lo[i]);
                    pl += add;
                    ph += (pl < add);
                    Lo += pl;
                    H += ph + (Lo < pl);
                }
                const uint64_t R = H + (Lo >> 63);
                for (uint32_t m = 0; m < M; ++m) {
                    const uint64_t bm = c->b[m];
                    uint64_t acc = 0;
                    for (uint32_t i = 0; i < L; ++i) acc = addm(acc, mulm(d[h][i][k] % bm, Wmod[i][m], bm), bm);
                    acc = addm(acc, R % bm, bm);
                    acc = addm(acc, mulm(d[h][L + m][k], tQinv[m], bm), bm);
                    z[m][k] = acc;
                }
            }
            // 4. exact B -> Q
            e[h] = exact_extend(*c, z, c->b, c->q);
        }
        // 5. relinearize e2 with the key for s^2
        const uint32_t LK = L + c->K;
        Rns s2(LK);
        for (uint32_t r = 0; r < LK; ++r) {
            const Ntt& T_ = c->ntt_qp(r);
            Poly sr = c->reduce_signed(c->s, T_.p);
            s2[r] = c->polymul(T_, sr, sr);
        }
        auto key = make_key(*c, 0, s2);
        auto u = key_switch(*c, e[2], key);
        for (uint32_t i = 0; i < L; ++i)
            for (uint32_t k = 0; k < c->n; ++k) {
                e[0][i][k] = addm(e[0][i][k], u[0][i][k], c->q[i]);
                e[1][i][k] = addm(e[1][i][k], u[1][i][k], c->q[i]);
            }
        pack(*c, e[0], out);
        pack(*c, e[1], out + (size_t)L * c->n);
    });
}

}  // extern "C"
