// extern "C" entry points (include/lola_b200.h). Translates exceptions into
// the status codes the header documents.
#include <cstring>
#include <new>
#include <string>

#include "../../include/lola_b200.h"
#include "bfv.hpp"
#include "capi_internal.hpp"
#include "context.hpp"
#include "host_math.hpp"

namespace lb::capi {
std::string& last_error() {
    static thread_local std::string err;
    return err;
}
}  // namespace lb::capi

namespace {

using lb::capi::guarded;
using lb::capi::need;

// NULL selects the legacy default stream, as everywhere in CUDA.
cudaStream_t pick(lb_context*, void* s) { return static_cast<cudaStream_t>(s); }

}  // namespace

extern "C" {

const char* lb_last_error(void) { return lb::capi::last_error().c_str(); }

int lb_find_primes(uint32_t bits, uint32_t log_mod, uint32_t count, const uint64_t* exclude,
                   uint32_t num_exclude, uint64_t* out) {
    return guarded([&] {
        need(out != nullptr, "null output");
        std::vector<uint64_t> ex(exclude, exclude + (exclude ? num_exclude : 0));
        auto v = lb::host::find_primes(static_cast<int>(bits), static_cast<int>(log_mod), count, ex);
        std::memcpy(out, v.data(), v.size() * sizeof(uint64_t));
    });
}

int lb_context_create(const lb_params* prm, lb_context** out) {
    return guarded([&] {
        need(prm && out, "null argument");
        lb::Params p;
        p.n = prm->n;
        p.q.assign(prm->q, prm->q + prm->num_q);
        if (prm->num_p) p.p.assign(prm->p, prm->p + prm->num_p);
        if (prm->num_b) p.b.assign(prm->b, prm->b + prm->num_b);
        if (prm->num_t) p.t.assign(prm->t, prm->t + prm->num_t);
        p.dnum = prm->dnum;
        p.seed = prm->seed;
        p.device = prm->device;
        *out = new lb_context(p);
    });
}

int lb_context_destroy(lb_context* cx) {
    return guarded([&] { delete cx; });
}

int lb_context_prime(const lb_context* cx, uint32_t index, uint64_t* prime, uint64_t* psi) {
    return guarded([&] {
        need(cx != nullptr, "null context");
        if (prime) *prime = cx->cx.prime(index);
        if (psi) *psi = cx->cx.psi(index);
    });
}

int lb_context_residue_bytes(const lb_context* cx, uint32_t* bytes) {
    return guarded([&] {
        need(cx && bytes, "null argument");
        *bytes = static_cast<uint32_t>(lb::residue_bytes(cx->cx.bfv()->dev));
    });
}

int lb_pool_reserve(lb_context* cx, uint64_t bytes) {
    return guarded([&] {
        need(cx != nullptr, "null context");
        cx->cx.activate();
        // grow the device's stream-ordered pool once (its release threshold
        // keeps freed memory): later allocations of the working set never map
        // fresh physical memory inside a timed region
        cudaStream_t s = cx->cx.stream();
        void* p = nullptr;
        LB_CUDA(cudaMallocAsync(&p, bytes, s));
        LB_CUDA(cudaFreeAsync(p, s));
        LB_CUDA(cudaStreamSynchronize(s));
    });
}

int lb_sync(lb_context* cx, void* stream) {
    return guarded([&] { LB_CUDA(cudaStreamSynchronize(pick(cx, stream))); });
}

int lb_ntt_forward(lb_context* cx, uint64_t* data, uint32_t polys, uint32_t limbs, uint32_t first_prime,
                   uint64_t poly_stride, void* stream) {
    return guarded([&] {
        if (cx) cx->cx.activate();
        need(cx && data, "null argument");
        cx->cx.ntt_forward(lb::LimbBatch{data, polys, limbs, first_prime, poly_stride}, pick(cx, stream));
    });
}

int lb_ntt_inverse(lb_context* cx, uint64_t* data, uint32_t polys, uint32_t limbs, uint32_t first_prime,
                   uint64_t poly_stride, void* stream) {
    return guarded([&] {
        if (cx) cx->cx.activate();
        need(cx && data, "null argument");
        cx->cx.ntt_inverse(lb::LimbBatch{data, polys, limbs, first_prime, poly_stride}, pick(cx, stream));
    });
}

int lb_ntt_forward_u32(lb_context* cx, uint32_t* data, uint32_t polys, uint32_t limbs, uint32_t first_prime,
                       uint64_t poly_stride, void* stream) {
    return guarded([&] {
        if (cx) cx->cx.activate();
        need(cx && data, "null argument");
        lb::LimbBatch b{reinterpret_cast<uint64_t*>(data), polys, limbs, first_prime, poly_stride};
        b.packed32 = true;
        cx->cx.ntt_forward(b, pick(cx, stream));
    });
}

int lb_ntt_inverse_u32(lb_context* cx, uint32_t* data, uint32_t polys, uint32_t limbs, uint32_t first_prime,
                       uint64_t poly_stride, void* stream) {
    return guarded([&] {
        if (cx) cx->cx.activate();
        need(cx && data, "null argument");
        lb::LimbBatch b{reinterpret_cast<uint64_t*>(data), polys, limbs, first_prime, poly_stride};
        b.packed32 = true;
        cx->cx.ntt_inverse(b, pick(cx, stream));
    });
}

int lb_encrypt_slots(lb_context* cx, const int64_t* values, uint32_t B, uint64_t id_base, void* out, void* stream) {
    return guarded([&] {
        if (cx) cx->cx.activate();
        need(cx && values && out, "null argument");
        if (id_base == UINT64_MAX) id_base = cx->cx.reserve_ciphertext_ids(uint64_t(B) * cx->cx.T());
        lb::encrypt_slots(cx->cx, values, B, id_base, out, pick(cx, stream));
    });
}

int lb_decrypt_slots(lb_context* cx, const void* ct, uint32_t B, uint64_t* out, void* stream) {
    return guarded([&] {
        if (cx) cx->cx.activate();
        need(cx && ct && out, "null argument");
        lb::decrypt_slots(cx->cx, ct, B, out, pick(cx, stream));
    });
}

int lb_decrypt_coeffs(lb_context* cx, const void* ct, uint32_t B, uint64_t* out, void* stream) {
    return guarded([&] {
        if (cx) cx->cx.activate();
        need(cx && ct && out, "null argument");
        lb::decrypt_coeffs(cx->cx, ct, B, out, pick(cx, stream));
    });
}

int lb_encode_plain(lb_context* cx, const int64_t* values, void* pt_mul, void* pt_add, void* stream) {
    return guarded([&] {
        if (cx) cx->cx.activate();
        need(cx && values && (pt_mul || pt_add), "null argument");
        lb::encode_plain(cx->cx, values, pt_mul, pt_add, pick(cx, stream));
    });
}

int lb_ct_add(lb_context* cx, const void* a, const void* b, void* out, uint32_t count, void* stream) {
    return guarded([&] {
        if (cx) cx->cx.activate();
        need(cx && a && b && out, "null argument");
        lb::ct_add(cx->cx, a, b, out, count, pick(cx, stream));
    });
}

int lb_ct_mul_scalar(lb_context* cx, const void* a, int64_t scalar, void* out, uint32_t count, void* stream) {
    return guarded([&] {
        if (cx) cx->cx.activate();
        need(cx && a && out, "null argument");
        lb::ct_mul_scalar(cx->cx, a, scalar, out, count, pick(cx, stream));
    });
}

int lb_ct_mul_plain(lb_context* cx, const void* a, const void* pt, void* out, uint32_t count, void* stream) {
    return guarded([&] {
        if (cx) cx->cx.activate();
        need(cx && a && pt && out, "null argument");
        lb::ct_mul_plain(cx->cx, a, pt, out, count, pick(cx, stream));
    });
}

int lb_ct_add_plain(lb_context* cx, const void* a, const void* pt, void* out, uint32_t count, void* stream) {
    return guarded([&] {
        if (cx) cx->cx.activate();
        need(cx && a && pt && out, "null argument");
        lb::ct_add_plain(cx->cx, a, pt, out, count, pick(cx, stream));
    });
}

int lb_ct_rotate(lb_context* cx, const void* a, uint64_t galois, void* out, uint32_t count, void* stream) {
    return guarded([&] {
        if (cx) cx->cx.activate();
        need(cx && a && out, "null argument");
        lb::ct_rotate(cx->cx, a, galois, out, count, pick(cx, stream));
    });
}

int lb_ct_mul(lb_context* cx, const void* a, const void* b, void* out, uint32_t count, void* stream) {
    return guarded([&] {
        if (cx) cx->cx.activate();
        need(cx && a && b && out, "null argument");
        lb::ct_mul(cx->cx, a, b, out, count, pick(cx, stream));
    });
}

int lb_keygen(lb_context* cx, uint64_t key_id, void* stream) {
    return guarded([&] {
        if (cx) cx->cx.activate();
        need(cx != nullptr, "null context");
        lb::ensure_key(cx->cx, key_id, pick(cx, stream));
    });
}

int lb_key_pointer(lb_context* cx, uint64_t key_id, const uint64_t** out) {
    return guarded([&] {
        if (cx) cx->cx.activate();
        need(cx && out, "null argument");
        *out = lb::key_ptr(cx->cx, key_id);
    });
}

int lb_automorphism(lb_context* cx, const void* in, void* out, uint32_t polys, uint32_t limbs, uint64_t galois,
                    void* stream) {
    return guarded([&] {
        if (cx) cx->cx.activate();
        need(cx && in && out, "null argument");
        need(limbs <= cx->cx.prime_count(), "too many limbs");
        lb::automorphism_ntt(cx->cx, in, out, polys, limbs, galois, pick(cx, stream));
    });
}

int lb_key_switch(lb_context* cx, const void* d, uint64_t key_id, void* u0, void* u1, uint32_t count, void* stream) {
    return guarded([&] {
        if (cx) cx->cx.activate();
        need(cx && d && u0 && u1, "null argument");
        lb::key_switch(cx->cx, d, key_id, u0, u1, count, pick(cx, stream));
    });
}

uint64_t lb_galois_exponent_columns(uint32_t n, uint32_t k) {
    // right shift by k = automorphism by 3^(n/2 - k) mod 2n (ring.cpp:173-182)
    const uint32_t half = n / 2;
    if (n < 4 || k >= half) return 0;
    const uint64_t two_n = 2ull * n;
    uint64_t e = 1, base = 3;
    for (uint64_t x = (half - k) % half; x; x >>= 1) {
        if (x & 1) e = e * base % two_n;
        base = base * base % two_n;
    }
    return e;
}

uint64_t lb_galois_exponent_rows(uint32_t n) { return 2ull * n - 1; }

}  // extern "C"
