// extern "C" entry points (include/lola_b200.h). Translates exceptions into
// the status codes the header documents.
#include <cstring>
#include <new>
#include <string>

#include "../../include/lola_b200.h"
#include "bfv.hpp"
#include "context.hpp"
#include "host_math.hpp"

struct lb_context {
    lb::Context cx;
    explicit lb_context(const lb::Params& p) : cx(p) {}
};

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 3;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return 3;
    } catch (const std::bad_alloc&) {
        g_err = "out of memory";
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// NULL selects the legacy default stream, as everywhere in CUDA.
cudaStream_t pick(lb_context*, void* s) { return static_cast<cudaStream_t>(s); }

void need(bool ok, const char* what) {
    if (!ok) throw std::invalid_argument(what);
}

}  // namespace

extern "C" {

const char* lb_last_error(void) { return g_err.c_str(); }

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
        if (prm->num_t) p.t.assign(prm->t, prm->t + prm->num_t);
        p.dnum = prm->dnum;
        p.seed = prm->seed;
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

int lb_sync(lb_context* cx, void* stream) {
    return guarded([&] { LB_CUDA(cudaStreamSynchronize(pick(cx, stream))); });
}

int lb_ntt_forward(lb_context* cx, uint64_t* data, uint32_t polys, uint32_t limbs, uint32_t first_prime,
                   uint64_t poly_stride, void* stream) {
    return guarded([&] {
        need(cx && data, "null argument");
        cx->cx.ntt_forward(lb::LimbBatch{data, polys, limbs, first_prime, poly_stride}, pick(cx, stream));
    });
}

int lb_ntt_inverse(lb_context* cx, uint64_t* data, uint32_t polys, uint32_t limbs, uint32_t first_prime,
                   uint64_t poly_stride, void* stream) {
    return guarded([&] {
        need(cx && data, "null argument");
        cx->cx.ntt_inverse(lb::LimbBatch{data, polys, limbs, first_prime, poly_stride}, pick(cx, stream));
    });
}

}  // extern "C"
