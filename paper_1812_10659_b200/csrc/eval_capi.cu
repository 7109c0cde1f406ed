// extern "C" evaluator boundary (include/lola_b200.h, §Evaluator): one entry
// point per method of the reference's Evaluator
// (proj/include/packnn/evaluator.hpp:50-91), messages as opaque handles.
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/lola_b200.h"
#include "capi_internal.hpp"
#include "lola_eval.hpp"

struct lb_evaluator {
    std::shared_ptr<lb::lola::EvalContext> ecx;
    std::unique_ptr<lb::lola::Evaluator> ev;
};

struct lb_message {
    lb::lola::Message m;
};

namespace {

using lb::capi::guarded;
using lb::capi::need;

lb_message* wrap(lb::lola::Message m) { return new lb_message{std::move(m)}; }

std::vector<int64_t> vec(const int64_t* v, uint64_t count) { return std::vector<int64_t>(v, v + (v ? count : 0)); }

}  // namespace

extern "C" {

int lb_eval_create(lb_context* cx, uint32_t batch, uint32_t max_depth, void* stream, lb_evaluator** out) {
    return guarded([&] {
        need(cx && out, "null argument");
        cx->cx.activate();
        auto e = std::make_unique<lb_evaluator>();
        e->ecx = std::make_shared<lb::lola::EvalContext>(cx->cx, batch, max_depth, static_cast<cudaStream_t>(stream));
        e->ev = std::make_unique<lb::lola::Evaluator>(*e->ecx);
        *out = e.release();
    });
}

int lb_eval_destroy(lb_evaluator* e) {
    return guarded([&] { delete e; });
}

int lb_eval_fork(const lb_evaluator* e, lb_evaluator** out) {
    return guarded([&] {
        need(e && out, "null argument");
        auto f = std::make_unique<lb_evaluator>();
        f->ecx = e->ecx;
        f->ev = std::make_unique<lb::lola::Evaluator>(e->ev->fork());
        *out = f.release();
    });
}

int lb_eval_absorb(lb_evaluator* e, const lb_evaluator* child) {
    return guarded([&] {
        need(e && child, "null argument");
        e->ev->absorb(*child->ev);
    });
}

int lb_eval_counters(const lb_evaluator* e, uint64_t* out) {
    return guarded([&] {
        need(e && out, "null argument");
        const auto v = e->ev->counters().ops.values();
        std::memcpy(out, v.data(), 7 * 8);
        out[7] = e->ev->counters().live_messages_peak;
    });
}

int lb_eval_note_live(lb_evaluator* e, uint64_t live) {
    return guarded([&] { e->ev->note_live(live); });
}

int lb_eval_lift(lb_evaluator* e, const int64_t* values, uint64_t count, int per_message, lb_message** out) {
    return guarded([&] {
        need(e && out && (values || count == 0), "null argument");
        const uint32_t B = e->ecx->batch();
        if (!per_message) {
            *out = wrap(e->ev->lift(vec(values, count)));
            return;
        }
        std::vector<std::vector<int64_t>> rows(B);
        for (uint32_t b = 0; b < B; ++b) rows[b] = vec(values + uint64_t(b) * count, count);
        *out = wrap(e->ev->lift_batch(rows));
    });
}

int lb_eval_lower(lb_evaluator* e, const lb_message* m, uint64_t* out) {
    return guarded([&] {
        need(e && m && out, "null argument");
        lb::DeviceBuffer d = e->ev->lower(m->m);
        LB_CUDA(cudaMemcpyAsync(out, d.get(), d.bytes(), cudaMemcpyDeviceToHost, e->ecx->stream()));
        LB_CUDA(cudaStreamSynchronize(e->ecx->stream()));
    });
}

int lb_eval_add(lb_evaluator* e, const lb_message* a, const lb_message* b, lb_message** out) {
    return guarded([&] { *out = wrap(e->ev->add(a->m, b->m)); });
}

int lb_eval_add_plain(lb_evaluator* e, const lb_message* a, const int64_t* values, uint64_t count, lb_message** out) {
    return guarded([&] { *out = wrap(e->ev->add_plain(a->m, vec(values, count))); });
}

int lb_eval_mul(lb_evaluator* e, const lb_message* a, const lb_message* b, lb_message** out) {
    return guarded([&] { *out = wrap(e->ev->mul(a->m, b->m)); });
}

int lb_eval_mul_plain(lb_evaluator* e, const lb_message* a, const int64_t* values, uint64_t count, lb_message** out) {
    return guarded([&] { *out = wrap(e->ev->mul_plain(a->m, vec(values, count))); });
}

int lb_eval_mask(lb_evaluator* e, const lb_message* a, const uint8_t* bits, uint64_t count, lb_message** out) {
    return guarded([&] { *out = wrap(e->ev->mask(a->m, std::vector<uint8_t>(bits, bits + (bits ? count : 0)))); });
}

int lb_eval_mul_scalar(lb_evaluator* e, const lb_message* a, int64_t s, lb_message** out) {
    return guarded([&] { *out = wrap(e->ev->mul_scalar(a->m, s)); });
}

int lb_eval_rotate_columns(lb_evaluator* e, const lb_message* a, int64_t k, lb_message** out) {
    return guarded([&] { *out = wrap(e->ev->rotate_columns(a->m, k)); });
}

int lb_eval_rotate_rows(lb_evaluator* e, const lb_message* a, lb_message** out) {
    return guarded([&] { *out = wrap(e->ev->rotate_rows(a->m)); });
}

int lb_eval_rotate_bundle(lb_evaluator* e, const lb_message* a, uint32_t amount, lb_message** out) {
    return guarded([&] { *out = wrap(e->ev->rotate_bundle(a->m, amount)); });
}

int lb_message_free(lb_message* m) {
    return guarded([&] { delete m; });
}

int lb_message_info(const lb_message* m, uint32_t* depth, uint32_t* plain_depth, char* magnitude, uint64_t cap) {
    return guarded([&] {
        need(m != nullptr, "null message");
        if (depth) *depth = m->m.depth;
        if (plain_depth) *plain_depth = m->m.plain_depth;
        if (magnitude) {
            const std::string s = m->m.magnitude.str();
            need(s.size() + 1 <= cap, "magnitude buffer too small");
            std::memcpy(magnitude, s.c_str(), s.size() + 1);
        }
    });
}

// device pointer of the message's ciphertexts [batch][T][2][L][n] (tests)
int lb_message_data(const lb_message* m, const void** out) {
    return guarded([&] {
        need(m && out, "null argument");
        *out = m->m.data();
    });
}

}  // extern "C"
