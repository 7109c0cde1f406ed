// Drop-in proof (test infrastructure): the reference's OWN Evaluator
// interface — proj/include/packnn/evaluator.hpp and message.hpp, UNMODIFIED —
// implemented over this repo's C-ABI (include/lola_b200.h, §Evaluator).
//
// oracle/Makefile links this file in place of the reference's
// proj/src/evaluator.cpp, together with the reference's unmodified
// modular.cpp, ring.cpp, representation.cpp, kernels.cpp, layers.cpp and
// plan.cpp (+ oracle/ref_shim.cpp), into oracle/_ref/libpackb200.so. The
// reference's own plan builders, kernels and execute() (plan.cpp:597-633)
// then drive real BFV ciphertexts on the B200: a third BackendKind, value
// B200 = 2 (evaluator.hpp:12 declares Slot and Ring; the enum is not edited,
// the new value is selected numerically, as a binding would).
//
// Mapping (evaluator.hpp:50-91 -> lb_eval_*):
//   * a Message's payload holds the lb_message handle (MessagePayload::limbs
//     is a per-backend opaque array, message.hpp:62-68; here one word), freed
//     with the payload;
//   * depth, plain depth and the magnitude bound are read back from the
//     device evaluator (lb_message_info), which applies the reference's rules;
//   * counters: the device evaluator counts with the reference's rules
//     (popcount for column rotations, ...); each call adds the delta it
//     produced to this Evaluator's OpCounters, so fork()/absorb() (inline in
//     the header) keep the reference's accounting. The device evaluator is
//     shared per EvalContext: callers run one op at a time (kernel threads 1);
//   * budget errors come back as status 4 and are rethrown as the reference's
//     depth_error / magnitude_error; bad arguments as std::invalid_argument.
//
// Ciphertext parameters (Q, P, auxiliary base, dnum, seed) have no place in
// the reference's EvalContext signature; pb2_set_params() supplies them
// before the context is built (the plaintext primes are the context's).
#include <bit>
#include <cstring>
#include <map>
#include <mutex>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "lola_b200.h"
#include "packnn/evaluator.hpp"

namespace packnn {
namespace {

constexpr BackendKind kB200 = static_cast<BackendKind>(2);

struct DeviceParams {
    std::vector<uint64_t> q, p, b;
    uint32_t dnum = 0;
    uint64_t seed = 1;
};
DeviceParams g_params;

struct Backend {
    lb_context* cx = nullptr;
    lb_evaluator* ev = nullptr;
};
std::mutex g_mu;
std::map<const EvalContext*, Backend> g_backends;

[[noreturn]] void raise(int status) {
    const std::string msg = lb_last_error();
    if (status == 4) {
        if (msg.find("depth") != std::string::npos) throw depth_error(msg);
        throw magnitude_error(msg);
    }
    if (status == 3) throw std::invalid_argument(msg);
    if (status == 5) throw std::logic_error(msg);
    throw std::runtime_error("lola_b200: " + msg);
}
void ok(int status) {
    if (status) raise(status);
}

// Ciphertext parameters when the caller (e.g. the CLI) set none: the
// repo's parameter sets by degree (paper_1812_10659_b200/params.py) —
// n >= 16384: 29-bit L=10, K=5, dnum=2 (lola-mnist); n = 8192: 30-bit L=5,
// K=2, dnum=3 (lola-small); smaller: 60-bit L=7, K=1, one prime per digit —
// with the auxiliary base of the exact tensor product next in the chain.
void default_params(uint32_t n) {
    uint32_t bits = 60, L = 7, K = 1, dnum = 7;
    if (n >= 16384) bits = 29, L = 10, K = 5, dnum = 2;
    else if (n == 8192) bits = 30, L = 5, K = 2, dnum = 3;
    const uint32_t M = L + (bits >= 59 ? 1 : 2);
    std::vector<uint64_t> all(L + K + M);
    ok(lb_find_primes(bits, 16, L + K + M, nullptr, 0, all.data()));
    g_params.q.assign(all.begin(), all.begin() + L);
    g_params.p.assign(all.begin() + L, all.begin() + L + K);
    g_params.b.assign(all.begin() + L + K, all.end());
    g_params.dnum = dnum;
    std::random_device rd;
    g_params.seed = ((uint64_t(rd()) << 32) | rd()) | 1;
}

Backend& backend(const EvalContext* cx) {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_backends.find(cx);
    if (it == g_backends.end()) throw std::logic_error("EvalContext has no B200 backend");
    return it->second;
}

lb_message* handle(const Message& m) {
    return reinterpret_cast<lb_message*>(static_cast<uintptr_t>(m.payload->limbs.at(0).at(0)));
}

CounterDelta device_counters(lb_evaluator* ev) {
    uint64_t c[8];
    ok(lb_eval_counters(ev, c));
    CounterDelta d;
    d.ct_ct_mul = c[0];
    d.ct_plain_mul = c[1];
    d.scalar_mul = c[2];
    d.mask_mul = c[3];
    d.add = c[4];
    d.rot_cols = c[5];
    d.rot_rows = c[6];
    return d;
}

CounterDelta minus(const CounterDelta& a, const CounterDelta& b) {
    CounterDelta d;
    d.ct_ct_mul = a.ct_ct_mul - b.ct_ct_mul;
    d.ct_plain_mul = a.ct_plain_mul - b.ct_plain_mul;
    d.scalar_mul = a.scalar_mul - b.scalar_mul;
    d.mask_mul = a.mask_mul - b.mask_mul;
    d.add = a.add - b.add;
    d.rot_cols = a.rot_cols - b.rot_cols;
    d.rot_rows = a.rot_rows - b.rot_rows;
    return d;
}

// Wrap a device message: the payload owns the handle.
Message wrap(lb_message* h) {
    Message m;
    auto* pl = new MessagePayload{{{static_cast<uint64_t>(reinterpret_cast<uintptr_t>(h))}}};
    m.payload = std::shared_ptr<const MessagePayload>(pl, [](const MessagePayload* p) {
        lb_message_free(reinterpret_cast<lb_message*>(static_cast<uintptr_t>(p->limbs[0][0])));
        delete p;
    });
    uint32_t depth = 0, plain_depth = 0;
    char mag[256];
    ok(lb_message_info(h, &depth, &plain_depth, mag, sizeof mag));
    m.depth = depth;
    m.plain_depth = plain_depth;
    m.magnitude = BigInt(mag);
    return m;
}

// One counted device op: run it, add the counter delta to `counters`.
template <class F>
Message counted(const EvalContext* cx, OpCounters& counters, F&& op) {
    Backend& be = backend(cx);
    const CounterDelta before = device_counters(be.ev);
    lb_message* out = nullptr;
    ok(op(be.ev, &out));
    counters.ops += minus(device_counters(be.ev), before);
    return wrap(out);
}

}  // namespace

std::string CounterDelta::brief() const {
    std::ostringstream os;
    const std::pair<const char*, uint64_t> parts[] = {{"mul", ct_ct_mul}, {"pmul", ct_plain_mul},
                                                       {"smul", scalar_mul}, {"mask", mask_mul},
                                                       {"add", add},        {"rotc", rot_cols},
                                                       {"rotr", rot_rows}};
    const char* sep = "";
    for (const auto& [k, v] : parts)
        if (v) {
            os << sep << k << ':' << v;
            sep = " ";
        }
    const std::string s = os.str();
    return s.empty() ? "-" : s;
}

const char* backend_name(BackendKind k) {
    if (k == kB200) return "b200";
    return k == BackendKind::Slot ? "slot" : "ring";
}

BackendKind backend_from_name(const std::string& s) {
    if (s == "b200" || s == "gpu") return kB200;
    throw std::invalid_argument("this build carries only the b200 backend: " + s);
}

EvalContext::EvalContext(BackendKind kind, uint32_t n, const std::vector<uint64_t>& primes, uint32_t max_depth,
                         bool corrupt_rotation)
    : kind_(kind),
      n_(n),
      modulus_(CrtModulus::create(primes, n)),
      capacity_(modulus_.capacity()),
      max_depth_(max_depth),
      corrupt_rotation_(corrupt_rotation) {
    if (kind != kB200) throw std::invalid_argument("this build carries only the b200 backend");
    if (corrupt_rotation) throw std::invalid_argument("the b200 backend has no corrupt_rotation hook");
    if (g_params.q.empty()) default_params(n);
    lb_params prm{};
    prm.n = n;
    prm.num_q = static_cast<uint32_t>(g_params.q.size());
    prm.num_p = static_cast<uint32_t>(g_params.p.size());
    prm.num_b = static_cast<uint32_t>(g_params.b.size());
    prm.num_t = static_cast<uint32_t>(primes.size());
    prm.q = g_params.q.data();
    prm.p = g_params.p.data();
    prm.b = g_params.b.data();
    prm.t = primes.data();
    prm.dnum = g_params.dnum;
    prm.seed = g_params.seed;
    prm.device = 0;
    Backend be;
    ok(lb_context_create(&prm, &be.cx));
    ok(lb_eval_create(be.cx, 1, max_depth, nullptr, &be.ev));
    std::lock_guard<std::mutex> lk(g_mu);
    g_backends[this] = be;
}

void Evaluator::check_magnitude(const BigInt& magnitude, const char* op) const {
    if (magnitude > cx_->capacity()) throw magnitude_error(std::string(op) + ": magnitude bound exceeds capacity");
}

Message Evaluator::lift_big(std::span<const BigInt> values) const {
    std::vector<int64_t> v(values.size());
    for (size_t i = 0; i < values.size(); ++i) {
        if (values[i] > BigInt(INT64_MAX) || values[i] < BigInt(INT64_MIN))
            throw std::invalid_argument("lift: value beyond int64 (b200 backend)");
        v[i] = static_cast<int64_t>(values[i]);
    }
    return lift(v);
}

Message Evaluator::lift(std::span<const int64_t> values) const {
    Backend& be = backend(cx_);
    lb_message* out = nullptr;
    ok(lb_eval_lift(be.ev, values.data(), values.size(), 0, &out));
    return wrap(out);
}

std::vector<BigInt> Evaluator::lower(const Message& m) const {
    Backend& be = backend(cx_);
    const uint32_t n = cx_->n();
    std::vector<uint64_t> words(size_t(n) * 4);
    ok(lb_eval_lower(be.ev, handle(m), words.data()));
    std::vector<BigInt> out(n);
    const BigInt two256 = BigInt(1) << 256;
    for (uint32_t i = 0; i < n; ++i) {
        BigInt v = 0;
        for (int w = 3; w >= 0; --w) v = (v << 64) | BigInt(words[size_t(i) * 4 + w]);
        if (words[size_t(i) * 4 + 3] >> 63) v = v - two256;  // two's complement
        out[i] = v;
    }
    return out;
}

Message Evaluator::add(const Message& a, const Message& b) {
    return counted(cx_, counters_, [&](lb_evaluator* ev, lb_message** o) { return lb_eval_add(ev, handle(a), handle(b), o); });
}

Message Evaluator::add_plain(const Message& a, std::span<const int64_t> values) {
    return counted(cx_, counters_, [&](lb_evaluator* ev, lb_message** o) {
        return lb_eval_add_plain(ev, handle(a), values.data(), values.size(), o);
    });
}

Message Evaluator::mul(const Message& a, const Message& b) {
    return counted(cx_, counters_, [&](lb_evaluator* ev, lb_message** o) { return lb_eval_mul(ev, handle(a), handle(b), o); });
}

Message Evaluator::mul_plain(const Message& a, std::span<const int64_t> values) {
    return counted(cx_, counters_, [&](lb_evaluator* ev, lb_message** o) {
        return lb_eval_mul_plain(ev, handle(a), values.data(), values.size(), o);
    });
}

Message Evaluator::mask(const Message& a, std::span<const uint8_t> bits) {
    return counted(cx_, counters_, [&](lb_evaluator* ev, lb_message** o) {
        return lb_eval_mask(ev, handle(a), bits.data(), bits.size(), o);
    });
}

Message Evaluator::mul_scalar(const Message& a, int64_t s) {
    return counted(cx_, counters_, [&](lb_evaluator* ev, lb_message** o) { return lb_eval_mul_scalar(ev, handle(a), s, o); });
}

Message Evaluator::rotate_columns(const Message& a, int64_t k) {
    return counted(cx_, counters_,
                   [&](lb_evaluator* ev, lb_message** o) { return lb_eval_rotate_columns(ev, handle(a), k, o); });
}

Message Evaluator::rotate_rows(const Message& a) {
    return counted(cx_, counters_, [&](lb_evaluator* ev, lb_message** o) { return lb_eval_rotate_rows(ev, handle(a), o); });
}

Message Evaluator::rotate_bundle(const Message& a, uint32_t amount) {
    return counted(cx_, counters_,
                   [&](lb_evaluator* ev, lb_message** o) { return lb_eval_rotate_bundle(ev, handle(a), amount, o); });
}

void Evaluator::absorb(const Evaluator& child) {
    counters_.ops += child.counters_.ops;
    counters_.note_live(child.counters_.live_messages_peak);
}

}  // namespace packnn

extern "C" {

// Ciphertext parameters for the next EvalContext(BackendKind(2), n, t...).
int pb2_set_params(const uint64_t* q, uint32_t L, const uint64_t* p, uint32_t K, const uint64_t* b, uint32_t M,
                   uint32_t dnum, uint64_t seed) {
    packnn::g_params.q.assign(q, q + L);
    packnn::g_params.p.assign(p, p + K);
    packnn::g_params.b.assign(b, b + M);
    packnn::g_params.dnum = dnum;
    packnn::g_params.seed = seed;
    return 0;
}

int pb2_available(void) { return 1; }

}  // extern "C"
