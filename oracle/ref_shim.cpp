// C-ABI shim over the UNMODIFIED reference (packnn, /root/reference/proj).
//
// TEST INFRASTRUCTURE ONLY — the checker, never the product. oracle/Makefile
// compiles this file together with the reference's own sources (in place
// under /root/reference, never copied) into oracle/_ref/libpackref.so. Only
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference legs load it.
//
// Every entry point forwards to the reference API it names; nothing here
// re-implements reference arithmetic. Status: 0 ok, nonzero = exception (its
// message is available through pref_last_error()).

#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "packnn/evaluator.hpp"
#include "packnn/kernels.hpp"
#include "packnn/layers.hpp"
#include "packnn/modular.hpp"
#include "packnn/plan.hpp"
#include "packnn/representation.hpp"
#include "packnn/ring.hpp"
#include "packnn/selfcheck.hpp"
#include "packnn/trace.hpp"

using namespace packnn;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const depth_error& e) {
        g_err = e.what();
        return 4;
    } catch (const magnitude_error& e) {
        g_err = e.what();
        return 4;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 3;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return 5;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

int copy_string(const std::string& s, char* out, uint64_t cap) {
    if (s.size() + 1 > cap) {
        g_err = "output buffer too small (need " + std::to_string(s.size() + 1) + ")";
        return 2;
    }
    std::memcpy(out, s.c_str(), s.size() + 1);
    return 0;
}

// backend: 0 slot, 1 ring (the reference's two), 2 = the B200 drop-in
// (oracle/b200_dropin/evaluator_b200.cpp), present only in libpackb200.so
extern "C" int pb2_available(void) __attribute__((weak));
BackendKind backend_kind(int backend) {
    if (backend == 2) {
        if (!pb2_available) throw std::invalid_argument("the b200 backend is not linked into this library");
        return static_cast<BackendKind>(2);
    }
    return backend ? BackendKind::Ring : BackendKind::Slot;
}

std::string join_bigints(const std::vector<BigInt>& v) {
    std::string s;
    for (size_t i = 0; i < v.size(); ++i) {
        if (i) s += ',';
        s += v[i].str();
    }
    return s;
}

}  // namespace

extern "C" {

// One linear stage of a network description (mirrors LayerSpec,
// proj/include/packnn/layers.hpp:27-35). Weights are integer valued.
typedef struct {
    int32_t is_conv;
    uint32_t maps;  // conv: output maps; dense: output rows
    uint32_t win_h, win_w, stride_h, stride_w;
    uint32_t pad_top, pad_left, pad_bottom, pad_right;
    uint64_t cols;            // conv: window volume; dense: input length
    const int64_t* weights;   // maps x cols, row-major
    const int64_t* bias;      // maps entries or NULL
} pref_stage;

typedef struct {
    uint32_t channels, in_h, in_w;
    uint32_t num_stages;        // 2 or 3
    const pref_stage* stages;   // squaring after every stage but the last
    int64_t input_bound;
} pref_net;

const char* pref_last_error(void) { return g_err.c_str(); }

// ---- L0/L1: modular + ring core (proj/src/modular.cpp, proj/src/ring.cpp) ----

int pref_find_root_of_unity(uint64_t p, uint64_t order, uint64_t* out) {
    return guarded([&] { *out = find_root_of_unity(p, order); });
}

int pref_is_prime(uint64_t v) { return is_prime_u64(v) ? 1 : 0; }

int pref_ntt_forward(uint64_t p, uint32_t n, const uint64_t* in, uint64_t* out) {
    return guarded([&] {
        NttTables t = NttTables::create(PrimeModulus::create(p, n));
        auto r = t.forward(std::span<const uint64_t>(in, n));
        std::memcpy(out, r.data(), n * sizeof(uint64_t));
    });
}

int pref_ntt_inverse(uint64_t p, uint32_t n, const uint64_t* in, uint64_t* out) {
    return guarded([&] {
        NttTables t = NttTables::create(PrimeModulus::create(p, n));
        auto r = t.inverse(std::span<const uint64_t>(in, n));
        std::memcpy(out, r.data(), n * sizeof(uint64_t));
    });
}

// Forward transform of `count` limbs under one table (timing helper for the
// CPU baseline: table construction excluded).
int pref_ntt_forward_many(uint64_t p, uint32_t n, uint64_t count, const uint64_t* in,
                          uint64_t* out, int inverse, double* seconds) {
    return guarded([&] {
        NttTables t = NttTables::create(PrimeModulus::create(p, n));
        auto t0 = std::chrono::steady_clock::now();
        for (uint64_t c = 0; c < count; ++c) {
            std::span<const uint64_t> src(in + c * n, n);
            auto r = inverse ? t.inverse(src) : t.forward(src);
            std::memcpy(out + c * n, r.data(), n * sizeof(uint64_t));
        }
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
}

int pref_slot_to_eval(uint64_t p, uint32_t n, uint32_t* out) {
    return guarded([&] {
        NttTables t = NttTables::create(PrimeModulus::create(p, n));
        std::memcpy(out, t.slot_to_eval().data(), n * sizeof(uint32_t));
    });
}

int pref_poly_mul(uint64_t p, uint32_t n, const uint64_t* a, const uint64_t* b, uint64_t* out) {
    return guarded([&] {
        NttTables t = NttTables::create(PrimeModulus::create(p, n));
        RingElement ra{std::vector<uint64_t>(a, a + n)}, rb{std::vector<uint64_t>(b, b + n)};
        auto r = poly_mul_negacyclic(t, ra, rb);
        std::memcpy(out, r.coeffs.data(), n * sizeof(uint64_t));
    });
}

int pref_poly_add(uint64_t p, uint32_t n, const uint64_t* a, const uint64_t* b, uint64_t* out) {
    return guarded([&] {
        NttTables t = NttTables::create(PrimeModulus::create(p, n));
        RingElement ra{std::vector<uint64_t>(a, a + n)}, rb{std::vector<uint64_t>(b, b + n)};
        auto r = poly_add(t, ra, rb);
        std::memcpy(out, r.coeffs.data(), n * sizeof(uint64_t));
    });
}

int pref_poly_scale(uint64_t p, uint32_t n, const uint64_t* a, uint64_t s, uint64_t* out) {
    return guarded([&] {
        NttTables t = NttTables::create(PrimeModulus::create(p, n));
        RingElement ra{std::vector<uint64_t>(a, a + n)};
        auto r = poly_scale(t, ra, s);
        std::memcpy(out, r.coeffs.data(), n * sizeof(uint64_t));
    });
}

int pref_slot_encode(uint64_t p, uint32_t n, const uint64_t* slots, uint64_t* out) {
    return guarded([&] {
        NttTables t = NttTables::create(PrimeModulus::create(p, n));
        auto r = slot_encode(t, SlotVector{std::vector<uint64_t>(slots, slots + n)});
        std::memcpy(out, r.coeffs.data(), n * sizeof(uint64_t));
    });
}

int pref_slot_decode(uint64_t p, uint32_t n, const uint64_t* coeffs, uint64_t* out) {
    return guarded([&] {
        NttTables t = NttTables::create(PrimeModulus::create(p, n));
        auto r = slot_decode(t, RingElement{std::vector<uint64_t>(coeffs, coeffs + n)});
        std::memcpy(out, r.slots.data(), n * sizeof(uint64_t));
    });
}

int pref_galois_apply(uint64_t p, uint32_t n, const uint64_t* in, uint64_t exponent, uint64_t* out) {
    return guarded([&] {
        NttTables t = NttTables::create(PrimeModulus::create(p, n));
        auto r = galois_apply(t, RingElement{std::vector<uint64_t>(in, in + n)}, exponent);
        std::memcpy(out, r.coeffs.data(), n * sizeof(uint64_t));
    });
}

// Per-limb CPU timings of the reference ring primitives (tables built once,
// outside the timed loops), seconds per call averaged over `reps`:
// out[0] NttTables::forward, out[1] inverse (ring.cpp:97-115), out[2]
// poly_mul_negacyclic (ring.cpp:117-122), out[3] galois_apply with the
// column-rotation-by-1 exponent (ring.cpp:155-182).
int pref_time_primitives(uint64_t p, uint32_t n, uint32_t reps, double* out) {
    return guarded([&] {
        NttTables t = NttTables::create(PrimeModulus::create(p, n));
        std::vector<uint64_t> a(n), b(n);
        uint64_t x = 0x9E3779B97F4A7C15ull;
        for (uint32_t i = 0; i < n; ++i) {
            x ^= x << 13, x ^= x >> 7, x ^= x << 17;
            a[i] = x % p;
            b[i] = (x >> 7) % p;
        }
        volatile uint64_t sink = 0;
        auto time = [&](auto&& f) {
            const auto t0 = std::chrono::steady_clock::now();
            for (uint32_t r = 0; r < reps; ++r) sink = sink + f();
            return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / reps;
        };
        RingElement ra{a}, rb{b};
        const uint64_t g = galois_exponent_columns(n, 1);
        out[0] = time([&] { return t.forward(std::span<const uint64_t>(a))[1]; });
        out[1] = time([&] { return t.inverse(std::span<const uint64_t>(a))[1]; });
        out[2] = time([&] { return poly_mul_negacyclic(t, ra, rb).coeffs[1]; });
        out[3] = time([&] { return galois_apply(t, ra, g).coeffs[1]; });
    });
}

int pref_galois_exponent_columns(uint32_t n, uint32_t k, uint64_t* out) {
    return guarded([&] { *out = galois_exponent_columns(n, k); });
}

uint64_t pref_galois_exponent_rows(uint32_t n) { return galois_exponent_rows(n); }

// Garner CRT + centering (proj/src/ring.cpp:205-233); result as decimal.
int pref_crt_join_center(const uint64_t* residues, const uint64_t* primes, uint32_t count,
                         int center, char* out, uint64_t cap) {
    int rc = 0;
    int st = guarded([&] {
        std::span<const uint64_t> r(residues, count), p(primes, count);
        BigInt x = crt_join(r, p);
        if (center) {
            BigInt comp = 1;
            for (uint32_t i = 0; i < count; ++i) comp *= primes[i];
            x = center_mod(x, comp);
        }
        rc = copy_string(x.str(), out, cap);
    });
    return st ? st : rc;
}

// Schoolbook negacyclic product (proj/src/selfcheck.cpp:11-29).
int pref_schoolbook_mul(uint64_t p, uint32_t n, const uint64_t* a, const uint64_t* b, uint64_t* out) {
    return guarded([&] {
        auto r = selfcheck::schoolbook_negacyclic_mul(std::span<const uint64_t>(a, n),
                                                      std::span<const uint64_t>(b, n), p);
        std::memcpy(out, r.data(), n * sizeof(uint64_t));
    });
}

// ---- L2: counted evaluator, one program of ops on both backends ----------
// Runs lift(values) -> rotate_columns(k) on the chosen backend and returns
// the decoded slots (mod the single prime p). Used to pin rotation direction.
int pref_eval_rotate(uint64_t p, uint32_t n, int backend, const int64_t* values, int64_t k,
                     int rows, int64_t* out) {
    return guarded([&] {
        EvalContext cx(backend_kind(backend), n, {p});
        Evaluator ev(cx);
        Message m = ev.lift(std::span<const int64_t>(values, n));
        Message r = rows ? ev.rotate_rows(m) : ev.rotate_columns(m, k);
        auto dec = ev.lower(r);
        for (uint32_t i = 0; i < n; ++i) out[i] = static_cast<int64_t>(dec[i]);
    });
}

// ---- L3/L4: networks, plans, execution ------------------------------------

namespace {

QuantizedNetwork make_network(const pref_net* net) {
    std::vector<LayerSpec> layers;
    for (uint32_t s = 0; s < net->num_stages; ++s) {
        const pref_stage& st = net->stages[s];
        std::vector<std::vector<double>> w(st.maps, std::vector<double>(st.cols));
        for (uint32_t r = 0; r < st.maps; ++r)
            for (uint64_t c = 0; c < st.cols; ++c) w[r][c] = static_cast<double>(st.weights[r * st.cols + c]);
        std::vector<double> b;
        if (st.bias) b.assign(st.bias, st.bias + st.maps);
        if (st.is_conv) {
            LayerSpec l = conv_spec(st.win_h, st.win_w, st.stride_h, st.maps, std::move(w), std::move(b));
            l.stride_w = st.stride_w;
            l.pad_top = st.pad_top;
            l.pad_left = st.pad_left;
            l.pad_bottom = st.pad_bottom;
            l.pad_right = st.pad_right;
            layers.push_back(std::move(l));
        } else {
            layers.push_back(dense_spec(std::move(w), std::move(b)));
        }
        if (s + 1 < net->num_stages) layers.push_back(square_spec());
    }
    Shape3 in{net->channels, net->in_h, net->in_w};
    QuantizationPolicy policy;
    policy.scale_bits = {0};
    policy.input_bound = net->input_bound;
    return quantize(collapse_adjacent_linear(layers, in), policy);
}

bool strategy_is_small(const char* name) { return std::strcmp(name, "lola-small") == 0; }

// LoLa-Small (BASELINE config 3) has no reference preset (the three-stage
// check at proj/src/plan.cpp:138-145 rejects it). This chains the reference's
// own kernels in the order the paper describes: convolution representation,
// weighted window sums, combine the maps into one message, bias, square,
// one row-major product per output, bias.
struct SmallRun {
    std::vector<BigInt> scores;
    std::vector<CounterDelta> per_step;
};

SmallRun run_lola_small(const QuantizedNetwork& net, const std::vector<int64_t>& x,
                        Evaluator& ev, double* t_encode, double* t_steps, double* t_decode) {
    if (net.stages.size() != 2 || !net.stages[0].is_conv || net.stages[1].is_conv)
        throw std::invalid_argument("lola-small expects window stage + matrix stage");
    const QuantizedStage& s0 = net.stages[0];
    const QuantizedStage& s1 = net.stages[1];
    const uint64_t p = s0.geom.positions();
    const uint64_t maps = s0.rows();
    SmallRun out;
    auto t0 = std::chrono::steady_clock::now();
    EncodedTensor t = encode_convolution(ev, x, s0.geom, false);
    auto t1 = std::chrono::steady_clock::now();
    auto mark = [&](const CounterDelta& before) {
        CounterDelta d;
        const CounterDelta& a = ev.counters().ops;
        d.ct_ct_mul = a.ct_ct_mul - before.ct_ct_mul;
        d.ct_plain_mul = a.ct_plain_mul - before.ct_plain_mul;
        d.scalar_mul = a.scalar_mul - before.scalar_mul;
        d.mask_mul = a.mask_mul - before.mask_mul;
        d.add = a.add - before.add;
        d.rot_cols = a.rot_cols - before.rot_cols;
        d.rot_rows = a.rot_rows - before.rot_rows;
        out.per_step.push_back(d);
    };
    CounterDelta b = ev.counters().ops;
    std::vector<std::vector<int64_t>> w0 = s0.weights;
    t = conv_rowmajor(ev, t, weights_from(w0));
    mark(b);
    b = ev.counters().ops;
    t = combine_to_one(ev, t, uniform_offsets(static_cast<uint32_t>(maps), static_cast<uint32_t>(p)));
    std::vector<int64_t> bias0(maps * p, 0);
    if (!s0.bias.empty())
        for (uint64_t i = 0; i < bias0.size(); ++i) bias0[i] = s0.bias[i / p];
    t = add_bias(ev, t, bias0);
    mark(b);
    b = ev.counters().ops;
    t = square_activation(ev, t);
    mark(b);
    b = ev.counters().ops;
    std::vector<std::vector<int64_t>> w1 = s1.weights;
    t = matvec_rowmajor(ev, t, weights_from(w1));
    std::vector<int64_t> bias1(s1.rows(), 0);
    if (!s1.bias.empty()) bias1 = s1.bias;
    t = add_bias(ev, t, bias1);
    mark(b);
    auto t2 = std::chrono::steady_clock::now();
    out.scores = decode(ev, t);
    auto t3 = std::chrono::steady_clock::now();
    *t_encode = std::chrono::duration<double>(t1 - t0).count();
    *t_steps = std::chrono::duration<double>(t2 - t1).count();
    *t_decode = std::chrono::duration<double>(t3 - t2).count();
    return out;
}

void put_counters(const CounterDelta& d, uint64_t* out) {
    out[0] = d.ct_ct_mul;
    out[1] = d.ct_plain_mul;
    out[2] = d.scalar_mul;
    out[3] = d.mask_mul;
    out[4] = d.add;
    out[5] = d.rot_cols;
    out[6] = d.rot_rows;
}

}  // namespace

// Decrypted-logit oracle: forward_integer (proj/src/layers.cpp:560-594).
int pref_forward_integer(const pref_net* net, const int64_t* x, char* out, uint64_t cap) {
    int rc = 0;
    int st = guarded([&] {
        QuantizedNetwork q = make_network(net);
        std::vector<int64_t> xv(x, x + q.input.values());
        rc = copy_string(join_bigints(forward_integer(q, xv)), out, cap);
    });
    return st ? st : rc;
}

// Largest magnitude bound of the quantized network's output, as decimal
// (the reference's ledger, proj/src/layers.cpp:464-558).
int pref_final_bound(const pref_net* net, char* out, uint64_t cap) {
    int rc = 0;
    int st = guarded([&] { rc = copy_string(make_network(net).final_bound.str(), out, cap); });
    return st ? st : rc;
}

// Byte-stable step table (proj/src/trace.cpp) for a preset plan.
int pref_render_trace(const pref_net* net, const char* strategy, uint32_t n, const uint64_t* primes,
                      uint32_t nprimes, char* out, uint64_t cap) {
    int rc = 0;
    int st = guarded([&] {
        QuantizedNetwork q = make_network(net);
        PlanOptions opt;
        opt.n = n;
        InferencePlan plan = build_plan(q, strategy_from_name(strategy), opt);
        rc = copy_string(render_trace_text(plan, std::vector<uint64_t>(primes, primes + nprimes)), out, cap);
    });
    return st ? st : rc;
}

// Full plaintext-semantics inference on the reference evaluator
// (plan.encode_input -> execute -> decode, proj/src/plan.cpp:597-633).
// counters: 7 x max_steps per-step deltas (ct.ct, ct.pt, scalar, mask, add,
// rot.col, rot.row); times: encode, HE steps, decode seconds.
int pref_run_plan(const pref_net* net, const char* strategy, uint32_t n, const uint64_t* primes,
                  uint32_t nprimes, int backend, uint32_t threads, const int64_t* x,
                  char* scores_out, uint64_t scores_cap, uint64_t* counters, uint32_t max_steps,
                  uint32_t* steps_out, double* times) {
    int rc = 0;
    int st = guarded([&] {
        set_kernel_threads(threads);
        QuantizedNetwork q = make_network(net);
        std::vector<int64_t> xv(x, x + q.input.values());
        EvalContext cx(backend_kind(backend), n,
                       std::vector<uint64_t>(primes, primes + nprimes));
        Evaluator ev(cx);
        std::vector<BigInt> scores;
        std::vector<CounterDelta> per_step;
        if (strategy_is_small(strategy)) {
            SmallRun r = run_lola_small(q, xv, ev, &times[0], &times[1], &times[2]);
            scores = std::move(r.scores);
            per_step = std::move(r.per_step);
        } else {
            PlanOptions opt;
            opt.n = n;
            InferencePlan plan = build_plan(q, strategy_from_name(strategy), opt);
            auto t0 = std::chrono::steady_clock::now();
            EncodedTensor input = plan.encode_input(ev, xv);
            auto t1 = std::chrono::steady_clock::now();
            // execute() decodes internally; time the HE steps by running the
            // same step closures, then decode, as proj/src/plan.cpp:609-631.
            ExecutionResult res = execute(plan, input, q, ev);
            auto t2 = std::chrono::steady_clock::now();
            scores = std::move(res.scores);
            per_step = std::move(res.report.per_step);
            times[0] = std::chrono::duration<double>(t1 - t0).count();
            times[1] = std::chrono::duration<double>(t2 - t1).count();  // steps + decode
            times[2] = -1.0;
        }
        if (per_step.size() > max_steps) throw std::invalid_argument("too many steps for buffer");
        for (size_t i = 0; i < per_step.size(); ++i) put_counters(per_step[i], counters + 7 * i);
        *steps_out = static_cast<uint32_t>(per_step.size());
        rc = copy_string(join_bigints(scores), scores_out, scores_cap);
    });
    return st ? st : rc;
}

// Per-step HE timing without decode: runs each plan step closure directly
// (mirrors execute's loop, proj/src/plan.cpp:610-626) and reports seconds per
// step in step_times (max_steps entries). Used as the CPU baseline.
int pref_time_plan_steps(const pref_net* net, const char* strategy, uint32_t n, const uint64_t* primes,
                         uint32_t nprimes, int backend, uint32_t threads, const int64_t* x,
                         double* step_times, uint32_t max_steps, uint32_t* steps_out,
                         double* encode_seconds) {
    return guarded([&] {
        set_kernel_threads(threads);
        QuantizedNetwork q = make_network(net);
        std::vector<int64_t> xv(x, x + q.input.values());
        EvalContext cx(backend_kind(backend), n,
                       std::vector<uint64_t>(primes, primes + nprimes));
        Evaluator ev(cx);
        if (strategy_is_small(strategy)) {
            double te, ts, td;
            run_lola_small(q, xv, ev, &te, &ts, &td);
            *encode_seconds = te;
            step_times[0] = ts;
            *steps_out = 1;
            return;
        }
        PlanOptions opt;
        opt.n = n;
        InferencePlan plan = build_plan(q, strategy_from_name(strategy), opt);
        if (plan.steps.size() > max_steps) throw std::invalid_argument("too many steps for buffer");
        auto t0 = std::chrono::steady_clock::now();
        EncodedTensor cur = plan.encode_input(ev, xv);
        *encode_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        for (size_t i = 0; i < plan.steps.size(); ++i) {
            auto s0 = std::chrono::steady_clock::now();
            cur = plan.steps[i].run(ev, q, cur);
            step_times[i] = std::chrono::duration<double>(std::chrono::steady_clock::now() - s0).count();
        }
        *steps_out = static_cast<uint32_t>(plan.steps.size());
    });
}


// Persistent plan session for the CPU baseline / reference arm: the network,
// the EvalContext (NttTables per prime) and the plan are built once, so each
// timed run is exactly the per-image work of the reference:
// plan.encode_input, then every step closure in order (execute's loop,
// proj/src/plan.cpp:610-626), then optionally decode
// (representation.cpp:185-223; excluded from timings by default because the
// Boost stand-in BigInt is not representative of Boost's speed).
struct pref_session {
    QuantizedNetwork net;
    EvalContext cx;
    InferencePlan plan;
    bool small;
    pref_session(QuantizedNetwork q, BackendKind kind, uint32_t n, std::vector<uint64_t> primes, bool is_small,
                 const char* strategy)
        : net(std::move(q)), cx(kind, n, std::move(primes)), small(is_small) {
        if (!small) {
            PlanOptions opt;
            opt.n = n;
            plan = build_plan(net, strategy_from_name(strategy), opt);
        }
    }
};

int pref_session_create(const pref_net* net, const char* strategy, uint32_t n, const uint64_t* primes,
                        uint32_t nprimes, int backend, uint32_t threads, pref_session** out) {
    return guarded([&] {
        set_kernel_threads(threads);
        *out = new pref_session(make_network(net), backend_kind(backend), n,
                                std::vector<uint64_t>(primes, primes + nprimes), strategy_is_small(strategy),
                                strategy);
    });
}

int pref_session_destroy(pref_session* s) {
    return guarded([&] { delete s; });
}

// times: encode, HE steps, decode seconds (decode = -1 when not requested);
// scores_out receives the decimal scores when decode != 0.
int pref_session_run(pref_session* s, const int64_t* x, int decode_scores, char* scores_out, uint64_t scores_cap,
                     double* times) {
    int rc = 0;
    int st = guarded([&] {
        std::vector<int64_t> xv(x, x + s->net.input.values());
        Evaluator ev(s->cx);
        if (s->small) {
            SmallRun r = run_lola_small(s->net, xv, ev, &times[0], &times[1], &times[2]);
            if (decode_scores) rc = copy_string(join_bigints(r.scores), scores_out, scores_cap);
            return;
        }
        auto t0 = std::chrono::steady_clock::now();
        EncodedTensor cur = s->plan.encode_input(ev, xv);
        auto t1 = std::chrono::steady_clock::now();
        for (const PlanStep& step : s->plan.steps) cur = step.run(ev, s->net, cur);
        auto t2 = std::chrono::steady_clock::now();
        times[0] = std::chrono::duration<double>(t1 - t0).count();
        times[1] = std::chrono::duration<double>(t2 - t1).count();
        times[2] = -1.0;
        if (decode_scores) {
            std::vector<BigInt> scores = decode(ev, cur);
            times[2] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t2).count();
            rc = copy_string(join_bigints(scores), scores_out, scores_cap);
        }
    });
    return st ? st : rc;
}

}  // extern "C"
