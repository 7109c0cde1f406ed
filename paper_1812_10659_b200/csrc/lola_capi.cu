// extern "C" entry points of the LoLa layer (include/lola_b200.h, §LoLa).
#include <chrono>
#include <cstring>
#include <memory>
#include <string>

#include "../../include/lola_b200.h"
#include "capi_internal.hpp"
#include "lola_plan.hpp"

namespace {

using lb::capi::guarded;

// lb_network -> quantized network (shapes chained as in layer_output_shape,
// proj/src/layers.cpp:333-363; a squaring after every stage but the last).
lb::lola::Network to_network(const lb_network* in) {
    using namespace lb::lola;
    if (!in || !in->stages || in->num_stages == 0) throw std::invalid_argument("empty network");
    Network net;
    net.input = {in->channels, in->in_h, in->in_w};
    net.input_bound = in->input_bound;
    Shape3 cur = net.input;
    for (uint32_t k = 0; k < in->num_stages; ++k) {
        const lb_stage& s = in->stages[k];
        Stage st;
        st.is_conv = s.is_conv != 0;
        st.rows = s.maps;
        st.cols = s.cols;
        st.in_shape = cur;
        if (!s.weights || s.maps == 0) throw std::invalid_argument("missing weights");
        st.weights.assign(s.weights, s.weights + uint64_t(s.maps) * s.cols);
        if (s.bias) st.bias.assign(s.bias, s.bias + s.maps);
        if (st.is_conv) {
            ConvGeometry& g = st.geom;
            g.channels = cur.c;
            g.in_h = cur.h;
            g.in_w = cur.w;
            g.win_h = s.win_h;
            g.win_w = s.win_w;
            g.stride_h = s.stride_h;
            g.stride_w = s.stride_w;
            g.pad_top = s.pad_top;
            g.pad_left = s.pad_left;
            g.pad_bottom = s.pad_bottom;
            g.pad_right = s.pad_right;
            if (s.cols != g.window_volume()) throw std::invalid_argument("weight row does not cover the window");
            st.out_shape = {s.maps, g.out_h(), g.out_w()};
        } else {
            if (s.cols != cur.values()) throw std::invalid_argument("weight row does not cover the input");
            st.out_shape = {s.maps, 1, 1};
        }
        cur = st.out_shape;
        net.stages.push_back(std::move(st));
        net.squares_after.push_back(k + 1 < in->num_stages ? 1 : 0);
    }
    return net;
}

void put_counters(const lb::lola::CounterDelta& d, uint64_t* out) {
    const auto v = d.values();
    std::memcpy(out, v.data(), 7 * sizeof(uint64_t));
}

}  // namespace

struct lb_lola_session {
    lb::lola::Network net;
    lb::lola::Plan plan;
    std::unique_ptr<lb::lola::EvalContext> ecx;
    std::unique_ptr<lb::lola::Evaluator> ev;
    uint32_t batch = 0;
    uint64_t outputs = 0;
    uint64_t input_values = 0;
    lb::lola::EncodedTensor input;   // encrypted input (kept by encrypt)
    lb::lola::EncodedTensor output;  // encrypted scores (kept by execute)
    std::vector<lb::lola::CounterDelta> per_step;
    // CUDA-graph mode (lb_lola_session_set_graph): the HE steps captured once
    // into a graph that reads `input`'s buffers and writes graph-allocated
    // outputs (valid until the next launch), replayed by every execute
    // the session's ops run on its own non-blocking stream (a graph cannot
    // capture the legacy default stream); every entry point orders it after
    // the caller's stream on entry and the caller's stream after it on exit
    cudaStream_t caller = nullptr, own = nullptr;
    cudaEvent_t in_ev = nullptr, out_ev = nullptr;
    bool use_graph = false;
    cudaGraphExec_t graph = nullptr;
    uint64_t graph_kernels = 0;          // kernel launches one replay performs
    std::vector<void*> graph_outputs;    // graph allocations the host still references
    ~lb_lola_session();
};

namespace {

void phase_encrypt(lb_lola_session* s, const int64_t* images, int on_device) {
    cudaStream_t st = s->ecx->stream();
    lb::DeviceBuffer dimg;
    const int64_t* img = images;
    if (!on_device) {
        dimg = lb::DeviceBuffer(uint64_t(s->batch) * s->input_values * 8, st);
        LB_CUDA(cudaMemcpyAsync(dimg.get(), images, uint64_t(s->batch) * s->input_values * 8, cudaMemcpyHostToDevice,
                                st));
        img = dimg.get<int64_t>();
    }
    lb::lola::EncodedTensor fresh = s->plan.encode_input(*s->ev, img);
    if (s->graph) {
        // the captured graph reads the input buffers it was captured with:
        // move the new ciphertexts into them
        if (fresh.messages.size() != s->input.messages.size()) throw std::logic_error("input shape changed");
        const size_t bytes = s->ecx->payload_bytes();
        for (size_t i = 0; i < fresh.messages.size(); ++i)
            LB_CUDA(cudaMemcpyAsync(s->input.messages[i].data(), fresh.messages[i].data(), bytes,
                                    cudaMemcpyDeviceToDevice, st));
        for (size_t i = 0; i < fresh.messages.size(); ++i) {
            lb::lola::Message keep = s->input.messages[i];
            s->input.messages[i] = std::move(fresh.messages[i]);
            s->input.messages[i].payload = keep.payload;  // same buffers, the new depth / magnitude
        }
        return;
    }
    s->input = std::move(fresh);
}

void phase_execute(lb_lola_session* s, bool keep_input) {
    if (s->input.messages.empty()) throw std::invalid_argument("no encrypted input: call encrypt first");
    lb::lola::Evaluator& ev = *s->ev;
    ev.counters() = lb::lola::OpCounters{};
    lb::lola::EncodedTensor in = keep_input ? s->input : std::move(s->input);
    lb::lola::ExecutionResult res = lb::lola::execute(s->plan, std::move(in), ev);
    s->output = std::move(res.output);
    s->per_step = std::move(res.per_step);
}

void free_graph(lb_lola_session* s) {
    cudaStream_t st = s->ecx->stream();
    s->output = {};
    for (void* p : s->graph_outputs) cudaFreeAsync(p, st);
    s->graph_outputs.clear();
    if (s->graph) {
        cudaStreamSynchronize(st);
        cudaGraphExecDestroy(s->graph);
        s->graph = nullptr;
    }
}

// execute through a CUDA graph: the first call runs the steps once
// uncaptured (key generation, plaintext encodings, side streams), then
// captures a second run (every counted op becomes graph nodes, the side-stream
// fan-out becomes parallel branches) and instantiates it; every call then
// replays it with one launch. Counters are the captured run's, which the
// plan checked step by step.
void phase_execute_graph(lb_lola_session* s) {
    cudaStream_t st = s->ecx->stream();
    if (!s->graph) {
        if (s->input.messages.empty()) throw std::invalid_argument("no encrypted input: call encrypt first");
        phase_execute(s, true);
        LB_CUDA(cudaDeviceSynchronize());
        s->output = {};
        auto& launches = lb::launch_counter();
        const uint64_t l0 = launches.load();
        s->ecx->set_capturing(true);
        LB_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
        cudaGraph_t g = nullptr;
        try {
            phase_execute(s, true);
        } catch (...) {
            cudaStreamEndCapture(st, &g);
            if (g) cudaGraphDestroy(g);
            s->ecx->set_capturing(false);
            s->output = {};
            throw;
        }
        s->ecx->set_capturing(false);
        LB_CUDA(cudaStreamEndCapture(st, &g));
        s->graph_kernels = launches.load() - l0;
        launches.fetch_sub(s->graph_kernels);  // captured, not launched
        const cudaError_t e = cudaGraphInstantiateWithFlags(&s->graph, g, cudaGraphInstantiateFlagAutoFreeOnLaunch);
        cudaGraphDestroy(g);
        LB_CUDA(e);
        // the outputs live in graph allocations: AutoFreeOnLaunch frees them at
        // the next launch, which re-creates them at the same addresses
        for (auto& m : s->output.messages)
            if (m.payload->buf.owned()) s->graph_outputs.push_back(m.payload->buf.disown());
    }
    LB_CUDA(cudaGraphLaunch(s->graph, st));
    lb::launch_counter().fetch_add(s->graph_kernels, std::memory_order_relaxed);
}

void phase_decrypt(lb_lola_session* s, uint64_t* scores, int on_device) {
    if (s->output.messages.empty()) throw std::invalid_argument("no result: call execute first");
    cudaStream_t st = s->ecx->stream();
    lb::DeviceBuffer dec = lb::lola::decode_values(*s->ev, s->output);
    const uint64_t bytes = uint64_t(s->batch) * s->outputs * 32;
    if (dec.bytes() != bytes) throw std::logic_error("decoded output size mismatch");
    LB_CUDA(cudaMemcpyAsync(scores, dec.get(), bytes, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                            st));
    LB_CUDA(cudaStreamSynchronize(st));
}

lb::lola::PlanOptions plan_options(const lb_plan_options* opt) {
    lb::lola::PlanOptions o;
    if (opt) o.window_matrix_threshold = opt->window_matrix_threshold;
    return o;
}

}  // namespace

lb_lola_session::~lb_lola_session() {
    try {
        if (ecx) free_graph(this);
    } catch (...) {
    }
    output = {};
    input = {};
    ev.reset();
    ecx.reset();
    plan = lb::lola::Plan{};  // cached device operands are freed on `own`
    if (own) {
        cudaStreamSynchronize(own);
        cudaStreamDestroy(own);
    }
    if (in_ev) cudaEventDestroy(in_ev);
    if (out_ev) cudaEventDestroy(out_ev);
}

namespace {

// caller's stream -> session stream on entry, session stream -> caller's on exit
struct StreamBridge {
    lb_lola_session* s;
    explicit StreamBridge(lb_lola_session* ss) : s(ss) {
        LB_CUDA(cudaEventRecord(s->in_ev, s->caller));
        LB_CUDA(cudaStreamWaitEvent(s->own, s->in_ev, 0));
    }
    ~StreamBridge() {
        if (cudaEventRecord(s->out_ev, s->own) == cudaSuccess) cudaStreamWaitEvent(s->caller, s->out_ev, 0);
    }
};

}  // namespace

extern "C" {

int lb_plan_counters(const lb_network* net, const char* strategy, uint32_t n, uint64_t* counters, uint32_t max_steps,
                     uint32_t* steps_out, uint32_t* depth_needed, uint64_t* predicted_peak) {
    return lb_plan_counters_ex(net, strategy, n, nullptr, counters, max_steps, steps_out, depth_needed,
                               predicted_peak);
}

int lb_plan_counters_ex(const lb_network* net, const char* strategy, uint32_t n, const lb_plan_options* opt,
                        uint64_t* counters, uint32_t max_steps, uint32_t* steps_out, uint32_t* depth_needed,
                        uint64_t* predicted_peak) {
    return guarded([&] {
        auto nw = to_network(net);
        auto plan = lb::lola::build_plan(nw, lb::lola::strategy_from_name(strategy), n, plan_options(opt));
        if (plan.steps.size() > max_steps) throw std::invalid_argument("too many steps for buffer");
        for (size_t i = 0; i < plan.steps.size(); ++i) put_counters(plan.steps[i].predicted, counters + 7 * i);
        if (steps_out) *steps_out = static_cast<uint32_t>(plan.steps.size());
        if (depth_needed) *depth_needed = plan.depth_needed;
        if (predicted_peak) *predicted_peak = plan.predicted_peak();
    });
}

int lb_lola_session_create(lb_context* cx, const lb_network* net, const char* strategy, uint32_t batch,
                           uint32_t max_depth, void* stream, lb_lola_session** out) {
    return lb_lola_session_create_ex(cx, net, strategy, batch, max_depth, nullptr, stream, out);
}

int lb_lola_session_create_ex(lb_context* cx, const lb_network* net, const char* strategy, uint32_t batch,
                              uint32_t max_depth, const lb_plan_options* opt, void* stream, lb_lola_session** out) {
    return guarded([&] {
        if (!cx || !out) throw std::invalid_argument("null argument");
        cx->cx.activate();
        auto s = std::make_unique<lb_lola_session>();
        s->net = to_network(net);
        const lb::lola::Strategy strat = lb::lola::strategy_from_name(strategy);
        s->plan = lb::lola::build_plan(s->net, strat, cx->cx.n(), plan_options(opt));
        // record tensors (cryptonets-simd) pack the images into the slots of
        // one message: one batch entry carrying `batch` records
        const bool records = strat == lb::lola::Strategy::CryptonetsSimd;
        if (records && (batch == 0 || batch > cx->cx.n()))
            throw std::invalid_argument("cryptonets-simd packs at most n images per session");
        s->caller = static_cast<cudaStream_t>(stream);
        LB_CUDA(cudaStreamCreateWithFlags(&s->own, cudaStreamNonBlocking));
        LB_CUDA(cudaEventCreateWithFlags(&s->in_ev, cudaEventDisableTiming));
        LB_CUDA(cudaEventCreateWithFlags(&s->out_ev, cudaEventDisableTiming));
        s->ecx = std::make_unique<lb::lola::EvalContext>(cx->cx, records ? 1 : batch, max_depth, s->own);
        if (records) s->ecx->set_records(batch);
        s->ev = std::make_unique<lb::lola::Evaluator>(*s->ecx);
        s->batch = batch;
        s->outputs = s->net.stages.back().out_shape.values();
        s->input_values = s->net.input.values();
        *out = s.release();
    });
}

int lb_lola_session_destroy(lb_lola_session* s) {
    return guarded([&] { delete s; });
}

int lb_lola_session_info(const lb_lola_session* s, uint32_t* steps, uint64_t* outputs, uint64_t* input_values) {
    return guarded([&] {
        if (steps) *steps = static_cast<uint32_t>(s->plan.steps.size());
        if (outputs) *outputs = s->outputs;
        if (input_values) *input_values = s->input_values;
    });
}

// images: [batch][input_values] int64, device (images_on_device = 1) or host;
// scores: [batch][outputs][4] signed 256-bit words, device or host alike.
int lb_lola_session_run(lb_lola_session* s, const int64_t* images, int images_on_device, uint64_t* scores,
                        int scores_on_device, uint64_t* counters, double* times) {
    return guarded([&] {
        using clock = std::chrono::steady_clock;
        StreamBridge bridge(s);
        cudaStream_t st = s->ecx->stream();
        const auto t0 = clock::now();
        phase_encrypt(s, images, images_on_device);
        if (times) LB_CUDA(cudaStreamSynchronize(st));
        const auto t1 = clock::now();
        if (s->use_graph)
            phase_execute_graph(s);
        else
            phase_execute(s, false);
        if (times) LB_CUDA(cudaStreamSynchronize(st));
        const auto t2 = clock::now();
        phase_decrypt(s, scores, scores_on_device);
        const auto t3 = clock::now();
        if (counters)
            for (size_t i = 0; i < s->per_step.size(); ++i) put_counters(s->per_step[i], counters + 7 * i);
        if (times) {
            times[0] = std::chrono::duration<double>(t1 - t0).count();
            times[1] = std::chrono::duration<double>(t2 - t1).count();
            times[2] = std::chrono::duration<double>(t3 - t2).count();
        }
    });
}

int lb_lola_session_encrypt(lb_lola_session* s, const int64_t* images, int images_on_device) {
    return guarded([&] {
        StreamBridge bridge(s);
        phase_encrypt(s, images, images_on_device);
    });
}

int lb_lola_session_execute(lb_lola_session* s, uint64_t* counters) {
    return guarded([&] {
        StreamBridge bridge(s);
        if (s->use_graph)
            phase_execute_graph(s);
        else
            phase_execute(s, true);
        if (counters)
            for (size_t i = 0; i < s->per_step.size(); ++i) put_counters(s->per_step[i], counters + 7 * i);
    });
}

int lb_lola_session_set_graph(lb_lola_session* s, int enable) {
    return guarded([&] {
        if (!s) throw std::invalid_argument("null session");
        if (!enable) free_graph(s);
        s->use_graph = enable != 0;
    });
}

int lb_lola_session_decrypt(lb_lola_session* s, uint64_t* scores, int scores_on_device) {
    return guarded([&] {
        StreamBridge bridge(s);
        phase_decrypt(s, scores, scores_on_device);
    });
}

uint64_t lb_launch_count(void) { return lb::launch_counter().load(); }

int lb_lola_session_output(const lb_lola_session* s, uint32_t index, const void** data, uint32_t* count) {
    return guarded([&] {
        if (count) *count = static_cast<uint32_t>(s->output.messages.size());
        if (data) {
            if (index >= s->output.messages.size()) throw std::invalid_argument("output index out of range");
            *data = s->output.messages[index].data();
        }
    });
}

}  // extern "C"
