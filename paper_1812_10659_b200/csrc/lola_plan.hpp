// LoLa layer evaluator on the device evaluator: representations (dense,
// sparse, stacked, interleaved, convolution), the packed kernels
// (conv-as-scalar-sums, rotate-and-sum dense layers, square activation) and
// the preset plans with exact predicted operation counts.
//
// Semantics, operation order and counting follow the reference
// (proj/src/representation.cpp, proj/src/kernels.cpp, proj/src/plan.cpp);
// cited per function in lola_plan.cu. The network description is the
// already-quantized integer network (the reference's collapse/quantize step,
// proj/src/layers.cpp:401-558, is offline preprocessing and out of scope).
#pragma once

#include <functional>
#include <optional>
#include <string>
#include <vector>

#include "lola_eval.hpp"

namespace lb::lola {

enum class RepKind { Dense, Sparse, Stacked, Interleaved, Convolution, Simd };
std::string rep_name(RepKind kind, bool hybrid = false);

struct Representation {
    RepKind kind = RepKind::Dense;
    uint64_t length = 0;
    uint64_t pad = 0;
    uint32_t copies = 1;
    bool broadcast = false;
    uint32_t value_slot = 0;
    uint32_t windows = 0;
    std::vector<uint32_t> slot_of;  // empty = identity
    bool dirty = false;

    bool identity_layout() const;
    uint32_t slot(uint64_t i) const { return slot_of.empty() ? static_cast<uint32_t>(i) : slot_of[i]; }
};

struct EncodedTensor {
    Representation rep;
    std::vector<Message> messages;
};

struct ConvGeometry {
    uint32_t in_h = 0, in_w = 0, channels = 1;
    uint32_t win_h = 1, win_w = 1;
    uint32_t stride_h = 1, stride_w = 1;
    uint32_t pad_top = 0, pad_left = 0, pad_bottom = 0, pad_right = 0;
    uint32_t out_h() const;
    uint32_t out_w() const;
    uint32_t positions() const { return out_h() * out_w(); }
    uint32_t window_volume() const { return channels * win_h * win_w; }
    std::optional<uint32_t> tap(uint32_t j, uint32_t w) const;
};

// Row-major weights produced on demand.
struct Weights {
    uint64_t rows = 0, cols = 0;
    std::function<int64_t(uint64_t, uint64_t)> at;
};

struct Shape3 {
    uint32_t c = 1, h = 1, w = 1;
    uint64_t values() const { return uint64_t(c) * h * w; }
};

// One quantized linear stage (window stencil or matrix).
struct Stage {
    bool is_conv = false;
    ConvGeometry geom;
    uint64_t rows = 0, cols = 0;  // conv: maps x window volume; dense: out x in
    std::vector<int64_t> weights; // rows x cols
    std::vector<int64_t> bias;    // rows or empty
    Shape3 in_shape, out_shape;
    int64_t w(uint64_t r, uint64_t c) const { return weights[r * cols + c]; }
};

struct Network {
    Shape3 input;
    std::vector<Stage> stages;
    std::vector<uint32_t> squares_after;
    int64_t input_bound = 255;
};

enum class Strategy { LolaMnist, LolaDenseMnist, LolaCifar, CryptonetsSimd, LolaSmall, LinearFeatures };
Strategy strategy_from_name(const std::string& name);
const char* strategy_name(Strategy s);

using StepFn = std::function<EncodedTensor(Evaluator&, const EncodedTensor&)>;

struct PlanStep {
    std::string op;
    uint64_t in_count = 0, in_dim = 0;
    std::string in_rep;
    CounterDelta predicted;
    StepFn run;
};

struct Plan {
    Strategy strategy = Strategy::LolaMnist;
    uint32_t n = 0;
    uint32_t depth_needed = 0;
    std::vector<PlanStep> steps;
    CounterDelta predicted_total;
    std::vector<uint64_t> live_entering;
    RepKind in_kind = RepKind::Dense;
    uint64_t in_messages = 0, in_length = 0;
    // device images [B][input_values] -> encoded input tensor
    std::function<EncodedTensor(Evaluator&, const int64_t* dev_images)> encode_input;
    uint64_t predicted_peak() const;
};

// PlanOptions (proj/include/packnn/plan.hpp:35-41): the degree is the
// context's, so only the window-matrix threshold is a free option here.
struct PlanOptions {
    // an interior window stage is realized as a row-major matrix when
    // window_volume * maps exceeds this; smaller ones are rejected
    uint64_t window_matrix_threshold = 100000;
};

// Host-only: builds the step table with exact predicted counters. Throws
// std::invalid_argument when the network does not fit the strategy.
Plan build_plan(const Network& net, Strategy s, uint32_t n, const PlanOptions& opt = PlanOptions{});

struct ExecutionResult {
    EncodedTensor output;
    std::vector<CounterDelta> per_step;
    CounterDelta total;
    uint64_t live_messages_peak = 0;
    uint32_t depth_consumed = 0;
};

// Runs the plan; std::logic_error when a step's counters deviate from the
// prediction (proj/src/plan.cpp:610-626).
ExecutionResult execute(const Plan& plan, EncodedTensor input, Evaluator& ev);

// Output scores of a sparse/dense result: device [B][values][4] words.
DeviceBuffer decode_values(Evaluator& ev, const EncodedTensor& t);

}  // namespace lb::lola
