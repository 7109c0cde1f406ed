// LoLa representations, packed kernels and plans over the device evaluator.
// Each function restates the reference's semantics (file:line cited) so the
// operation sequence — and therefore every counter — is identical; the
// payload work behind each counted op runs batched on the GPU.
#include <algorithm>
#include <mutex>
#include <numeric>
#include <stdexcept>

#include "lola_plan.hpp"

namespace lb::lola {

namespace {

void require(bool cond, const std::string& what) {
    if (!cond) throw std::invalid_argument(what);
}

uint64_t pad_for(uint64_t length) {  // representation.cpp:75-80
    require(length > 0, "empty vector");
    uint64_t p = 1;
    while (p < length) p <<= 1;
    return p;
}

uint32_t ctz64(uint64_t v) { return v ? static_cast<uint32_t>(__builtin_ctzll(v)) : 64; }

uint32_t shifted_slot(uint32_t slot, uint32_t offset, uint32_t half) {  // representation.cpp:19-23
    return slot / half * half + (slot % half + offset) % half;
}

// column shift by a signed amount counted as one rotation (representation.cpp:11-17)
Message bundle_signed(Evaluator& ev, const Message& m, int64_t shift) {
    const int64_t half = ev.context().half();
    int64_t a = shift % half;
    if (a < 0) a += half;
    return ev.rotate_bundle(m, static_cast<uint32_t>(a));
}

}  // namespace

std::string rep_name(RepKind kind, bool hybrid) {  // representation.cpp:31-42
    switch (kind) {
        case RepKind::Dense: return "dense";
        case RepKind::Sparse: return "sparse";
        case RepKind::Stacked: return hybrid ? "stacked-interleave" : "stacked";
        case RepKind::Interleaved: return "interleave";
        case RepKind::Convolution: return hybrid ? "convolution-interleave" : "convolution";
        case RepKind::Simd: return "simd";
    }
    return "?";
}

bool Representation::identity_layout() const {
    for (size_t i = 0; i < slot_of.size(); ++i)
        if (slot_of[i] != i) return false;
    return true;
}

uint32_t ConvGeometry::out_h() const {
    const uint32_t padded = in_h + pad_top + pad_bottom;
    require(padded >= win_h, "window taller than padded input");
    return (padded - win_h) / stride_h + 1;
}

uint32_t ConvGeometry::out_w() const {
    const uint32_t padded = in_w + pad_left + pad_right;
    require(padded >= win_w, "window wider than padded input");
    return (padded - win_w) / stride_w + 1;
}

// Source flat index of window offset j at window position w, or none when the
// tap falls into the zero padding (representation.cpp:62-73).
std::optional<uint32_t> ConvGeometry::tap(uint32_t j, uint32_t w) const {
    const uint32_t c = j / (win_h * win_w), dy = (j / win_w) % win_h, dx = j % win_w;
    const uint32_t a = w / out_w(), b = w % out_w();
    const int64_t y = int64_t(a) * stride_h + dy - pad_top;
    const int64_t x = int64_t(b) * stride_w + dx - pad_left;
    if (y < 0 || x < 0 || y >= in_h || x >= in_w) return std::nullopt;
    return c * in_h * in_w + uint32_t(y) * in_w + uint32_t(x);
}

namespace {

// ---- stream fan-out -------------------------------------------------------------------
// Independent op chains (rows of a row-major product, calls of the stacked
// product, output maps, per-message masks and squares) run on forked
// evaluators bound to the context's side streams: the GPU analogue of the
// reference's per-row thread fan-out with fork/absorb (kernels.cpp:161-195).
// Children start after the parent's queued work (event), the parent resumes
// after all children (events), counters are absorbed in child order, and
// messages produced by children are rebound to the parent stream so their
// frees are ordered after the parent's uses.
class FanOut {
public:
    FanOut(Evaluator& ev, uint64_t tasks) : ev_(ev) {
        const uint32_t S = static_cast<uint32_t>(std::min<uint64_t>(ev.context().fanout(), tasks));
        if (S <= 1) return;
        cudaEvent_t start;
        LB_CUDA(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
        LB_CUDA(cudaEventRecord(start, ev.stream()));
        for (uint32_t i = 0; i < S; ++i) {
            cudaStream_t st = ev.context().side_stream(i);
            LB_CUDA(cudaStreamWaitEvent(st, start, 0));
            kids_.push_back(ev.fork_on(st));
        }
        LB_CUDA(cudaEventDestroy(start));
    }
    Evaluator& operator[](uint64_t task) { return kids_.empty() ? ev_ : kids_[task % kids_.size()]; }
    uint32_t width() const { return kids_.empty() ? 1u : static_cast<uint32_t>(kids_.size()); }
    // join, then adopt the produced messages on the parent stream
    void join(std::vector<Message>& produced) {
        if (kids_.empty()) return;
        for (Evaluator& k : kids_) {
            cudaEvent_t done;
            LB_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
            LB_CUDA(cudaEventRecord(done, k.stream()));
            LB_CUDA(cudaStreamWaitEvent(ev_.stream(), done, 0));
            LB_CUDA(cudaEventDestroy(done));
            ev_.absorb(k);
        }
        for (Message& m : produced) m.payload->buf.rebind(ev_.stream());
        kids_.clear();
    }

private:
    Evaluator& ev_;
    std::vector<Evaluator> kids_;
};

// ---- encoders (input side; images already on the device) ------------------------

// encode_convolution (representation.cpp:131-165): message j carries the tap
// under window offset j at the layout slot of every window position.
EncodedTensor encode_convolution(Evaluator& ev, const int64_t* dev_images, uint64_t stride, const ConvGeometry& g,
                                 bool row_split, int64_t max_abs) {
    const uint32_t n = ev.context().n(), half = n / 2, positions = g.positions(), r = g.window_volume();
    require(positions <= n, "more window positions than slots");
    std::vector<uint32_t> layout(positions);
    const uint32_t split = (positions + 1) / 2;
    if (row_split) require(split <= half && positions - split <= half, "row split overflow");
    for (uint32_t w = 0; w < positions; ++w) layout[w] = (row_split && w >= split) ? half + (w - split) : w;
    EncodedTensor t;
    t.rep.kind = RepKind::Convolution;
    t.rep.length = positions;
    t.rep.windows = r;
    if (row_split) t.rep.slot_of = layout;
    std::vector<std::vector<int32_t>> maps(r, std::vector<int32_t>(n, -1));
    for (uint32_t j = 0; j < r; ++j)
        for (uint32_t w = 0; w < positions; ++w) {
            auto src = g.tap(j, w);
            if (src) maps[j][layout[w]] = static_cast<int32_t>(*src);
        }
    t.messages = ev.lift_gather_many(dev_images, stride, maps, max_abs);
    return t;
}

// encode_dense_image (representation.cpp:92-115): rows at a fixed stride.
EncodedTensor encode_dense_image(Evaluator& ev, const int64_t* dev_images, uint64_t stride, const ConvGeometry& g,
                                 uint32_t row_stride, int64_t max_abs) {
    require(row_stride >= g.in_w, "row stride narrower than image");
    const uint64_t span = uint64_t(g.channels) * g.in_h * row_stride;
    require(span <= ev.context().n(), "strided image exceeds slot count");
    std::vector<int32_t> map(span, -1);
    for (uint32_t c = 0; c < g.channels; ++c)
        for (uint32_t y = 0; y < g.in_h; ++y)
            for (uint32_t x = 0; x < g.in_w; ++x)
                map[uint64_t(c) * g.in_h * row_stride + uint64_t(y) * row_stride + x] =
                    static_cast<int32_t>(uint64_t(c) * g.in_h * g.in_w + uint64_t(y) * g.in_w + x);
    EncodedTensor t;
    t.rep.kind = RepKind::Dense;
    t.rep.length = span;
    t.rep.pad = pad_for(span);
    t.messages.push_back(ev.lift_gather(dev_images, stride, map, max_abs));
    return t;
}

EncodedTensor encode_dense(Evaluator& ev, const int64_t* dev_images, uint64_t stride, uint64_t length, int64_t max_abs) {
    require(length <= ev.context().n(), "vector longer than slot count");
    std::vector<int32_t> map(length);
    std::iota(map.begin(), map.end(), 0);
    EncodedTensor t;
    t.rep.kind = RepKind::Dense;
    t.rep.length = length;
    t.rep.pad = pad_for(length);
    t.messages.push_back(ev.lift_gather(dev_images, stride, map, max_abs));
    return t;
}

// ---- converters ----------------------------------------------------------------------

EncodedTensor stack_copies(Evaluator& ev, const EncodedTensor& t, uint32_t copies) {  // representation.cpp:225-259
    require(t.messages.size() == 1, "stacking expects a single message");
    require(t.rep.kind == RepKind::Dense || t.rep.kind == RepKind::Interleaved,
            "stacking expects a dense or interleaved layout");
    require(!t.rep.dirty, "stacking would duplicate dirty slots");
    require(copies >= 1 && (copies & (copies - 1)) == 0, "copies must be a power of two");
    const uint32_t n = ev.context().n(), half = n / 2;
    const uint64_t pad = t.rep.pad ? t.rep.pad : pad_for(t.rep.length);
    require(pad * copies <= n, "copies do not fit the message");
    std::vector<char> cls(pad, 0);
    for (uint64_t i = 0; i < t.rep.length; ++i) {
        const uint32_t s = t.rep.slot(i);
        require(s < half, "stacking layout must stay in slot row 0");
        require(!cls[s % pad], "layout collides with itself mod pad");
        cls[s % pad] = 1;
    }
    EncodedTensor out;
    out.rep = t.rep;
    out.rep.kind = RepKind::Stacked;
    out.rep.pad = pad;
    out.rep.copies = copies;
    Message m = t.messages[0];
    for (uint64_t shift = pad; shift < pad * copies; shift <<= 1)  // m = add(m, rotated m), fused
        m = shift == half ? ev.rotate_rows_add(m, m) : ev.rotate_bundle_add(m, m, static_cast<uint32_t>(shift));
    out.messages.push_back(std::move(m));
    return out;
}

EncodedTensor combine_to_one(Evaluator& ev, const EncodedTensor& parts, const std::vector<uint32_t>& offsets,
                             uint64_t logical_limit = 0) {  // representation.cpp:261-308
    require(!parts.messages.empty(), "nothing to combine");
    require(offsets.size() == parts.messages.size(), "one offset per part required");
    require(!parts.rep.dirty, "combining dirty parts would mix garbage");
    const uint32_t n = ev.context().n(), half = n / 2;
    const uint64_t per_part = parts.rep.length;
    uint64_t total = per_part * parts.messages.size();
    if (logical_limit) {
        require(logical_limit <= total, "limit exceeds combined length");
        total = logical_limit;
    }
    std::vector<char> used(n, 0);
    std::vector<uint32_t> slot_of(total);
    for (size_t p = 0; p < parts.messages.size(); ++p)
        for (uint64_t j = 0; j < per_part; ++j) {
            const uint32_t s = shifted_slot(parts.rep.slot(j), offsets[p], half);
            require(!used[s], "combined parts collide");
            used[s] = 1;
            const uint64_t idx = p * per_part + j;
            if (idx < total) slot_of[idx] = s;
        }
    Message acc = offsets[0] ? ev.rotate_bundle(parts.messages[0], offsets[0]) : parts.messages[0];
    for (size_t p = 1; p < parts.messages.size(); ++p)  // acc = add(acc, rotated part), fused
        acc = ev.rotate_bundle_add(acc, parts.messages[p], offsets[p]);
    EncodedTensor out;
    out.rep.kind = RepKind::Interleaved;
    out.rep.length = total;
    out.rep.pad = pad_for(total);
    out.rep.slot_of = std::move(slot_of);
    if (out.rep.identity_layout()) {
        out.rep.kind = RepKind::Dense;
        out.rep.slot_of.clear();
    }
    out.messages.push_back(std::move(acc));
    return out;
}

EncodedTensor sparse_to_dense(Evaluator& ev, const EncodedTensor& t) {  // representation.cpp:310-347
    require(t.rep.kind == RepKind::Sparse, "expected a sparse tensor");
    require(t.rep.broadcast, "only broadcast sparse values can be re-slotted");
    const uint32_t n = ev.context().n();
    require(t.rep.length <= n, "target slot out of range");
    // per-stream partial sums, then their sum: v masks and v - 1 additions
    // in any association, exactly as the reference counts them
    FanOut fan(ev, t.rep.length);
    const uint32_t S = fan.width();
    std::vector<Message> partial(S);
    std::vector<bool> started(S, false);
    for (uint64_t i = 0; i < t.rep.length; ++i) {
        std::vector<uint8_t> bits(n, 0);
        bits[i] = 1;
        Evaluator& e = fan[i];
        const uint32_t k = static_cast<uint32_t>(i % S);
        Message picked = e.mask(t.messages[i], bits);
        partial[k] = started[k] ? e.add(partial[k], picked) : picked;
        started[k] = true;
    }
    std::vector<Message> used;
    for (uint32_t k = 0; k < S; ++k)
        if (started[k]) used.push_back(partial[k]);
    fan.join(used);
    Message acc = used[0];
    for (size_t k = 1; k < used.size(); ++k) acc = ev.add(acc, used[k]);
    EncodedTensor out;
    out.rep.kind = RepKind::Dense;  // identity targets
    out.rep.length = t.rep.length;
    out.rep.pad = pad_for(t.rep.length);
    out.messages.push_back(std::move(acc));
    return out;
}

EncodedTensor mask_active(Evaluator& ev, const EncodedTensor& t) {  // representation.cpp:349-361
    require(t.rep.kind == RepKind::Dense || t.rep.kind == RepKind::Interleaved,
            "masking expects a dense or interleaved layout");
    require(!t.messages.empty() && t.rep.length > 0, "nothing to mask");
    std::vector<uint8_t> bits(ev.context().n(), 0);
    for (uint64_t i = 0; i < t.rep.length; ++i) bits[t.rep.slot(i)] = 1;
    EncodedTensor out;
    out.rep = t.rep;
    out.rep.dirty = false;
    FanOut fan(ev, t.messages.size());
    for (size_t i = 0; i < t.messages.size(); ++i) out.messages.push_back(fan[i].mask(t.messages[i], bits));
    fan.join(out.messages);
    return out;
}

std::vector<uint32_t> window_grid_slots(const ConvGeometry& g, uint32_t row_stride) {  // representation.cpp:380-388
    const uint32_t oh = g.out_h(), ow = g.out_w();
    std::vector<uint32_t> base(size_t(oh) * ow);
    for (uint32_t a = 0; a < oh; ++a)
        for (uint32_t b = 0; b < ow; ++b) base[size_t(a) * ow + b] = a * g.stride_h * row_stride + b * g.stride_w;
    return base;
}

// LoLa-Dense front end (representation.cpp:390-428)
EncodedTensor dense_to_convolution(Evaluator& ev, const EncodedTensor& d, const ConvGeometry& g, uint32_t row_stride) {
    require(d.messages.size() == 1 && d.rep.kind == RepKind::Dense, "mask source must be a single dense message");
    const uint32_t n = ev.context().n(), half = n / 2, r = g.window_volume(), positions = g.positions();
    const auto base = window_grid_slots(g, row_stride);
    EncodedTensor out;
    out.rep.kind = RepKind::Convolution;
    out.rep.length = positions;
    out.rep.windows = r;
    out.rep.slot_of = base;
    for (uint32_t j = 0; j < r; ++j) {
        const uint32_t c = j / (g.win_h * g.win_w), dy = (j / g.win_w) % g.win_h, dx = j % g.win_w;
        const int64_t offset = int64_t(c) * g.in_h * row_stride + (int64_t(dy) - g.pad_top) * row_stride +
                               (int64_t(dx) - g.pad_left);
        std::vector<uint8_t> bits(n, 0);
        bool any = false;
        for (uint32_t w = 0; w < positions; ++w) {
            if (!g.tap(j, w)) continue;
            const int64_t s = base[w] + offset;
            require(s >= 0 && s < half, "masked window leaves slot row 0");
            bits[uint32_t(s)] = 1;
            any = true;
        }
        require(any, "window offset reads only padding");
        Message picked = ev.mask(d.messages[0], bits);
        out.messages.push_back(offset != 0 ? bundle_signed(ev, picked, -offset) : std::move(picked));
    }
    return out;
}

struct MaskPacking {
    uint32_t row_stride;
    std::vector<uint32_t> map_shifts;
};

MaskPacking find_mask_packing(const ConvGeometry& g, uint32_t maps, uint64_t pad, uint32_t n) {  // representation.cpp:430-467
    const uint32_t half = n / 2;
    for (uint32_t stride = g.in_w; stride <= g.in_w + 256; ++stride) {
        if (uint64_t(g.channels) * g.in_h * stride > half) break;
        const auto base = window_grid_slots(g, stride);
        const uint32_t top = *std::max_element(base.begin(), base.end());
        std::vector<char> self(pad, 0);
        bool injective = true;
        for (uint32_t s : base) {
            if (self[s % pad]) {
                injective = false;
                break;
            }
            self[s % pad] = 1;
        }
        if (!injective) continue;
        std::vector<char> used(pad, 0);
        std::vector<uint32_t> shifts;
        for (uint64_t s = 0; s < pad && shifts.size() < maps; ++s) {
            if (top + s >= half) break;
            bool ok = true;
            for (uint32_t b : base)
                if (used[(b + s) % pad]) {
                    ok = false;
                    break;
                }
            if (!ok) continue;
            for (uint32_t b : base) used[(b + s) % pad] = 1;
            shifts.push_back(static_cast<uint32_t>(s));
        }
        if (shifts.size() == maps) return {stride, std::move(shifts)};
    }
    throw std::invalid_argument("no row stride packs the window grids disjointly");
}

std::vector<uint32_t> uniform_offsets(uint32_t parts, uint32_t stride) {
    std::vector<uint32_t> out(parts);
    for (uint32_t i = 0; i < parts; ++i) out[i] = i * stride;
    return out;
}

// ---- kernels and their cost models (kernels.cpp) ----------------------------------

uint64_t reduction_span(const Representation& rep, uint32_t n) {  // kernels.cpp:54-63
    require(rep.length > 0, "empty layout");
    uint32_t max_slot = 0;
    for (uint64_t i = 0; i < rep.length; ++i) max_slot = std::max(max_slot, rep.slot(i));
    require(max_slot < n, "layout slot out of range");
    return max_slot < n / 2 ? pad_for(max_slot + 1) : n;
}

CounterDelta dot_product_cost(uint32_t n, uint64_t span) {  // kernels.cpp:65-73
    const uint32_t stages = ctz64(span);
    CounterDelta d;
    d.ct_plain_mul = 1;
    d.rot_rows = (span == n && stages > 0) ? 1 : 0;
    d.rot_cols = stages - d.rot_rows;
    d.add = stages;
    return d;
}

CounterDelta scaled(const CounterDelta& one, uint64_t k) {
    CounterDelta d;
    d.ct_ct_mul = one.ct_ct_mul * k;
    d.ct_plain_mul = one.ct_plain_mul * k;
    d.scalar_mul = one.scalar_mul * k;
    d.mask_mul = one.mask_mul * k;
    d.add = one.add * k;
    d.rot_cols = one.rot_cols * k;
    d.rot_rows = one.rot_rows * k;
    return d;
}

CounterDelta matvec_rowmajor_cost(uint32_t n, uint64_t span, uint64_t rows) {
    return scaled(dot_product_cost(n, span), rows);
}

CounterDelta matvec_stacked_cost(uint32_t n, uint64_t pad, uint32_t copies, uint64_t rows) {  // kernels.cpp:92-102
    const uint64_t calls = (rows + copies - 1) / copies;
    const uint32_t stages = ctz64(pad);
    CounterDelta d;
    d.ct_plain_mul = calls;
    d.rot_rows = (pad == n && stages > 0) ? calls : 0;
    d.rot_cols = calls * stages - d.rot_rows;
    d.add = calls * stages;
    return d;
}

CounterDelta conv_rowmajor_cost(uint64_t maps, uint64_t windows) {
    CounterDelta d;
    d.scalar_mul = maps * windows;
    d.add = windows ? maps * (windows - 1) : 0;
    return d;
}

CounterDelta square_cost(uint64_t m) {
    CounterDelta d;
    d.ct_ct_mul = m;
    return d;
}

CounterDelta add_bias_cost(uint64_t m) {
    CounterDelta d;
    d.add = m;
    return d;
}

CounterDelta mask_active_cost(uint64_t m) {
    CounterDelta d;
    d.mask_mul = m;
    d.ct_plain_mul = m;
    return d;
}

CounterDelta combine_cost(const std::vector<uint32_t>& offsets, bool with_bias) {  // plan.cpp:147-153
    CounterDelta d;
    for (uint32_t o : offsets) d.rot_cols += o != 0;
    d.add = offsets.size() - 1 + (with_bias ? 1 : 0);
    return d;
}

CounterDelta stack_cost(uint32_t copies, bool fills_message) {  // plan.cpp:155-164
    CounterDelta d;
    const uint32_t steps = ctz64(copies);
    d.add = steps;
    d.rot_rows = fills_message ? 1 : 0;
    d.rot_cols = steps - d.rot_rows;
    return d;
}

CounterDelta sparse_to_dense_cost(uint64_t v) {
    CounterDelta d;
    d.mask_mul = v;
    d.ct_plain_mul = v;
    d.add = v - 1;
    return d;
}

// rotate-and-sum ladder of sizes 1, 2, ..., span/2 (kernels.cpp:26-36)
Message reduce_rotate_add(Evaluator& ev, Message m, uint64_t span, bool toward_low) {
    const uint32_t half = ev.context().half();
    for (uint64_t size = 1; size < span; size <<= 1)  // m = add(m, rotated m), fused
        m = size == half ? ev.rotate_rows_add(m, m)
                         : ev.rotate_columns_add(m, m, toward_low ? -int64_t(size) : int64_t(size));
    return m;
}

Message dot_product(Evaluator& ev, const Message& v, const std::vector<int64_t>& w_by_slot, uint64_t span) {
    const uint32_t n = ev.context().n();
    require(span >= 1 && (span & (span - 1)) == 0 && span <= n, "bad reduction span");
    require(w_by_slot.size() == n, "weights must cover every slot");
    return reduce_rotate_add(ev, ev.mul_plain(v, w_by_slot), span, true);
}

EncodedTensor matvec_rowmajor(Evaluator& ev, const EncodedTensor& x, const Weights& W) {  // kernels.cpp:145-196
    require(x.messages.size() == 1, "row-major multiply expects a single message");
    require(x.rep.kind == RepKind::Dense || x.rep.kind == RepKind::Interleaved,
            "row-major multiply expects a dense or interleaved vector");
    require(W.at && W.rows >= 1, "missing weights");
    require(W.cols == x.rep.length, "weight columns do not match vector length");
    const uint32_t n = ev.context().n();
    const uint64_t span = reduction_span(x.rep, n);
    EncodedTensor out;
    out.rep.kind = RepKind::Sparse;
    out.rep.length = W.rows;
    out.rep.broadcast = span == n;
    out.rep.value_slot = 0;
    out.rep.dirty = !out.rep.broadcast;
    std::vector<int64_t> w(n);
    FanOut fan(ev, W.rows);
    for (uint64_t row = 0; row < W.rows; ++row) {
        std::fill(w.begin(), w.end(), 0);
        for (uint64_t i = 0; i < W.cols; ++i) w[x.rep.slot(i)] = W.at(row, i);
        out.messages.push_back(dot_product(fan[row], x.messages[0], w, span));
    }
    fan.join(out.messages);
    return out;
}

EncodedTensor matvec_stacked_rowmajor(Evaluator& ev, const EncodedTensor& x, const Weights& W) {  // kernels.cpp:223-267
    require(x.rep.kind == RepKind::Stacked && x.messages.size() == 1, "stacked multiply expects a single stacked message");
    require(W.at && W.rows >= 1, "missing weights");
    require(W.cols == x.rep.length, "weight columns do not match vector length");
    const uint32_t n = ev.context().n();
    const uint64_t pad = x.rep.pad;
    const uint32_t copies = x.rep.copies;
    require(pad >= 2 && (pad & (pad - 1)) == 0, "bad stacked pad");
    require(uint64_t(copies) * pad == n, "stacked vector must fill the message");
    std::vector<char> cls(pad, 0);
    for (uint64_t i = 0; i < x.rep.length; ++i) {
        const uint32_t c = x.rep.slot(i) & (pad - 1);
        require(!cls[c], "stacked layout collides mod pad");
        cls[c] = 1;
    }
    const uint64_t calls = (W.rows + copies - 1) / copies;
    EncodedTensor out;
    out.rep.kind = RepKind::Interleaved;
    out.rep.length = copies;
    out.rep.pad = pad_for(copies);
    out.rep.dirty = true;
    out.rep.slot_of.resize(copies);
    for (uint32_t d = 0; d < copies; ++d) out.rep.slot_of[d] = static_cast<uint32_t>((d + 1) * pad - 1);
    std::vector<int64_t> w(n);
    FanOut fan(ev, calls);
    for (uint64_t c = 0; c < calls; ++c) {
        std::fill(w.begin(), w.end(), 0);
        for (uint32_t d = 0; d < copies; ++d) {
            const uint64_t row = c * copies + d;
            if (row >= W.rows) break;
            for (uint64_t i = 0; i < W.cols; ++i) w[d * pad + (x.rep.slot(i) & (pad - 1))] = W.at(row, i);
        }
        Evaluator& e = fan[c];
        out.messages.push_back(reduce_rotate_add(e, e.mul_plain(x.messages[0], w), pad, false));
    }
    fan.join(out.messages);
    return out;
}

// A stage's full row-major matrix, materialised once per plan (host for the
// magnitude bookkeeping, device for the kernel).
struct SimdMatrix {
    uint64_t rows = 0, cols = 0;
    std::vector<int64_t> host;
    DeviceBuffer dev;
    std::mutex mu;
};

void materialise(Evaluator& ev, const Weights& W, SimdMatrix& M) {
    std::lock_guard<std::mutex> lock(M.mu);
    if (M.dev.get()) return;
    M.rows = W.rows;
    M.cols = W.cols;
    M.host.resize(W.rows * W.cols);
    for (uint64_t r = 0; r < W.rows; ++r)
        for (uint64_t c = 0; c < W.cols; ++c) M.host[r * W.cols + c] = W.at(r, c);
    cudaStream_t s = ev.stream();
    M.dev = DeviceBuffer(M.host.size() * 8, s);
    LB_CUDA(cudaMemcpyAsync(M.dev.get(), M.host.data(), M.host.size() * 8, cudaMemcpyHostToDevice, s));
    LB_CUDA(cudaStreamSynchronize(s));
    M.dev.rebind(nullptr);  // outlives the session's streams
}

// Every output map is sum_j W[map][j] * window_j (the reference's
// mul_scalar + add chain per map, same counters, depths and magnitude checks:
// Evaluator::weighted_sums replays the chain where a bound would trip); all
// maps run as one pass over the window messages instead of a
// read-modify-write of the accumulator per term.
EncodedTensor conv_rowmajor(Evaluator& ev, const EncodedTensor& x, const Weights& W, SimdMatrix& M) {  // kernels.cpp:269-292
    require(x.rep.kind == RepKind::Convolution, "expected a convolution tensor");
    require(x.messages.size() == x.rep.windows && x.rep.windows >= 1, "window count does not match messages");
    require(W.at && W.rows >= 1, "missing weights");
    require(W.cols == x.rep.windows, "weight columns do not match window count");
    EncodedTensor out;
    out.rep.kind = RepKind::Interleaved;
    out.rep.length = x.rep.length;
    out.rep.pad = pad_for(x.rep.length);
    out.rep.slot_of = x.rep.slot_of;
    if (out.rep.identity_layout()) {
        out.rep.kind = RepKind::Dense;
        out.rep.slot_of.clear();
    }
    materialise(ev, W, M);
    bool small = true;  // weighted_sums' 128-bit bookkeeping takes |w| < 2^31
    for (int64_t w : M.host) small = small && w > -(int64_t(1) << 31) && w < (int64_t(1) << 31);
    if (small) {
        out.messages = ev.weighted_sums(x.messages, W.rows, M.host.data(), M.dev.get<int64_t>());
        return out;
    }
    FanOut fan(ev, W.rows);
    for (uint64_t map = 0; map < W.rows; ++map) {
        Evaluator& e = fan[map];
        Message acc = e.mul_scalar(x.messages[0], W.at(map, 0));
        for (uint64_t j = 1; j < W.cols; ++j)  // acc = add(acc, mul_scalar(x_j, w)), fused
            acc = e.mul_scalar_add(acc, x.messages[j], W.at(map, j));
        out.messages.push_back(std::move(acc));
    }
    fan.join(out.messages);
    return out;
}

EncodedTensor square_activation(Evaluator& ev, const EncodedTensor& x) {  // kernels.cpp:294-300
    require(!x.messages.empty(), "empty tensor");
    EncodedTensor out;
    out.rep = x.rep;
    FanOut fan(ev, x.messages.size());
    for (size_t i = 0; i < x.messages.size(); ++i) out.messages.push_back(fan[i].mul(x.messages[i], x.messages[i]));
    fan.join(out.messages);
    return out;
}

EncodedTensor add_bias(Evaluator& ev, const EncodedTensor& x, const std::vector<int64_t>& bias) {  // kernels.cpp:320-354
    require(!x.messages.empty(), "empty tensor");
    const uint32_t n = ev.context().n();
    EncodedTensor out;
    out.rep = x.rep;
    if (x.rep.kind == RepKind::Sparse) {
        require(bias.size() == x.messages.size(), "one bias per message required");
        std::vector<int64_t> b(n);
        FanOut fan(ev, x.messages.size());
        for (size_t i = 0; i < x.messages.size(); ++i) {
            std::fill(b.begin(), b.end(), 0);
            if (x.rep.broadcast)
                std::fill(b.begin(), b.end(), bias[i]);
            else
                b[x.rep.value_slot] = bias[i];
            out.messages.push_back(fan[i].add_plain(x.messages[i], b));
        }
        fan.join(out.messages);
        return out;
    }
    if (x.rep.kind == RepKind::Simd) {
        // bias of message i in the slots of every record (kernels.cpp:338-346)
        require(bias.size() == x.messages.size(), "one bias per message required");
        FanOut fan(ev, x.messages.size());
        std::vector<int64_t> b(n, 0);
        for (size_t i = 0; i < x.messages.size(); ++i) {
            std::fill(b.begin(), b.begin() + x.rep.copies, bias[i]);
            out.messages.push_back(fan[i].add_plain(x.messages[i], b));
        }
        fan.join(out.messages);
        return out;
    }
    require(x.messages.size() == 1, "per-value bias needs a single message");
    require(bias.size() == x.rep.length, "one bias per value required");
    std::vector<int64_t> b(n, 0);
    for (uint64_t i = 0; i < x.rep.length; ++i) b[x.rep.slot(i)] = bias[i];
    out.messages.push_back(ev.add_plain(x.messages[0], b));
    return out;
}

// ---- record (SIMD) tensors -----------------------------------------------------------

// One message per feature; slot r of message j = record r's feature j
// (representation.cpp:167-183). The records are the session's images, packed
// into the slots of a single batch entry.
EncodedTensor encode_simd(Evaluator& ev, const int64_t* dev_images, uint64_t features, int64_t max_abs) {
    const uint32_t recs = ev.context().records();
    require(ev.context().batch() == 1, "record tensors pack the records into the slots of one message");
    require(recs >= 1 && recs <= ev.context().n(), "more records than slots");
    require(uint64_t(recs) * features < (1ull << 31), "record tensor too large");
    EncodedTensor t;
    t.rep.kind = RepKind::Simd;
    t.rep.length = features;
    t.rep.copies = recs;
    // in groups (the gathered slot values of a group are staged at once)
    constexpr uint64_t kGroup = 64;
    for (uint64_t j0 = 0; j0 < features; j0 += kGroup) {
        std::vector<std::vector<int32_t>> maps;
        for (uint64_t j = j0; j < std::min(features, j0 + kGroup); ++j) {
            std::vector<int32_t> map(recs);
            for (uint32_t r = 0; r < recs; ++r) map[r] = static_cast<int32_t>(uint64_t(r) * features + j);
            maps.push_back(std::move(map));
        }
        for (Message& m : ev.lift_gather_many(dev_images, features, maps, max_abs)) t.messages.push_back(std::move(m));
    }
    return t;
}

EncodedTensor simd_dense(Evaluator& ev, const EncodedTensor& x, const Weights& W, SimdMatrix& M) {  // kernels.cpp:302-318
    require(x.rep.kind == RepKind::Simd, "expected a record tensor");
    require(x.messages.size() == x.rep.length && x.rep.length >= 1, "bad record tensor");
    require(W.at && W.rows >= 1, "missing weights");
    require(W.cols == x.rep.length, "weight columns do not match feature count");
    materialise(ev, W, M);
    EncodedTensor out;
    out.rep = x.rep;
    out.rep.length = W.rows;
    out.messages = ev.weighted_sums(x.messages, W.rows, M.host.data(), M.dev.get<int64_t>());
    return out;
}

// ---- plans (plan.cpp) ---------------------------------------------------------------

struct Probe {
    uint64_t count = 0, dim = 0;
    std::string rep;
};

Probe probe_of(const EncodedTensor& t) {  // plan.cpp:104-115
    Probe p;
    p.count = t.messages.size();
    switch (t.rep.kind) {
        case RepKind::Sparse: p.dim = 1; break;
        case RepKind::Simd: p.dim = t.rep.copies; break;
        case RepKind::Stacked: p.dim = t.rep.length * t.rep.copies; break;
        default: p.dim = t.rep.length; break;
    }
    p.rep = rep_name(t.rep.kind, !t.rep.identity_layout());
    return p;
}

std::vector<int64_t> output_bias(const Stage& s) {  // plan.cpp:42-53
    std::vector<int64_t> b(s.out_shape.values(), 0);
    if (s.bias.empty()) return b;
    if (s.is_conv) {
        const uint64_t positions = s.geom.positions();
        for (uint64_t i = 0; i < b.size(); ++i) b[i] = s.bias[i / positions];
    } else {
        for (uint64_t i = 0; i < s.bias.size() && i < b.size(); ++i) b[i] = s.bias[i];
    }
    return b;
}

Weights window_rows(const Stage& s) {
    return {s.rows, s.cols, [&s](uint64_t m, uint64_t j) { return s.w(m, j); }};
}

// any stage as a flat matrix over the flattened input (plan.cpp:63-87)
Weights matrix_rows(const Stage& s) {
    if (!s.is_conv) return {s.rows, s.cols, [&s](uint64_t r, uint64_t c) { return s.w(r, c); }};
    const ConvGeometry g = s.geom;
    const uint64_t positions = g.positions(), plane = uint64_t(g.in_h) * g.in_w;
    return {s.out_shape.values(), s.in_shape.values(), [&s, g, positions, plane](uint64_t row, uint64_t col) -> int64_t {
                const uint64_t m = row / positions;
                const uint32_t pos = static_cast<uint32_t>(row % positions);
                const int64_t oy = pos / g.out_w(), ox = pos % g.out_w();
                const uint64_t cin = col / plane;
                const int64_t y = static_cast<int64_t>((col % plane) / g.in_w);
                const int64_t x = static_cast<int64_t>(col % g.in_w);
                const int64_t dy = y - (oy * g.stride_h - g.pad_top);
                const int64_t dx = x - (ox * g.stride_w - g.pad_left);
                if (dy < 0 || dy >= g.win_h || dx < 0 || dx >= g.win_w) return 0;
                return s.w(m, (cin * g.win_h + uint64_t(dy)) * g.win_w + uint64_t(dx));
            }};
}

void add_step(Plan& plan, uint64_t in_count, uint64_t in_dim, std::string in_rep, std::string op,
              const CounterDelta& predicted, StepFn run) {
    PlanStep st;
    st.op = std::move(op);
    st.in_count = in_count;
    st.in_dim = in_dim;
    st.in_rep = std::move(in_rep);
    st.predicted = predicted;
    st.run = std::move(run);
    plan.live_entering.push_back(in_count);
    plan.predicted_total += predicted;
    plan.steps.push_back(std::move(st));
}

std::string num(uint64_t v) { return std::to_string(v); }

void require_lola_shape(const Network& net) {  // plan.cpp:138-145
    require(net.stages.size() == 3, "strategy expects three linear stages");
    require(net.squares_after.size() == 3, "malformed network");
    require(net.squares_after[0] == 1 && net.squares_after[1] == 1 && net.squares_after[2] == 0,
            "strategy expects squarings after the first and second stages only");
    require(net.stages[0].is_conv, "strategy expects a window first stage");
    require(!net.stages[2].is_conv, "strategy expects a matrix final stage");
}

// shared tail of the lola-mnist presets (plan.cpp:177-238)
void add_lola_tail(Plan& plan, const Network& net, uint32_t n, uint64_t combined, const std::string& vec_rep,
                   bool hybrid_stack, uint64_t r1, uint64_t r2) {
    const uint64_t pad = pad_for(combined);
    require(2 * pad <= n, "stacked layer wider than the message degree");
    const uint32_t copies = static_cast<uint32_t>(n / pad);
    const uint64_t calls = (r1 + copies - 1) / copies;
    const Network* np = &net;
    add_step(plan, 1, combined, vec_rep, "square", square_cost(1),
             [](Evaluator& ev, const EncodedTensor& x) { return square_activation(ev, x); });
    add_step(plan, 1, combined, vec_rep, "stack " + num(copies) + " copies", stack_cost(copies, true),
             [copies](Evaluator& ev, const EncodedTensor& x) { return stack_copies(ev, x, copies); });
    add_step(plan, 1, combined * copies, rep_name(RepKind::Stacked, hybrid_stack),
             "stacked row-major products, " + num(calls) + " calls of " + num(copies) + " rows",
             matvec_stacked_cost(n, pad, copies, r1), [np](Evaluator& ev, const EncodedTensor& x) {
                 return matvec_stacked_rowmajor(ev, x, matrix_rows(np->stages[1]));
             });
    const std::vector<uint32_t> call_offsets = uniform_offsets(static_cast<uint32_t>(calls), 1);
    CounterDelta recombine = mask_active_cost(calls);
    recombine += combine_cost(call_offsets, true);
    add_step(plan, calls, copies, rep_name(RepKind::Interleaved),
             "mask and combine " + num(calls) + " messages into one", recombine,
             [np, call_offsets, r1](Evaluator& ev, const EncodedTensor& x) {
                 EncodedTensor t = mask_active(ev, x);
                 t = combine_to_one(ev, t, call_offsets, r1);
                 return add_bias(ev, t, output_bias(np->stages[1]));
             });
    add_step(plan, 1, r1, rep_name(RepKind::Interleaved), "square", square_cost(1),
             [](Evaluator& ev, const EncodedTensor& x) { return square_activation(ev, x); });
    const uint32_t half = n / 2;
    uint64_t max_slot = 0;
    for (uint64_t d = 0; d < r1; ++d) {
        const uint64_t base = (d % copies + 1) * pad - 1;
        max_slot = std::max(max_slot, base / half * half + (base % half + d / copies) % half);
    }
    const uint64_t fc_span = max_slot < half ? pad_for(max_slot + 1) : n;
    CounterDelta fc = matvec_rowmajor_cost(n, fc_span, r2);
    fc += add_bias_cost(r2);
    add_step(plan, 1, r1, rep_name(RepKind::Interleaved), "row-major products, " + num(r2) + " rows", fc,
             [np](Evaluator& ev, const EncodedTensor& x) {
                 EncodedTensor t = matvec_rowmajor(ev, x, matrix_rows(np->stages[2]));
                 return add_bias(ev, t, output_bias(np->stages[2]));
             });
}

void build_lola_mnist(Plan& plan, const Network& net, uint32_t n) {  // plan.cpp:240-286
    require_lola_shape(net);
    require(!net.stages[1].is_conv, "strategy expects a matrix second stage");
    const Stage& s0 = net.stages[0];
    const ConvGeometry g = s0.geom;
    const uint64_t p = g.positions(), v = g.window_volume(), maps = s0.rows, combined = maps * p;
    require(net.stages[1].cols == combined, "second stage does not match the window outputs");
    const uint64_t r1 = net.stages[1].rows;
    require(net.stages[2].cols == r1, "final stage does not match the second");
    const uint64_t r2 = net.stages[2].rows;
    require(combined >= 2, "strategy needs at least two window outputs");
    require(combined <= n / 2, "combined window outputs do not fit slot row 0");
    const Network* np = &net;
    plan.in_kind = RepKind::Convolution;
    plan.in_messages = v;
    plan.in_length = p;
    const uint64_t stride = s0.in_shape.values();
    const int64_t bound = net.input_bound;
    plan.encode_input = [g, stride, bound](Evaluator& ev, const int64_t* imgs) {
        return encode_convolution(ev, imgs, stride, g, false, bound);
    };
    add_step(plan, v, p, rep_name(RepKind::Convolution), "weighted sum of window messages per map",
             conv_rowmajor_cost(maps, v),
             [np, M = std::make_shared<SimdMatrix>()](Evaluator& ev, const EncodedTensor& x) {
                 return conv_rowmajor(ev, x, window_rows(np->stages[0]), *M);
             });
    const auto offsets = uniform_offsets(static_cast<uint32_t>(maps), static_cast<uint32_t>(p));
    add_step(plan, maps, p, rep_name(RepKind::Dense), "combine " + num(maps) + " messages into one",
             combine_cost(offsets, true), [np, offsets](Evaluator& ev, const EncodedTensor& x) {
                 return add_bias(ev, combine_to_one(ev, x, offsets), output_bias(np->stages[0]));
             });
    add_lola_tail(plan, net, n, combined, rep_name(RepKind::Dense), false, r1, r2);
    plan.depth_needed = 2;
    plan.live_entering.push_back(r2);
}

void build_lola_dense_mnist(Plan& plan, const Network& net, uint32_t n) {  // plan.cpp:288-362
    require_lola_shape(net);
    require(!net.stages[1].is_conv, "strategy expects a matrix second stage");
    const Stage& s0 = net.stages[0];
    const ConvGeometry g = s0.geom;
    const uint64_t p = g.positions(), v = g.window_volume(), maps = s0.rows, combined = maps * p;
    require(net.stages[1].cols == combined, "second stage does not match the window outputs");
    const uint64_t r1 = net.stages[1].rows;
    require(net.stages[2].cols == r1, "final stage does not match the second");
    const uint64_t r2 = net.stages[2].rows;
    require(combined >= 2, "strategy needs at least two window outputs");
    const uint64_t pad = pad_for(combined);
    require(2 * pad <= n, "stacked layer wider than the message degree");
    const MaskPacking packing = find_mask_packing(g, static_cast<uint32_t>(maps), pad, n);
    const std::vector<uint32_t> base = window_grid_slots(g, packing.row_stride);
    const Network* np = &net;
    plan.in_kind = RepKind::Dense;
    plan.in_messages = 1;
    plan.in_length = uint64_t(g.channels) * g.in_h * packing.row_stride;
    const uint32_t row_stride = packing.row_stride;
    const uint64_t stride = s0.in_shape.values();
    const int64_t bound = net.input_bound;
    plan.encode_input = [g, row_stride, stride, bound](Evaluator& ev, const int64_t* imgs) {
        return encode_dense_image(ev, imgs, stride, g, row_stride, bound);
    };
    CounterDelta carve;
    carve.mask_mul = v;
    carve.ct_plain_mul = v;
    carve.rot_cols = v - 1;
    add_step(plan, 1, s0.in_shape.values(), rep_name(RepKind::Dense), "mask input to create " + num(v) + " messages",
             carve, [g, row_stride](Evaluator& ev, const EncodedTensor& x) {
                 return dense_to_convolution(ev, x, g, row_stride);
             });
    bool grid_identity = true;
    for (size_t i = 0; i < base.size(); ++i) grid_identity &= base[i] == i;
    add_step(plan, v, p, rep_name(RepKind::Convolution, !grid_identity), "weighted sum of window messages per map",
             conv_rowmajor_cost(maps, v),
             [np, M = std::make_shared<SimdMatrix>()](Evaluator& ev, const EncodedTensor& x) {
                 return conv_rowmajor(ev, x, window_rows(np->stages[0]), *M);
             });
    const std::vector<uint32_t> shifts = packing.map_shifts;
    add_step(plan, maps, p, rep_name(grid_identity ? RepKind::Dense : RepKind::Interleaved),
             "combine " + num(maps) + " messages into one", combine_cost(shifts, true),
             [np, shifts](Evaluator& ev, const EncodedTensor& x) {
                 return add_bias(ev, combine_to_one(ev, x, shifts), output_bias(np->stages[0]));
             });
    const uint32_t half = n / 2;
    bool combined_identity = true;
    for (uint64_t m = 0; m < maps; ++m)
        for (uint64_t w = 0; w < p; ++w) combined_identity &= (base[w] + shifts[m]) % half == m * p + w;
    add_lola_tail(plan, net, n, combined, rep_name(combined_identity ? RepKind::Dense : RepKind::Interleaved),
                  !combined_identity, r1, r2);
    plan.depth_needed = 2;
    plan.live_entering.push_back(r2);
}

void build_lola_cifar(Plan& plan, const Network& net, uint32_t n, const PlanOptions& opt) {  // plan.cpp:364-462
    require_lola_shape(net);
    const Stage& s0 = net.stages[0];
    const Stage& s1 = net.stages[1];
    const ConvGeometry g = s0.geom;
    const uint64_t p = g.positions(), v = g.window_volume(), maps = s0.rows, combined = maps * p;
    require(p >= 2, "strategy needs at least two window positions per map");
    if (s1.is_conv)
        require(uint64_t(s1.geom.window_volume()) * s1.rows > opt.window_matrix_threshold,
                "interior window stage below the matrix threshold has no packed route");
    require(s1.is_conv ? s1.in_shape.values() == combined : s1.cols == combined,
            "second stage does not match the window outputs");
    const uint64_t mid = s1.out_shape.values();
    require(net.stages[2].cols == mid, "final stage does not match the second");
    const uint64_t r2 = net.stages[2].rows;
    const uint32_t half = n / 2;
    const uint32_t split = static_cast<uint32_t>((p + 1) / 2);
    require(maps * split <= half, "combined map outputs do not fit the slot rows");
    require(mid <= n, "second stage outputs do not fit one message");
    const bool split_identity = split == half;
    const std::string part_rep = rep_name(split_identity ? RepKind::Dense : RepKind::Interleaved);
    const std::string vec_rep = rep_name(split_identity && maps == 1 ? RepKind::Dense : RepKind::Interleaved);
    const Network* np = &net;
    plan.in_kind = RepKind::Convolution;
    plan.in_messages = v;
    plan.in_length = p;
    const uint64_t stride = s0.in_shape.values();
    const int64_t bound = net.input_bound;
    plan.encode_input = [g, stride, bound](Evaluator& ev, const int64_t* imgs) {
        return encode_convolution(ev, imgs, stride, g, true, bound);
    };
    add_step(plan, v, p, rep_name(RepKind::Convolution, !split_identity), "weighted sum of window messages per map",
             conv_rowmajor_cost(maps, v),
             [np, M = std::make_shared<SimdMatrix>()](Evaluator& ev, const EncodedTensor& x) {
                 return conv_rowmajor(ev, x, window_rows(np->stages[0]), *M);
             });
    const auto offsets = uniform_offsets(static_cast<uint32_t>(maps), split);
    add_step(plan, maps, p, part_rep, "combine " + num(maps) + " messages into one", combine_cost(offsets, true),
             [np, offsets](Evaluator& ev, const EncodedTensor& x) {
                 return add_bias(ev, combine_to_one(ev, x, offsets), output_bias(np->stages[0]));
             });
    add_step(plan, 1, combined, vec_rep, "square", square_cost(1),
             [](Evaluator& ev, const EncodedTensor& x) { return square_activation(ev, x); });
    CounterDelta mv = matvec_rowmajor_cost(n, n, mid);
    mv += add_bias_cost(mid);
    add_step(plan, 1, combined, vec_rep, "row-major products, " + num(mid) + " rows", mv,
             [np](Evaluator& ev, const EncodedTensor& x) {
                 EncodedTensor t = matvec_rowmajor(ev, x, matrix_rows(np->stages[1]));
                 return add_bias(ev, t, output_bias(np->stages[1]));
             });
    add_step(plan, mid, 1, rep_name(RepKind::Sparse), "place sparse values into one dense message",
             sparse_to_dense_cost(mid), [](Evaluator& ev, const EncodedTensor& x) { return sparse_to_dense(ev, x); });
    add_step(plan, 1, mid, rep_name(RepKind::Dense), "square", square_cost(1),
             [](Evaluator& ev, const EncodedTensor& x) { return square_activation(ev, x); });
    const uint64_t span = mid <= half ? pad_for(mid) : n;
    CounterDelta fc = matvec_rowmajor_cost(n, span, r2);
    fc += add_bias_cost(r2);
    add_step(plan, 1, mid, rep_name(RepKind::Dense), "row-major products, " + num(r2) + " rows", fc,
             [np](Evaluator& ev, const EncodedTensor& x) {
                 EncodedTensor t = matvec_rowmajor(ev, x, matrix_rows(np->stages[2]));
                 return add_bias(ev, t, output_bias(np->stages[2]));
             });
    plan.depth_needed = 2;
    plan.live_entering.push_back(r2);
}

// LoLa-Small (BASELINE config 3; the reference has no preset — the
// three-stage check at plan.cpp:138-145 rejects two-stage nets): windows in
// convolution representation, weighted sums, combine the maps into one
// message, bias, square, one row-major product per output, bias. The chain is
// the reference's own kernels in that order (oracle/ref_shim.cpp runs the
// same chain on the reference for parity).
void build_lola_small(Plan& plan, const Network& net, uint32_t n) {
    require(net.stages.size() == 2, "lola-small expects two linear stages");
    require(net.squares_after.size() == 2 && net.squares_after[0] == 1 && net.squares_after[1] == 0,
            "lola-small expects one squaring after the first stage");
    require(net.stages[0].is_conv && !net.stages[1].is_conv, "lola-small expects window + matrix stages");
    const Stage& s0 = net.stages[0];
    const ConvGeometry g = s0.geom;
    const uint64_t p = g.positions(), v = g.window_volume(), maps = s0.rows, combined = maps * p;
    require(net.stages[1].cols == combined, "second stage does not match the window outputs");
    require(combined <= n / 2, "combined window outputs do not fit slot row 0");
    const uint64_t rows = net.stages[1].rows;
    const Network* np = &net;
    plan.in_kind = RepKind::Convolution;
    plan.in_messages = v;
    plan.in_length = p;
    const uint64_t stride = s0.in_shape.values();
    const int64_t bound = net.input_bound;
    plan.encode_input = [g, stride, bound](Evaluator& ev, const int64_t* imgs) {
        return encode_convolution(ev, imgs, stride, g, false, bound);
    };
    add_step(plan, v, p, rep_name(RepKind::Convolution), "weighted sum of window messages per map",
             conv_rowmajor_cost(maps, v),
             [np, M = std::make_shared<SimdMatrix>()](Evaluator& ev, const EncodedTensor& x) {
                 return conv_rowmajor(ev, x, window_rows(np->stages[0]), *M);
             });
    const auto offsets = uniform_offsets(static_cast<uint32_t>(maps), static_cast<uint32_t>(p));
    add_step(plan, maps, p, rep_name(RepKind::Dense), "combine " + num(maps) + " messages into one",
             combine_cost(offsets, true), [np, offsets](Evaluator& ev, const EncodedTensor& x) {
                 return add_bias(ev, combine_to_one(ev, x, offsets), output_bias(np->stages[0]));
             });
    add_step(plan, 1, combined, rep_name(RepKind::Dense), "square", square_cost(1),
             [](Evaluator& ev, const EncodedTensor& x) { return square_activation(ev, x); });
    CounterDelta fc = matvec_rowmajor_cost(n, pad_for(combined), rows);
    fc += add_bias_cost(rows);
    add_step(plan, 1, combined, rep_name(RepKind::Dense), "row-major products, " + num(rows) + " rows", fc,
             [np](Evaluator& ev, const EncodedTensor& x) {
                 EncodedTensor t = matvec_rowmajor(ev, x, matrix_rows(np->stages[1]));
                 return add_bias(ev, t, output_bias(np->stages[1]));
             });
    plan.depth_needed = 1;
    plan.live_entering.push_back(rows);
}

CounterDelta simd_dense_cost(uint64_t nodes, uint64_t fan_in) {  // kernels.cpp:116-121
    CounterDelta d;
    d.scalar_mul = nodes * fan_in;
    d.add = fan_in ? nodes * (fan_in - 1) : 0;
    return d;
}

void build_cryptonets_simd(Plan& plan, const Network& net) {  // plan.cpp:464-502
    require(!net.stages.empty(), "empty network");
    require(net.squares_after.size() == net.stages.size(), "malformed network");
    plan.in_kind = RepKind::Simd;
    plan.in_messages = net.stages[0].in_shape.values();
    plan.in_length = plan.in_messages;
    const uint64_t features = plan.in_messages;
    const int64_t bound = net.input_bound;
    plan.encode_input = [features, bound](Evaluator& ev, const int64_t* imgs) {
        return encode_simd(ev, imgs, features, bound);
    };
    const Network* np = &net;
    uint32_t depth = 0;
    for (size_t k = 0; k < net.stages.size(); ++k) {
        const uint64_t fan_in = net.stages[k].in_shape.values();
        const uint64_t nodes = net.stages[k].out_shape.values();
        CounterDelta d = simd_dense_cost(nodes, fan_in);
        d += add_bias_cost(nodes);
        auto M = std::make_shared<SimdMatrix>();
        add_step(plan, fan_in, 1, rep_name(RepKind::Simd), "per-value weighted sums, " + num(nodes) + " outputs", d,
                 [np, k, M](Evaluator& ev, const EncodedTensor& x) {
                     EncodedTensor t = simd_dense(ev, x, matrix_rows(np->stages[k]), *M);
                     return add_bias(ev, t, output_bias(np->stages[k]));
                 });
        for (uint32_t q = 0; q < net.squares_after[k]; ++q) {
            add_step(plan, nodes, 1, rep_name(RepKind::Simd), "square every message", square_cost(nodes),
                     [](Evaluator& ev, const EncodedTensor& x) { return square_activation(ev, x); });
            depth += 1;
        }
    }
    plan.depth_needed = depth;
    plan.live_entering.push_back(net.stages.back().out_shape.values());
}

void build_linear_features(Plan& plan, const Network& net, uint32_t n) {  // plan.cpp:505-539
    require(net.stages.size() == 1 && !net.stages[0].is_conv, "strategy expects a single matrix stage");
    require(net.squares_after.size() == 1 && net.squares_after[0] == 0, "strategy expects no squarings");
    const uint64_t cols = net.stages[0].cols, rows = net.stages[0].rows;
    require(cols <= n, "feature vector does not fit one message");
    const Network* np = &net;
    plan.in_kind = RepKind::Dense;
    plan.in_messages = 1;
    plan.in_length = cols;
    const int64_t bound = net.input_bound;
    plan.encode_input = [cols, bound](Evaluator& ev, const int64_t* imgs) {
        return encode_dense(ev, imgs, cols, cols, bound);
    };
    const uint64_t span = cols <= n / 2 ? pad_for(cols) : n;
    CounterDelta d = matvec_rowmajor_cost(n, span, rows);
    d += add_bias_cost(rows);
    add_step(plan, 1, cols, rep_name(RepKind::Dense), "row-major products, " + num(rows) + " rows", d,
             [np](Evaluator& ev, const EncodedTensor& x) {
                 EncodedTensor t = matvec_rowmajor(ev, x, matrix_rows(np->stages[0]));
                 return add_bias(ev, t, output_bias(np->stages[0]));
             });
    plan.depth_needed = 0;
    plan.live_entering.push_back(rows);
}

}  // namespace

Strategy strategy_from_name(const std::string& name) {
    for (Strategy s : {Strategy::LolaMnist, Strategy::LolaDenseMnist, Strategy::LolaCifar, Strategy::CryptonetsSimd,
                       Strategy::LolaSmall, Strategy::LinearFeatures})
        if (name == strategy_name(s)) return s;
    throw std::invalid_argument("unknown strategy: " + name);
}

const char* strategy_name(Strategy s) {
    switch (s) {
        case Strategy::LolaMnist: return "lola-mnist";
        case Strategy::LolaDenseMnist: return "lola-dense-mnist";
        case Strategy::LolaCifar: return "lola-cifar";
        case Strategy::CryptonetsSimd: return "cryptonets-simd";
        case Strategy::LolaSmall: return "lola-small";
        case Strategy::LinearFeatures: return "linear-features";
    }
    return "?";
}

uint64_t Plan::predicted_peak() const {
    uint64_t peak = 0;
    for (uint64_t v : live_entering) peak = std::max(peak, v);
    return peak;
}

Plan build_plan(const Network& net, Strategy s, uint32_t n, const PlanOptions& opt) {
    Plan plan;
    plan.strategy = s;
    plan.n = n;
    require(n >= 4 && (n & (n - 1)) == 0, "degree must be a power of two");
    switch (s) {
        case Strategy::LolaMnist: build_lola_mnist(plan, net, n); break;
        case Strategy::LolaDenseMnist: build_lola_dense_mnist(plan, net, n); break;
        case Strategy::LolaCifar: build_lola_cifar(plan, net, n, opt); break;
        case Strategy::LolaSmall: build_lola_small(plan, net, n); break;
        case Strategy::CryptonetsSimd: build_cryptonets_simd(plan, net); break;
        case Strategy::LinearFeatures: build_linear_features(plan, net, n); break;
    }
    return plan;
}

ExecutionResult execute(const Plan& plan, EncodedTensor input, Evaluator& ev) {  // plan.cpp:597-633
    if (plan.depth_needed > ev.context().max_depth())
        throw depth_error("plan needs depth " + std::to_string(plan.depth_needed) + " but the budget allows " +
                          std::to_string(ev.context().max_depth()));
    if (input.rep.kind != plan.in_kind || input.messages.size() != plan.in_messages ||
        input.rep.length != plan.in_length)
        throw std::invalid_argument("input tensor does not match the plan's first step");
    ExecutionResult res;
    uint64_t peak = input.messages.size();
    ev.note_live(peak);
    EncodedTensor cur = std::move(input);  // inputs die after the first step
    for (size_t i = 0; i < plan.steps.size(); ++i) {
        const PlanStep& st = plan.steps[i];
        if (i > 0) {
            const Probe pr = probe_of(cur);
            // record tensors: the reference plans a single record (dim 1); a
            // session packs `records` of them, so only count and rep compare
            const bool dim_ok = pr.dim == st.in_dim || (cur.rep.kind == RepKind::Simd && st.in_dim == 1);
            if (pr.count != st.in_count || !dim_ok || pr.rep != st.in_rep)
                throw std::logic_error("plan row diverged before step: " + st.op);
        }
        const CounterDelta before = ev.counters().ops;
        cur = st.run(ev, cur);
        const CounterDelta spent = ev.counters().ops - before;
        if (!(spent == st.predicted)) throw std::logic_error("operation count diverged at step: " + st.op);
        peak = std::max<uint64_t>(peak, cur.messages.size());
        ev.note_live(cur.messages.size());
        res.per_step.push_back(spent);
        res.total += spent;
    }
    res.live_messages_peak = peak;
    for (const Message& m : cur.messages) res.depth_consumed = std::max(res.depth_consumed, m.depth);
    res.output = std::move(cur);
    return res;
}

// decode (representation.cpp:185-223) restricted to the values the caller
// reads: device [B][values][4] signed 256-bit words.
DeviceBuffer decode_values(Evaluator& ev, const EncodedTensor& t) {
    const uint32_t B = ev.context().batch();
    cudaStream_t s = ev.context().stream();
    std::vector<DeviceBuffer> parts;
    std::vector<uint64_t> widths;
    if (t.rep.kind == RepKind::Sparse) {
        require(t.messages.size() == t.rep.length, "one message per value expected");
        for (const auto& m : t.messages) {
            parts.push_back(ev.lower_slots(m, {t.rep.broadcast ? 0u : t.rep.value_slot}));
            widths.push_back(1);
        }
    } else if (t.rep.kind == RepKind::Simd) {
        // value j of record r sits in slot r of message j: [records][values]
        const uint32_t recs = t.rep.copies;
        require(B == 1 && recs == ev.context().records(), "record tensor does not match the evaluator");
        std::vector<uint32_t> slots(recs);
        for (uint32_t r = 0; r < recs; ++r) slots[r] = r;
        const uint64_t total = t.messages.size();
        DeviceBuffer out(uint64_t(recs) * total * 32, s);
        for (uint64_t j = 0; j < total; ++j) {
            DeviceBuffer part = ev.lower_slots(t.messages[j], slots);  // [1][recs][4]
            LB_CUDA(cudaMemcpy2DAsync(out.get() + j * 4, total * 32, part.get(), 32, 32, recs,
                                      cudaMemcpyDeviceToDevice, s));
        }
        return out;
    } else {
        std::vector<uint32_t> slots(t.rep.length);
        for (uint64_t i = 0; i < t.rep.length; ++i) slots[i] = t.rep.slot(i);
        for (const auto& m : t.messages) {
            parts.push_back(ev.lower_slots(m, slots));
            widths.push_back(t.rep.length);
        }
    }
    uint64_t total = 0;
    for (uint64_t w : widths) total += w;
    DeviceBuffer out(uint64_t(B) * total * 32, s);
    uint64_t col = 0;
    for (size_t k = 0; k < parts.size(); ++k) {
        LB_CUDA(cudaMemcpy2DAsync(out.get() + col * 4, total * 32, parts[k].get(), widths[k] * 32, widths[k] * 32, B,
                                  cudaMemcpyDeviceToDevice, s));
        col += widths[k];
    }
    return out;
}

}  // namespace lb::lola
