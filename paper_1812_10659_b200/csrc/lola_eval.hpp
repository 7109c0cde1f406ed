// Host C++ mirror of the reference evaluator boundary (proj/include/packnn/
// message.hpp:14-75, evaluator.hpp:12-91) running on device BFV ciphertexts.
//
// Same names, argument meaning, counting rules and exceptions as the
// reference; two B200-first differences:
//   * a Message is a BATCH of B independent messages (one per image) held as
//     one device buffer [B][T][2][L][n] — every op is one set of kernels over
//     all B*T ciphertexts, plaintext operands are broadcast;
//   * plaintext operands are encoded on the device once and cached by value.
// Counters, depth and magnitude budgets stay on the host and follow
// proj/src/evaluator.cpp exactly.
#pragma once

#include <array>
#include <cstdint>
#include <deque>
#include <memory>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "bfv.hpp"
#include "context.hpp"

namespace lb::lola {

// Thrown when an operation would exceed the multiplicative depth budget
// (proj/include/packnn/message.hpp:14-18).
class depth_error : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
// Thrown when a magnitude bound would exceed the plaintext CRT capacity
// (message.hpp:20-24).
class magnitude_error : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

// Non-negative magnitude bound, fixed 320-bit, saturating (replaces the
// reference's BigInt magnitude, message.hpp:74; every capacity here is below
// 2^256 so saturation only ever means "too big").
struct Mag {
    std::array<uint64_t, 5> w{};
    Mag() = default;
    Mag(uint64_t v) { w[0] = v; }  // NOLINT
    static Mag saturated() {
        Mag m;
        m.w.fill(~uint64_t{0});
        return m;
    }
    friend Mag operator+(const Mag& a, const Mag& b);
    friend Mag operator*(const Mag& a, const Mag& b);
    friend bool operator<(const Mag& a, const Mag& b);
    friend bool operator>(const Mag& a, const Mag& b) { return b < a; }
    friend bool operator==(const Mag& a, const Mag& b) { return a.w == b.w; }
    Mag half_floor() const;  // floor(x / 2)
    Mag minus_one() const;
    std::string str() const;  // decimal
};

struct CounterDelta {
    uint64_t ct_ct_mul = 0, ct_plain_mul = 0, scalar_mul = 0, mask_mul = 0, add = 0, rot_cols = 0, rot_rows = 0;
    CounterDelta& operator+=(const CounterDelta& o);
    friend CounterDelta operator+(CounterDelta a, const CounterDelta& b) { return a += b; }
    friend CounterDelta operator-(const CounterDelta& a, const CounterDelta& b);
    friend bool operator==(const CounterDelta& a, const CounterDelta& b);
    uint64_t rotations() const { return rot_cols + rot_rows; }
    std::array<uint64_t, 7> values() const {
        return {ct_ct_mul, ct_plain_mul, scalar_mul, mask_mul, add, rot_cols, rot_rows};
    }
};

struct OpCounters {
    CounterDelta ops;
    uint64_t live_messages_peak = 0;
    void note_live(uint64_t live) {
        if (live > live_messages_peak) live_messages_peak = live;
    }
};

// Device payload: [B][T][2][L][n] residue words (u32 when every ciphertext
// and special prime is below 2^30, else u64), NTT domain.
struct Payload {
    DeviceBuffer buf;
};

struct Message {
    std::shared_ptr<Payload> payload;
    uint32_t depth = 0;
    uint32_t plain_depth = 0;
    Mag magnitude;
    void* data() const { return payload->buf.get(); }
};

// Shared execution parameters (evaluator.hpp:16-41): device context, batch
// size (images per message), depth budget, the stream all ops run on.
class EvalContext {
public:
    EvalContext(Context& cx, uint32_t batch, uint32_t max_depth = 8, cudaStream_t stream = nullptr);
    Context& device() const { return *cx_; }
    uint32_t n() const { return cx_->n(); }
    uint32_t half() const { return cx_->n() / 2; }
    uint32_t batch() const { return batch_; }
    // records packed into the slots of one message (record/SIMD tensors,
    // representation.cpp:167-183); defaults to 1
    uint32_t records() const { return records_; }
    void set_records(uint32_t r) { records_ = r; }
    uint32_t primes() const { return cx_->T(); }  // plaintext CRT primes
    uint32_t max_depth() const { return max_depth_; }
    const Mag& capacity() const { return capacity_; }
    cudaStream_t stream() const { return stream_; }
    uint64_t cts() const { return uint64_t(batch_) * cx_->T(); }
    size_t payload_bytes() const { return cts() * 2 * cx_->L() * cx_->n() * residue_bytes(cx_->bfv()->dev); }
    // Side streams for fanning independent op chains out (the GPU analogue
    // of the reference's thread fan-out, proj/src/kernels.cpp:161-195).
    // LB_STREAMS (default 8) sets the count; 1 disables the fan-out.
    uint32_t fanout() const;
    cudaStream_t side_stream(uint32_t i) const;
    // true while a session captures the plan into a CUDA graph: every op must
    // then be stream-ordered device work (no host syncs, no pageable uploads,
    // no waits on events recorded before the capture began)
    bool capturing() const { return capturing_; }
    void set_capturing(bool c) const { capturing_ = c; }
    ~EvalContext();

private:
    Context* cx_;
    uint32_t batch_;
    uint32_t records_ = 1;
    uint32_t max_depth_;
    cudaStream_t stream_;
    Mag capacity_;
    mutable std::vector<cudaStream_t> side_;
    mutable bool capturing_ = false;
};

// Shared cache of device-encoded plaintext operands keyed by value.
struct PlainCache {
    struct Entry {
        std::vector<int64_t> values;
        DeviceBuffer pt;  // [T][L][n]
        cudaStream_t made_on = nullptr;
        cudaEvent_t ready = nullptr;  // recorded after encoding on made_on
        ~Entry() {
            if (ready) cudaEventDestroy(ready);
        }
    };
    std::unordered_map<uint64_t, std::vector<std::unique_ptr<Entry>>> mul, add;
    // Device bytes held by entries. Above the budget (LB_PLAIN_CACHE_GB,
    // default 8) new operands are encoded into transient buffers instead:
    // lola-cifar's 8,160 weight rows and 4,075 masks would otherwise pin
    // ~53 GB, which is what bounds its batch. A transient is freed once a
    // few newer ones exist: every op enqueues its kernel before the next
    // plain() call, so the stream-ordered free follows its last use.
    size_t bytes = 0;
    std::deque<DeviceBuffer> transient;
};

class Evaluator {
public:
    explicit Evaluator(const EvalContext& cx);

    const EvalContext& context() const { return *cx_; }
    OpCounters& counters() { return counters_; }
    const OpCounters& counters() const { return counters_; }

    // Encoding boundary (no counters). lift: the same values for every
    // message of the batch; lift_batch: values[b] per message; lift_gather:
    // slot s of message b = images[b * stride + map[s]] (0 where map < 0),
    // images already on the device.
    Message lift(const std::vector<int64_t>& values) const;
    Message lift_batch(const std::vector<std::vector<int64_t>>& values) const;
    Message lift_gather(const int64_t* dev_images, uint64_t stride, const std::vector<int32_t>& map,
                        int64_t max_abs) const;
    // lift_gather for several maps at once (one upload of the maps, one
    // gather, then the messages' encryptions back to back with no host sync);
    // messages and ciphertext ids in map order, as repeated lift_gather calls
    std::vector<Message> lift_gather_many(const int64_t* dev_images, uint64_t stride,
                                          const std::vector<std::vector<int32_t>>& maps, int64_t max_abs) const;
    // Decrypt + CRT + center every slot: device [B][n] signed 256-bit
    // (4 little-endian words, two's complement). lower_slots gathers only
    // the listed slots: [B][slots.size()] words.
    DeviceBuffer lower(const Message& m) const;
    DeviceBuffer lower_slots(const Message& m, const std::vector<uint32_t>& slots) const;

    Message add(const Message& a, const Message& b);
    Message add_plain(const Message& a, const std::vector<int64_t>& values);
    Message mul(const Message& a, const Message& b);
    Message mul_plain(const Message& a, const std::vector<int64_t>& values);
    Message mask(const Message& a, const std::vector<uint8_t>& bits);
    Message mul_scalar(const Message& a, int64_t s);
    Message rotate_columns(const Message& a, int64_t k);
    Message rotate_rows(const Message& a);
    Message rotate_bundle(const Message& a, uint32_t amount);

    // Fused forms: exactly the counters, budgets and results of the two-op
    // sequences they replace, one kernel pass instead of two.
    //   mul_scalar_add(acc, x, s)       == add(acc, mul_scalar(x, s))
    //   rotate_columns_add(b, x, k)     == add(b, rotate_columns(x, k))
    //   rotate_rows_add(b, x)           == add(b, rotate_rows(x))
    //   rotate_bundle_add(b, x, amount) == add(b, rotate_bundle(x, amount))
    Message mul_scalar_add(const Message& acc, const Message& x, int64_t s);
    Message rotate_columns_add(const Message& base, const Message& x, int64_t k);
    Message rotate_rows_add(const Message& base, const Message& x);
    Message rotate_bundle_add(const Message& base, const Message& x, uint32_t amount);

    // Record-tensor dense layer (simd_dense, kernels.cpp:302-318): row r of
    // the rows x xs.size() row-major integer matrix gives
    //   out_r = mul_scalar(x_0, W[r][0]) + ... + mul_scalar(x_k, W[r][k])
    // with exactly the reference's counters, depth and magnitude checks (and
    // error texts) of that sequence, computed as one batched kernel.
    // host_w feeds the bookkeeping, dev_w (same matrix on the device) the kernel.
    std::vector<Message> weighted_sums(const std::vector<Message>& xs, uint64_t rows, const int64_t* host_w,
                                       const int64_t* dev_w);

    void note_live(uint64_t live) { counters_.note_live(live); }
    Evaluator fork() const;
    void absorb(const Evaluator& child);
    // fork whose device work goes to stream `s` (shares the plaintext cache;
    // ciphertext ids come from the context's counter)
    Evaluator fork_on(cudaStream_t s) const;
    cudaStream_t stream() const { return stream_; }

private:
    const EvalContext* cx_;
    cudaStream_t stream_;
    OpCounters counters_;
    std::shared_ptr<PlainCache> cache_;

    Message fresh(uint32_t depth, uint32_t plain_depth, Mag mag) const;
    void check_magnitude(const Mag& m, const char* op) const;
    const void* plain(const std::vector<int64_t>& values, bool for_add);
    Message shift_columns(const Message& a, uint32_t right_by, const Message* base = nullptr);
};

}  // namespace lb::lola
