// Evaluator mirror on device ciphertexts; semantics follow
// proj/src/evaluator.cpp line by line (cited per method).
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "host_math.hpp"
#include "lola_eval.hpp"

namespace lb::lola {

// ---- Mag -----------------------------------------------------------------------

Mag operator+(const Mag& a, const Mag& b) {
    Mag r;
    unsigned __int128 c = 0;
    for (int i = 0; i < 5; ++i) {
        c += static_cast<unsigned __int128>(a.w[i]) + b.w[i];
        r.w[i] = static_cast<uint64_t>(c);
        c >>= 64;
    }
    return c ? Mag::saturated() : r;
}

Mag operator*(const Mag& a, const Mag& b) {
    uint64_t t[10] = {};
    for (int i = 0; i < 5; ++i) {
        unsigned __int128 c = 0;
        for (int j = 0; j < 5; ++j) {
            c += static_cast<unsigned __int128>(a.w[i]) * b.w[j] + t[i + j];
            t[i + j] = static_cast<uint64_t>(c);
            c >>= 64;
        }
        for (int k = i + 5; c && k < 10; ++k) {
            c += t[k];
            t[k] = static_cast<uint64_t>(c);
            c >>= 64;
        }
    }
    for (int k = 5; k < 10; ++k)
        if (t[k]) return Mag::saturated();
    Mag r;
    std::memcpy(r.w.data(), t, 40);
    return r;
}

bool operator<(const Mag& a, const Mag& b) {
    for (int i = 4; i >= 0; --i)
        if (a.w[i] != b.w[i]) return a.w[i] < b.w[i];
    return false;
}

Mag Mag::half_floor() const {
    Mag r;
    for (int i = 0; i < 5; ++i) r.w[i] = (w[i] >> 1) | (i < 4 ? (w[i + 1] << 63) : 0);
    return r;
}

Mag Mag::minus_one() const {
    Mag r = *this;
    for (int i = 0; i < 5; ++i) {
        if (r.w[i]--) break;
    }
    return r;
}

std::string Mag::str() const {
    std::array<uint64_t, 5> v = w;
    std::string d;
    auto zero = [&] { return std::all_of(v.begin(), v.end(), [](uint64_t x) { return x == 0; }); };
    if (zero()) return "0";
    while (!zero()) {
        unsigned __int128 rem = 0;
        for (int i = 4; i >= 0; --i) {
            unsigned __int128 cur = (rem << 64) | v[i];
            v[i] = static_cast<uint64_t>(cur / 10);
            rem = cur % 10;
        }
        d.push_back(static_cast<char>('0' + static_cast<int>(rem)));
    }
    std::reverse(d.begin(), d.end());
    return d;
}

// ---- counters ---------------------------------------------------------------------

CounterDelta& CounterDelta::operator+=(const CounterDelta& o) {
    ct_ct_mul += o.ct_ct_mul;
    ct_plain_mul += o.ct_plain_mul;
    scalar_mul += o.scalar_mul;
    mask_mul += o.mask_mul;
    add += o.add;
    rot_cols += o.rot_cols;
    rot_rows += o.rot_rows;
    return *this;
}

CounterDelta operator-(const CounterDelta& a, const CounterDelta& b) {
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

bool operator==(const CounterDelta& a, const CounterDelta& b) { return a.values() == b.values(); }

// ---- device kernels -----------------------------------------------------------------

namespace {

constexpr int kBlock = 256;
inline unsigned blocks(uint64_t work) { return static_cast<unsigned>(std::max<uint64_t>(1, (work + kBlock - 1) / kBlock)); }

// out[m][b][s] = images[b * stride + map[m][s]] (0 where the map is < 0)
__global__ void k_gather_lift(const int64_t* __restrict__ images, uint64_t stride, const int32_t* __restrict__ map,
                              uint32_t n, uint32_t B, uint32_t maps, int64_t* __restrict__ out) {
    const uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (idx >= uint64_t(maps) * B * n) return;
    const uint32_t s = idx % n;
    const uint64_t b = (idx / n) % B;
    const uint64_t m = idx / (uint64_t(n) * B);
    const int32_t src = map[m * n + s];
    out[idx] = src < 0 ? 0 : images[b * stride + src];
}

struct CrtTab {
    uint32_t T;
    uint64_t t[8];
    uint64_t inv[8];      // (t_0 ... t_{k-1})^-1 mod t_k
    uint64_t pre[8][8];   // (t_0 ... t_{i-1}) mod t_k, i < k
    uint64_t M[4];        // product
    uint64_t halfM[4];    // (M - 1) / 2
};

__device__ __forceinline__ uint64_t mulmod_small(uint64_t a, uint64_t b, uint64_t t) {
    return static_cast<uint64_t>((static_cast<unsigned __int128>(a) * b) % t);
}

// Garner CRT over the plaintext primes + centering (replaces crt_join +
// center_mod, proj/src/ring.cpp:205-233, per slot); residues [B][T][n] ->
// out [B][nslots][4] two's complement 256-bit.
__global__ void k_crt_center(const uint64_t* __restrict__ res, uint32_t n, uint32_t B, const uint32_t* __restrict__ slots,
                             uint32_t nslots, CrtTab tab, uint64_t* __restrict__ out) {
    const uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (idx >= uint64_t(B) * nslots) return;
    const uint32_t si = idx % nslots;
    const uint64_t b = idx / nslots;
    const uint32_t s = slots ? slots[si] : si;
    uint64_t v[8];
    for (uint32_t k = 0; k < tab.T; ++k) {
        const uint64_t tk = tab.t[k];
        uint64_t acc = 0;
        for (uint32_t i = 0; i < k; ++i) acc = (acc + mulmod_small(v[i], tab.pre[k][i], tk)) % tk;
        const uint64_t r = res[(b * tab.T + k) * n + s];
        v[k] = mulmod_small((r + tk - acc) % tk, tab.inv[k], tk);
    }
    uint64_t x[4] = {v[tab.T - 1], 0, 0, 0};
    for (int k = int(tab.T) - 2; k >= 0; --k) {
        unsigned __int128 c = v[k];
        for (int w = 0; w < 4; ++w) {
            c += static_cast<unsigned __int128>(x[w]) * tab.t[k];
            x[w] = static_cast<uint64_t>(c);
            c >>= 64;
        }
    }
    bool gt = false;
    for (int w = 3; w >= 0; --w) {
        if (x[w] != tab.halfM[w]) {
            gt = x[w] > tab.halfM[w];
            break;
        }
    }
    if (gt) {
        uint64_t borrow = 0;
        for (int w = 0; w < 4; ++w) {
            const uint64_t a = x[w], m = tab.M[w];
            const uint64_t d = a - m - borrow;
            borrow = (a < m) || (a == m && borrow) ? 1 : 0;
            x[w] = d;
        }
    }
    uint64_t* o = out + idx * 4;
    for (int w = 0; w < 4; ++w) o[w] = x[w];
}

uint64_t hash_values(const std::vector<int64_t>& v) {
    uint64_t h = 1469598103934665603ull ^ v.size();
    for (int64_t x : v) {
        h ^= static_cast<uint64_t>(x);
        h *= 1099511628211ull;
        h ^= h >> 29;
    }
    return h;
}

}  // namespace

// ---- pointer tables --------------------------------------------------------------------

constexpr uint32_t kPtrChunk = 500;
struct PtrChunk {
    const void* p[kPtrChunk];
};

__global__ void k_put_pointers(PtrChunk c, uint32_t count, const void** dst) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) dst[i] = c.p[i];
}

void put_pointers(const void* const* host, uint64_t count, const void** dst, cudaStream_t s) {
    for (uint64_t b = 0; b < count; b += kPtrChunk) {
        PtrChunk c{};
        const uint32_t k = static_cast<uint32_t>(std::min<uint64_t>(kPtrChunk, count - b));
        std::copy(host + b, host + b + k, c.p);
        k_put_pointers<<<(k + 127) / 128, 128, 0, s>>>(c, k, dst + b);
        LB_KERNEL_DONE();
    }
}

// ---- EvalContext ---------------------------------------------------------------------

uint32_t EvalContext::fanout() const {
    static const uint32_t n = [] {
        const char* e = std::getenv("LB_STREAMS");
        const int v = e ? std::atoi(e) : 8;
        return static_cast<uint32_t>(std::max(1, std::min(v, 32)));
    }();
    return n;
}

cudaStream_t EvalContext::side_stream(uint32_t i) const {
    while (side_.size() <= i) {
        cudaStream_t s;
        LB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        side_.push_back(s);
    }
    return side_[i];
}

EvalContext::~EvalContext() {
    for (cudaStream_t s : side_) {
        cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
    }
}

EvalContext::EvalContext(Context& cx, uint32_t batch, uint32_t max_depth, cudaStream_t stream)
    : cx_(&cx), batch_(batch), max_depth_(max_depth), stream_(stream) {
    if (batch == 0) throw std::invalid_argument("batch must be positive");
    if (cx.T() == 0 || cx.T() > 8) throw std::invalid_argument("need 1..8 plaintext primes");
    Mag comp(1);
    for (uint32_t j = 0; j < cx.T(); ++j) comp = comp * Mag(cx.prime(cx.t_index(j)));
    // the device CRT (k_crt_center) writes centered values as 256-bit two's
    // complement: the composite must stay below 2^255 (Mag saturates above
    // 2^320, which this check also rejects)
    if (comp.w[4] != 0 || (comp.w[3] >> 63) != 0)
        throw std::invalid_argument("product of the plaintext primes must be below 2^255");
    capacity_ = comp.minus_one().half_floor();  // (composite - 1) / 2, ring.hpp:30
}

// ---- Evaluator -------------------------------------------------------------------------

Evaluator::Evaluator(const EvalContext& cx)
    : cx_(&cx), stream_(cx.stream()), cache_(std::make_shared<PlainCache>()) {}

Evaluator Evaluator::fork() const { return fork_on(stream_); }

Evaluator Evaluator::fork_on(cudaStream_t s) const {
    Evaluator e(*cx_);
    e.stream_ = s;
    e.cache_ = cache_;
    return e;
}

void Evaluator::absorb(const Evaluator& child) {  // evaluator.cpp:334-337
    counters_.ops += child.counters_.ops;
    counters_.note_live(child.counters_.live_messages_peak);
}

Message Evaluator::fresh(uint32_t depth, uint32_t plain_depth, Mag mag) const {
    cx_->device().activate();  // every counted op starts here
    Message m;
    m.payload = std::make_shared<Payload>();
    m.payload->buf = DeviceBuffer(cx_->payload_bytes(), stream_);
    m.depth = depth;
    m.plain_depth = plain_depth;
    m.magnitude = mag;
    return m;
}

void Evaluator::check_magnitude(const Mag& m, const char* op) const {  // evaluator.cpp:48-55
    if (m > cx_->capacity())
        throw magnitude_error(std::string(op) + ": magnitude bound " + m.str() + " exceeds modulus capacity " +
                              cx_->capacity().str());
}

Message Evaluator::lift(const std::vector<int64_t>& values) const {
    return lift_batch(std::vector<std::vector<int64_t>>(cx_->batch(), values));
}

Message Evaluator::lift_batch(const std::vector<std::vector<int64_t>>& values) const {  // evaluator.cpp:67-96
    const uint32_t n = cx_->n(), B = cx_->batch();
    if (values.size() != B) throw std::invalid_argument("lift: one value vector per batch entry");
    std::vector<int64_t> host(uint64_t(B) * n, 0);
    Mag mag(0);
    for (uint32_t b = 0; b < B; ++b) {
        if (values[b].size() > n) throw std::invalid_argument("lift: more values than slots");
        for (size_t i = 0; i < values[b].size(); ++i) {
            const int64_t v = values[b][i];
            const uint64_t a = v < 0 ? uint64_t(-(v + 1)) + 1 : uint64_t(v);
            if (Mag(a) > mag) mag = Mag(a);
            host[uint64_t(b) * n + i] = v;
        }
    }
    check_magnitude(mag, "lift");
    cudaStream_t s = stream_;
    DeviceBuffer dv(host.size() * 8, s);
    LB_CUDA(cudaMemcpyAsync(dv.get(), host.data(), host.size() * 8, cudaMemcpyHostToDevice, s));
    Message m = fresh(0, 0, mag);
    const uint64_t id = cx_->device().reserve_ciphertext_ids(cx_->cts());
    encrypt_slots(cx_->device(), dv.get<int64_t>(), B, id, m.data(), s);
    LB_CUDA(cudaStreamSynchronize(s));  // `host` is pageable and local
    return m;
}

Message Evaluator::lift_gather(const int64_t* dev_images, uint64_t stride, const std::vector<int32_t>& map,
                               int64_t max_abs) const {
    return lift_gather_many(dev_images, stride, {map}, max_abs).front();
}

std::vector<Message> Evaluator::lift_gather_many(const int64_t* dev_images, uint64_t stride,
                                                 const std::vector<std::vector<int32_t>>& maps,
                                                 int64_t max_abs) const {
    const uint32_t n = cx_->n(), B = cx_->batch();
    const uint32_t count = static_cast<uint32_t>(maps.size());
    if (!count) return {};
    std::vector<int32_t> full(uint64_t(count) * n, -1);
    for (uint32_t m = 0; m < count; ++m) {
        if (maps[m].size() > n) throw std::invalid_argument("lift: more values than slots");
        std::copy(maps[m].begin(), maps[m].end(), full.begin() + uint64_t(m) * n);
    }
    const Mag mag(static_cast<uint64_t>(max_abs < 0 ? -max_abs : max_abs));
    check_magnitude(mag, "lift");
    cudaStream_t s = stream_;
    DeviceBuffer dmap(full.size() * 4, s), slots(uint64_t(count) * B * n * 8, s);
    LB_CUDA(cudaMemcpyAsync(dmap.get(), full.data(), full.size() * 4, cudaMemcpyHostToDevice, s));
    k_gather_lift<<<blocks(uint64_t(count) * B * n), kBlock, 0, s>>>(dev_images, stride, dmap.get<int32_t>(), n, B,
                                                                      count, slots.get<int64_t>());
    LB_KERNEL_DONE();
    std::vector<Message> out;
    out.reserve(count);
    for (uint32_t m = 0; m < count; ++m) {
        out.push_back(fresh(0, 0, mag));
        const uint64_t id = cx_->device().reserve_ciphertext_ids(cx_->cts());
        encrypt_slots(cx_->device(), slots.get<int64_t>() + uint64_t(m) * B * n, B, id, out.back().data(), s);
    }
    return out;
}

DeviceBuffer Evaluator::lower_slots(const Message& m, const std::vector<uint32_t>& slots) const {
    Context& dc = cx_->device();
    dc.activate();
    const uint32_t n = cx_->n(), B = cx_->batch(), T = dc.T();
    cudaStream_t s = stream_;
    DeviceBuffer res(uint64_t(B) * T * n * 8, s);
    decrypt_slots(dc, m.data(), B, res.get(), s);
    CrtTab tab{};
    tab.T = T;
    for (uint32_t k = 0; k < T; ++k) tab.t[k] = dc.prime(dc.t_index(k));
    for (uint32_t k = 0; k < T; ++k) {
        uint64_t prod = 1 % tab.t[k];
        for (uint32_t i = 0; i < k; ++i) {
            tab.pre[k][i] = prod;
            prod = static_cast<uint64_t>((static_cast<unsigned __int128>(prod) * (tab.t[i] % tab.t[k])) % tab.t[k]);
        }
        tab.inv[k] = k ? host::invm(prod, tab.t[k]) : 1;
    }
    Mag M(1);
    for (uint32_t k = 0; k < T; ++k) M = M * Mag(tab.t[k]);
    const Mag half = M.minus_one().half_floor();
    for (int w = 0; w < 4; ++w) {
        tab.M[w] = M.w[w];
        tab.halfM[w] = half.w[w];
    }
    const uint32_t ns = slots.empty() ? n : static_cast<uint32_t>(slots.size());
    DeviceBuffer dsl;
    if (!slots.empty()) {
        dsl = DeviceBuffer(slots.size() * 4, s);
        LB_CUDA(cudaMemcpyAsync(dsl.get(), slots.data(), slots.size() * 4, cudaMemcpyHostToDevice, s));
    }
    DeviceBuffer out(uint64_t(B) * ns * 4 * 8, s);
    k_crt_center<<<blocks(uint64_t(B) * ns), kBlock, 0, s>>>(res.get(), n, B, slots.empty() ? nullptr : dsl.get<uint32_t>(),
                                                             ns, tab, out.get());
    LB_KERNEL_DONE();
    // no host sync: a pageable host-to-device cudaMemcpyAsync has staged its
    // source before returning, so `slots` may go out of scope
    return out;
}

DeviceBuffer Evaluator::lower(const Message& m) const { return lower_slots(m, {}); }

const void* Evaluator::plain(const std::vector<int64_t>& values, bool for_add) {
    auto& table = for_add ? cache_->add : cache_->mul;
    const uint64_t h = hash_values(values);
    auto& bucket = table[h];
    for (auto& e : bucket)
        if (e->values == values) {
            // (entries used under graph capture were made, and synchronised,
            // before the capture began)
            if (e->made_on != stream_ && !cx_->capturing()) LB_CUDA(cudaStreamWaitEvent(stream_, e->ready, 0));
            return e->pt.get();
        }
    if (cx_->capturing()) throw std::logic_error("plaintext operand first seen under graph capture");
    const uint32_t n = cx_->n();
    Context& dc = cx_->device();
    cudaStream_t s = stream_;
    std::vector<int64_t> full(n, 0);
    std::copy(values.begin(), values.end(), full.begin());
    DeviceBuffer dv(uint64_t(n) * 8, s);
    LB_CUDA(cudaMemcpyAsync(dv.get(), full.data(), uint64_t(n) * 8, cudaMemcpyHostToDevice, s));
    const size_t pt_bytes = uint64_t(dc.T()) * dc.L() * n * residue_bytes(dc.bfv()->dev);
    static const size_t budget = [] {
        const char* e = std::getenv("LB_PLAIN_CACHE_GB");
        return static_cast<size_t>((e ? std::atof(e) : 8.0) * (1ull << 30));
    }();
    if (cache_->bytes + pt_bytes > budget) {
        DeviceBuffer t(pt_bytes, s);
        encode_plain(dc, dv.get<int64_t>(), for_add ? nullptr : t.get(), for_add ? t.get() : nullptr, s);
        const void* p = t.get();
        cache_->transient.push_back(std::move(t));
        while (cache_->transient.size() > 4) cache_->transient.pop_front();
        return p;
    }
    cache_->bytes += pt_bytes;
    auto e = std::make_unique<PlainCache::Entry>();
    e->values = values;
    e->pt = DeviceBuffer(uint64_t(dc.T()) * dc.L() * n * residue_bytes(dc.bfv()->dev), s);
    encode_plain(dc, dv.get<int64_t>(), for_add ? nullptr : e->pt.get(), for_add ? e->pt.get() : nullptr, s);
    e->made_on = s;
    LB_CUDA(cudaEventCreateWithFlags(&e->ready, cudaEventDisableTiming));
    LB_CUDA(cudaEventRecord(e->ready, s));
    const void* p = e->pt.get();
    bucket.push_back(std::move(e));
    return p;
}

Message Evaluator::add(const Message& a, const Message& b) {  // evaluator.cpp:137-152
    const Mag mag = a.magnitude + b.magnitude;
    check_magnitude(mag, "add");
    counters_.ops.add += 1;
    Message r = fresh(std::max(a.depth, b.depth), std::max(a.plain_depth, b.plain_depth), mag);
    ct_add(cx_->device(), a.data(), b.data(), r.data(), static_cast<uint32_t>(cx_->cts()), stream_);
    return r;
}

static uint64_t max_abs(const std::vector<int64_t>& v) {
    uint64_t m = 0;
    for (int64_t x : v) m = std::max<uint64_t>(m, x < 0 ? uint64_t(-(x + 1)) + 1 : uint64_t(x));
    return m;
}

Message Evaluator::add_plain(const Message& a, const std::vector<int64_t>& values) {  // evaluator.cpp:154-176
    const Mag mag = a.magnitude + Mag(max_abs(values));
    check_magnitude(mag, "add_plain");
    counters_.ops.add += 1;
    if (values.size() > cx_->n()) throw std::invalid_argument("plain operand: more values than slots");
    const void* pt = plain(values, true);
    Message r = fresh(a.depth, a.plain_depth, mag);
    ct_add_plain(cx_->device(), a.data(), pt, r.data(), static_cast<uint32_t>(cx_->cts()), stream_);
    return r;
}

Message Evaluator::mul(const Message& a, const Message& b) {  // evaluator.cpp:178-202
    const uint32_t depth = std::max(a.depth, b.depth) + 1;
    if (depth > cx_->max_depth())
        throw depth_error("mul: depth " + std::to_string(depth) + " exceeds budget " + std::to_string(cx_->max_depth()));
    const Mag mag = a.magnitude * b.magnitude;
    check_magnitude(mag, "mul");
    counters_.ops.ct_ct_mul += 1;
    Message r = fresh(depth, std::max(a.plain_depth, b.plain_depth), mag);
    ct_mul(cx_->device(), a.data(), b.data(), r.data(), static_cast<uint32_t>(cx_->cts()), stream_);
    return r;
}

Message Evaluator::mul_plain(const Message& a, const std::vector<int64_t>& values) {  // evaluator.cpp:204-226
    const Mag mag = a.magnitude * Mag(max_abs(values));
    check_magnitude(mag, "mul_plain");
    counters_.ops.ct_plain_mul += 1;
    if (values.size() > cx_->n()) throw std::invalid_argument("plain operand: more values than slots");
    const void* pt = plain(values, false);
    Message r = fresh(a.depth, a.plain_depth + 1, mag);
    ct_mul_plain(cx_->device(), a.data(), pt, r.data(), static_cast<uint32_t>(cx_->cts()), stream_);
    return r;
}

Message Evaluator::mask(const Message& a, const std::vector<uint8_t>& bits) {  // evaluator.cpp:228-240
    if (bits.size() > cx_->n()) throw std::invalid_argument("mask: more bits than slots");
    bool any = false;
    for (uint8_t b : bits) {
        if (b > 1) throw std::invalid_argument("mask: entries must be 0 or 1");
        any |= (b == 1);
    }
    if (!any) throw std::invalid_argument("mask: empty mask");
    counters_.ops.mask_mul += 1;
    return mul_plain(a, std::vector<int64_t>(bits.begin(), bits.end()));
}

std::vector<Message> Evaluator::weighted_sums(const std::vector<Message>& xs, uint64_t rows, const int64_t* host_w,
                                             const int64_t* dev_w) {  // kernels.cpp:302-318
    const uint64_t F = xs.size();
    if (F == 0 || rows == 0) throw std::invalid_argument("weighted sums: empty operand");
    auto absu = [](int64_t v) { return v < 0 ? uint64_t(-(v + 1)) + 1 : uint64_t(v); };
    uint32_t depth = 0, plain_depth = 0;
    bool small = true;  // every magnitude < 2^64: 128-bit bookkeeping suffices
    for (const Message& x : xs) {
        depth = std::max(depth, x.depth);
        plain_depth = std::max(plain_depth, x.plain_depth + 1);
        for (size_t k = 1; k < x.magnitude.w.size(); ++k) small = small && x.magnitude.w[k] == 0;
    }
    const Mag& cap = cx_->capacity();
    bool small_w = true;
    for (uint64_t k = 0; k < rows * F; ++k) small_w = small_w && absu(host_w[k]) < (1u << 15);
    std::vector<Mag> mags(rows);
    for (uint64_t r = 0; r < rows; ++r) {
        const int64_t* wr = host_w + r * F;
        bool over = false;
        if (small) {
            unsigned __int128 acc = 0;
            for (uint64_t i = 0; i < F; ++i) {
                const uint64_t aw = absu(wr[i]);
                if (aw >> 31) throw std::invalid_argument("weighted sums: |weight| must be below 2^31");
                acc += static_cast<unsigned __int128>(xs[i].magnitude.w[0]) * aw;  // < 2^95 per term, F < 2^17
            }
            Mag m;
            m.w[0] = static_cast<uint64_t>(acc);
            m.w[1] = static_cast<uint64_t>(acc >> 64);
            mags[r] = m;
            over = m > cap;
        } else {
            Mag m(0);
            for (uint64_t i = 0; i < F; ++i) m = m + xs[i].magnitude * Mag(absu(wr[i]));
            mags[r] = m;
            over = m > cap;
        }
        if (over) {
            // replay the reference's sequence to raise at the same operation
            counters_.ops.scalar_mul += r * F;
            counters_.ops.add += r * (F - 1);
            Mag acc = xs[0].magnitude * Mag(absu(wr[0]));
            check_magnitude(acc, "mul_scalar");
            counters_.ops.scalar_mul += 1;
            for (uint64_t i = 1; i < F; ++i) {
                const Mag p = xs[i].magnitude * Mag(absu(wr[i]));
                check_magnitude(p, "mul_scalar");
                counters_.ops.scalar_mul += 1;
                acc = acc + p;
                check_magnitude(acc, "add");
                counters_.ops.add += 1;
            }
            throw std::logic_error("weighted sums: magnitude bookkeeping diverged");
        }
    }
    counters_.ops.scalar_mul += rows * F;
    counters_.ops.add += rows * (F - 1);
    std::vector<Message> out;
    out.reserve(rows);
    std::vector<const void*> xp(F);
    std::vector<void*> op(rows);
    for (uint64_t i = 0; i < F; ++i) xp[i] = xs[i].data();
    for (uint64_t r = 0; r < rows; ++r) {
        out.push_back(fresh(depth, plain_depth, mags[r]));
        op[r] = out.back().data();
    }
    cudaStream_t s = stream_;
    DeviceBuffer dx(F * 8, s), dout(rows * 8, s);
    // pointer tables travel as kernel parameters (captured by value, so the
    // sequence is also valid inside a CUDA graph)
    put_pointers(xp.data(), F, dx.get<const void*>(), s);
    put_pointers(const_cast<const void* const*>(op.data()), rows, dout.get<const void*>(), s);
    simd_weighted_sums(cx_->device(), reinterpret_cast<const void* const*>(dx.get()), static_cast<uint32_t>(F),
                       reinterpret_cast<void* const*>(dout.get()), static_cast<uint32_t>(rows), dev_w, small_w,
                       static_cast<uint32_t>(cx_->cts()), s);
    // dx / dout are freed stream-ordered after the kernel (cudaFreeAsync on s);
    // the host arrays were staged by the pageable-memory copies already
    return out;
}

Message Evaluator::mul_scalar(const Message& a, int64_t sc) {  // evaluator.cpp:242-258
    const uint64_t as = sc < 0 ? uint64_t(-(sc + 1)) + 1 : uint64_t(sc);
    const Mag mag = a.magnitude * Mag(as);
    check_magnitude(mag, "mul_scalar");
    counters_.ops.scalar_mul += 1;
    Message r = fresh(a.depth, a.plain_depth + 1, mag);
    ct_mul_scalar(cx_->device(), a.data(), sc, r.data(), static_cast<uint32_t>(cx_->cts()), stream_);
    return r;
}

// Right shift of both slot rows (evaluator.cpp:260-287): one automorphism
// x -> x^(3^(half - shift)) plus a key switch; with `base`, the sum
// base + shifted (the caller counts both operations).
Message Evaluator::shift_columns(const Message& a, uint32_t right_by, const Message* base) {
    const uint32_t half = cx_->half();
    const uint32_t shift = right_by % half;
    const uint64_t two_n = 2ull * cx_->n();
    uint64_t g = 1, b3 = 3;
    for (uint64_t e = (half - shift) % half; e; e >>= 1) {
        if (e & 1) g = g * b3 % two_n;
        b3 = b3 * b3 % two_n;
    }
    const uint32_t cts = static_cast<uint32_t>(cx_->cts());
    if (base) {
        Message r = fresh(std::max(a.depth, base->depth), std::max(a.plain_depth, base->plain_depth),
                          a.magnitude + base->magnitude);
        if (g == 1)
            ct_add(cx_->device(), base->data(), a.data(), r.data(), cts, stream_);
        else
            ct_rotate_add(cx_->device(), base->data(), a.data(), g, r.data(), cts, stream_);
        return r;
    }
    Message r = fresh(a.depth, a.plain_depth, a.magnitude);
    if (g == 1) {
        LB_CUDA(cudaMemcpyAsync(r.data(), a.data(), cx_->payload_bytes(), cudaMemcpyDeviceToDevice, stream_));
    } else {
        ct_rotate(cx_->device(), a.data(), g, r.data(), cts, stream_);
    }
    return r;
}

Message Evaluator::rotate_columns(const Message& a, int64_t k) {  // evaluator.cpp:289-299
    const int64_t half = cx_->half();
    if (k <= -half || k >= half) throw std::invalid_argument("rotate_columns: |k| must be below n/2");
    if (k == 0) return a;
    const uint64_t amount = static_cast<uint64_t>(k < 0 ? -k : k);
    counters_.ops.rot_cols += static_cast<uint64_t>(__builtin_popcountll(amount));
    const uint32_t right_by = k > 0 ? static_cast<uint32_t>(k) : static_cast<uint32_t>(half + k);
    return shift_columns(a, right_by);
}

Message Evaluator::rotate_rows(const Message& a) {  // evaluator.cpp:301-324
    counters_.ops.rot_rows += 1;
    Message r = fresh(a.depth, a.plain_depth, a.magnitude);
    ct_rotate(cx_->device(), a.data(), 2ull * cx_->n() - 1, r.data(), static_cast<uint32_t>(cx_->cts()),
              stream_);
    return r;
}

Message Evaluator::rotate_bundle(const Message& a, uint32_t amount) {  // evaluator.cpp:326-332
    if (amount >= cx_->half()) throw std::invalid_argument("rotate_bundle: amount must be below n/2");
    if (amount == 0) return a;
    counters_.ops.rot_cols += 1;
    return shift_columns(a, amount);
}

// ---- fused forms ------------------------------------------------------------------

Message Evaluator::mul_scalar_add(const Message& acc, const Message& x, int64_t sc) {
    const uint64_t as = sc < 0 ? uint64_t(-(sc + 1)) + 1 : uint64_t(sc);
    const Mag prod = x.magnitude * Mag(as);
    check_magnitude(prod, "mul_scalar");
    counters_.ops.scalar_mul += 1;
    const Mag mag = acc.magnitude + prod;
    check_magnitude(mag, "add");
    counters_.ops.add += 1;
    Message r = fresh(std::max(acc.depth, x.depth), std::max(acc.plain_depth, x.plain_depth + 1), mag);
    ct_mul_scalar_add(cx_->device(), acc.data(), x.data(), sc, r.data(), static_cast<uint32_t>(cx_->cts()),
                      stream_);
    return r;
}

Message Evaluator::rotate_columns_add(const Message& base, const Message& x, int64_t k) {
    const int64_t half = cx_->half();
    if (k <= -half || k >= half) throw std::invalid_argument("rotate_columns: |k| must be below n/2");
    if (k == 0) return add(base, x);
    const uint64_t amount = static_cast<uint64_t>(k < 0 ? -k : k);
    counters_.ops.rot_cols += static_cast<uint64_t>(__builtin_popcountll(amount));
    const Mag mag = base.magnitude + x.magnitude;
    check_magnitude(mag, "add");
    counters_.ops.add += 1;
    const uint32_t right_by = k > 0 ? static_cast<uint32_t>(k) : static_cast<uint32_t>(half + k);
    return shift_columns(x, right_by, &base);
}

Message Evaluator::rotate_bundle_add(const Message& base, const Message& x, uint32_t amount) {
    if (amount >= cx_->half()) throw std::invalid_argument("rotate_bundle: amount must be below n/2");
    if (amount == 0) return add(base, x);
    counters_.ops.rot_cols += 1;
    const Mag mag = base.magnitude + x.magnitude;
    check_magnitude(mag, "add");
    counters_.ops.add += 1;
    return shift_columns(x, amount, &base);
}

Message Evaluator::rotate_rows_add(const Message& base, const Message& x) {
    counters_.ops.rot_rows += 1;
    const Mag mag = base.magnitude + x.magnitude;
    check_magnitude(mag, "add");
    counters_.ops.add += 1;
    Message r = fresh(std::max(x.depth, base.depth), std::max(x.plain_depth, base.plain_depth), mag);
    ct_rotate_add(cx_->device(), base.data(), x.data(), 2ull * cx_->n() - 1, r.data(),
                  static_cast<uint32_t>(cx_->cts()), stream_);
    return r;
}

}  // namespace lb::lola
