// Device context: ring degree, the RNS prime table and its NTT tables, and
// (filled in by bfv.cu) the BFV constants and key material.
//
// Prime table order: [q_0 .. q_{L-1}] ciphertext primes, [p_0 .. p_{K-1}]
// special (key-switching) primes, [b_0 .. b_{M-1}] auxiliary base of the
// exact tensor product, [t_0 .. t_{T-1}] plaintext CRT primes.
// Limb-major RNS layout everywhere: a polynomial is `limbs` contiguous
// length-N u64 arrays, a ciphertext is 2 polynomials, a batch is contiguous.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "modarith.cuh"
#include "ntt.cuh"

namespace lb {

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define LB_CUDA(expr)                                                                              \
    do {                                                                                           \
        cudaError_t _e = (expr);                                                                   \
        if (_e != cudaSuccess)                                                                     \
            throw ::lb::CudaError(std::string(#expr) + ": " + cudaGetErrorString(_e));             \
    } while (0)

// Kernels launched by this library (bench.py reports the count inside its
// timed region).
std::atomic<uint64_t>& launch_counter();
#define LB_KERNEL_DONE()                                          \
    do {                                                          \
        LB_CUDA(cudaGetLastError());                              \
        ::lb::launch_counter().fetch_add(1, std::memory_order_relaxed); \
    } while (0)

// Owning device allocation (stream-ordered pool).
class DeviceBuffer {
public:
    DeviceBuffer() = default;
    DeviceBuffer(size_t bytes, cudaStream_t s) : bytes_(bytes), stream_(s) {
        if (bytes) LB_CUDA(cudaMallocAsync(&ptr_, bytes, s));
    }
    ~DeviceBuffer() { release(); }
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    DeviceBuffer(DeviceBuffer&& o) noexcept { *this = std::move(o); }
    DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
        if (this != &o) {
            release();
            ptr_ = o.ptr_;
            bytes_ = o.bytes_;
            stream_ = o.stream_;
            owned_ = o.owned_;
            o.ptr_ = nullptr;
            o.bytes_ = 0;
            o.owned_ = true;
        }
        return *this;
    }
    template <class T = uint64_t>
    T* get() const { return static_cast<T*>(ptr_); }
    size_t bytes() const { return bytes_; }
    // Frees go to `s` from now on (the caller orders `s` after every use on
    // the allocating stream, e.g. through an event).
    void rebind(cudaStream_t s) { stream_ = s; }
    // Stop owning the memory (the pointer stays valid for readers): for
    // buffers a CUDA graph allocated, which the graph's owner frees.
    void* disown() {
        owned_ = false;
        return ptr_;
    }
    bool owned() const { return owned_; }

private:
    void release() {
        if (ptr_ && owned_) cudaFreeAsync(ptr_, stream_);
        ptr_ = nullptr;
    }
    void* ptr_ = nullptr;
    size_t bytes_ = 0;
    cudaStream_t stream_ = nullptr;
    bool owned_ = true;
};

struct Params {
    uint32_t n = 0;
    std::vector<uint64_t> q, p, b, t;
    uint32_t dnum = 0;
    uint64_t seed = 0;
    int device = 0;
};

struct BfvState;  // bfv.cu

class Context {
public:
    explicit Context(const Params& prm);
    ~Context();

    uint32_t n() const { return n_; }
    int logn() const { return logn_; }
    uint32_t L() const { return static_cast<uint32_t>(prm_.q.size()); }
    uint32_t K() const { return static_cast<uint32_t>(prm_.p.size()); }
    uint32_t M() const { return static_cast<uint32_t>(prm_.b.size()); }
    uint32_t T() const { return static_cast<uint32_t>(prm_.t.size()); }
    uint32_t dnum() const { return dnum_; }
    uint32_t alpha() const { return (L() + dnum_ - 1) / dnum_; }
    uint32_t prime_count() const { return static_cast<uint32_t>(all_.size()); }
    uint64_t prime(uint32_t i) const { return all_.at(i); }
    uint32_t p_index(uint32_t k) const { return L() + k; }
    uint32_t b_index(uint32_t m) const { return L() + K() + m; }
    uint32_t t_index(uint32_t j) const { return L() + K() + M() + j; }
    uint64_t psi(uint32_t i) const { return psi_.at(i); }
    const Params& params() const { return prm_; }
    const PrimeDev* dev_primes() const { return d_primes_.get<PrimeDev>(); }
    const PrimeDev& host_prime(uint32_t i) const { return host_primes_.at(i); }  // constants only
    const PrimeTab32& tab32() const { return tab32_; }
    const Modulus& modulus(uint32_t i) const { return mods_.at(i); }
    cudaStream_t stream() const { return stream_; }
    int device() const { return prm_.device; }
    // make this context's device current for the calling thread
    void activate() const;

    // Batched transforms over [polys][limbs][N] with limb l using prime
    // first_prime + l.
    // true when every prime of the batch is below 2^30 (and LB_WORD32 != 0):
    // the transform then runs on 32-bit words
    bool batch_word32(const LimbBatch& b) const;
    static bool word32_enabled();
    // paired 32-bit transforms: bit 0 forward (0.55 -> 0.63 of the roof), bit 1
    // inverse (three planes, 4 CTAs per SM: 0.51 -> 0.545); both on,
    // LB_NTT_PAIR overrides
    static int ntt_pairs();
    // smallest batch (polys / ciphertexts per launch) that runs the paired
    // kernels (LB_PAIR_MIN overrides; default 32)
    static uint32_t pair_min_count();
    // every prime of [first, first + count) is below 2^30
    bool primes_small(uint32_t first, uint32_t count) const {
        if (!tab32_.count) return false;  // no kernel-parameter table: 64-bit words
        for (uint32_t i = first; i < first + count; ++i)
            if (all_.at(i) >= kWord32Bound) return false;
        return true;
    }
    void ntt_forward(const LimbBatch& b, cudaStream_t s) const;
    void ntt_inverse(const LimbBatch& b, cudaStream_t s) const;

    BfvState* bfv() const { return bfv_.get(); }

    // Ciphertext ids select the encryption randomness (the
    // streams of a and e). They come from ONE counter per context, shared by
    // every evaluator, fork and session on it, so no two encryptions under
    // this context's keys reuse (a, e). Returns the first of `count` ids.
    uint64_t reserve_ciphertext_ids(uint64_t count) const { return next_ct_id_.fetch_add(count); }

private:
    Params prm_;
    uint32_t n_;
    int logn_;
    uint32_t dnum_;
    std::vector<uint64_t> all_;
    std::vector<uint64_t> psi_;
    std::vector<Modulus> mods_;
    std::vector<PrimeDev> host_primes_;
    DeviceBuffer d_tables32_;
    PrimeTab32 tab32_;
    cudaStream_t stream_ = nullptr;
    DeviceBuffer d_tables_;
    DeviceBuffer d_primes_;
    std::unique_ptr<BfvState> bfv_;
    mutable std::atomic<uint64_t> next_ct_id_{1};
    friend struct BfvState;
    friend void bfv_setup(Context&);
};

void bfv_setup(Context& cx);

dim3 grid_xyz(uint32_t x, uint64_t items);

}  // namespace lb
