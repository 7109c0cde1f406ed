#include <algorithm>
#include <cstdlib>

#include "bfv.hpp"
#include "context.hpp"
#include "host_math.hpp"

namespace lb {

std::atomic<uint64_t>& launch_counter() {
    static std::atomic<uint64_t> count{0};
    return count;
}

// x blocks per work item, `items` work items over grid.y (and z beyond 65535)
dim3 grid_xyz(uint32_t x, uint64_t items) {
    const uint64_t y = std::min<uint64_t>(items, 32768);
    const uint64_t z = (items + y - 1) / std::max<uint64_t>(y, 1);
    if (z > 65535) throw std::invalid_argument("batch too large for one launch");
    return dim3(x, static_cast<unsigned>(std::max<uint64_t>(y, 1)), static_cast<unsigned>(std::max<uint64_t>(z, 1)));
}

void Context::activate() const {
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess || cur != prm_.device) LB_CUDA(cudaSetDevice(prm_.device));
}

Context::Context(const Params& prm) : prm_(prm), n_(prm.n) {
    activate();
    if (n_ < 4096 || n_ > 32768 || (n_ & (n_ - 1)))
        throw std::invalid_argument("ring degree must be a power of two in [4096, 32768]");
    logn_ = host::ilog2(n_);
    if (prm.q.empty()) throw std::invalid_argument("need at least one ciphertext prime");
    all_.insert(all_.end(), prm.q.begin(), prm.q.end());
    all_.insert(all_.end(), prm.p.begin(), prm.p.end());
    all_.insert(all_.end(), prm.b.begin(), prm.b.end());
    all_.insert(all_.end(), prm.t.begin(), prm.t.end());
    for (size_t i = 0; i < all_.size(); ++i) {
        const uint64_t q = all_[i];
        if (q >= (uint64_t{1} << 62)) throw std::invalid_argument("primes must be below 2^62");
        if ((q - 1) % (2ull * n_)) throw std::invalid_argument("prime " + std::to_string(q) + " != 1 mod 2n");
        for (size_t j = 0; j < i; ++j)
            if (all_[j] == q) throw std::invalid_argument("repeated prime " + std::to_string(q));
    }
    dnum_ = prm.dnum ? prm.dnum : L();
    if (dnum_ > L()) throw std::invalid_argument("dnum exceeds the number of ciphertext primes");

    LB_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    {
        // keep freed temporaries cached in the stream-ordered pool
        int dev = 0;
        cudaMemPool_t pool;
        LB_CUDA(cudaGetDevice(&dev));
        LB_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
        uint64_t threshold = UINT64_MAX;
        LB_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
    }

    // Twiddle tables: per prime, fwd[N] and inv[N] (value, Shoup companion).
    const size_t per_prime = 2ull * n_;  // ulonglong2 entries
    std::vector<ulonglong2> tables(per_prime * all_.size());
    std::vector<PrimeDev> devs(all_.size());
    d_tables_ = DeviceBuffer(tables.size() * sizeof(ulonglong2), stream_);
    auto* d_tab = d_tables_.get<ulonglong2>();
    for (size_t i = 0; i < all_.size(); ++i) {
        const uint64_t q = all_[i];
        const uint64_t psi = host::root_of_unity(q, 2ull * n_);
        const uint64_t psi_inv = host::invm(psi, q);
        psi_.push_back(psi);
        std::vector<uint64_t> pw(n_), ipw(n_);
        uint64_t a = 1, b = 1;
        for (uint32_t k = 0; k < n_; ++k) {
            pw[k] = a;
            ipw[k] = b;
            a = host::mulm(a, psi, q);
            b = host::mulm(b, psi_inv, q);
        }
        ulonglong2* fwd = &tables[per_prime * i];
        ulonglong2* inv = fwd + n_;
        for (uint32_t k = 0; k < n_; ++k) {
            const uint64_t w = pw[host::bitrev(k, logn_)];
            const uint64_t iw = ipw[host::bitrev(k, logn_)];
            fwd[k] = make_ulonglong2(w, shoup_companion(w, q));
            inv[k] = make_ulonglong2(iw, shoup_companion(iw, q));
        }
        Modulus m;
        m.q = q;
        const unsigned __int128 ratio = ~static_cast<unsigned __int128>(0) / q;  // floor((2^128-1)/q)
        m.ratio_lo = static_cast<uint64_t>(ratio);
        m.ratio_hi = static_cast<uint64_t>(ratio >> 64);
        mods_.push_back(m);
        PrimeDev& d = devs[i];
        d.q = q;
        d.ratio_lo = m.ratio_lo;
        d.ratio_hi = m.ratio_hi;
        d.fwd = d_tab + per_prime * i;
        d.inv = d_tab + per_prime * i + n_;
        const uint64_t ninv = host::invm(n_, q);
        d.ninv = ninv;
        d.ninv_shoup = shoup_companion(ninv, q);
        d.inv1n = host::mulm(inv[1].x, ninv, q);
        d.inv1n_shoup = shoup_companion(d.inv1n, q);
    }
    LB_CUDA(cudaMemcpyAsync(d_tab, tables.data(), tables.size() * sizeof(ulonglong2), cudaMemcpyHostToDevice,
                            stream_));
    // 32-bit twiddles for the primes below 2^30
    {
        std::vector<uint32_t> small;
        for (size_t i = 0; i < all_.size(); ++i)
            if (all_[i] < kWord32Bound) small.push_back(static_cast<uint32_t>(i));
        if (!small.empty()) {
            std::vector<uint2> t32(per_prime * small.size());
            d_tables32_ = DeviceBuffer(t32.size() * sizeof(uint2), stream_);
            auto* d32 = d_tables32_.get<uint2>();
            for (size_t j = 0; j < small.size(); ++j) {
                const uint32_t i = small[j];
                const uint64_t q = all_[i];
                const ulonglong2* src = &tables[per_prime * i];
                for (size_t k = 0; k < per_prime; ++k)
                    t32[per_prime * j + k] = make_uint2(static_cast<uint32_t>(src[k].x), shoup_companion32(src[k].x, q));
                PrimeDev& d = devs[i];
                d.fwd32 = d32 + per_prime * j;
                d.inv32 = d32 + per_prime * j + n_;
                d.ninv32 = make_uint2(static_cast<uint32_t>(d.ninv), shoup_companion32(d.ninv, q));
                d.inv1n32 = make_uint2(static_cast<uint32_t>(d.inv1n), shoup_companion32(d.inv1n, q));
            }
            LB_CUDA(cudaMemcpyAsync(d32, t32.data(), t32.size() * sizeof(uint2), cudaMemcpyHostToDevice, stream_));
            // kernel-parameter table (q, table slot) of the 32-bit primes
            if (all_.size() <= size_t(kTabPrimes)) {
                tab32_.tw = d32;
                tab32_.count = static_cast<uint32_t>(all_.size());
                for (size_t j = 0; j < small.size(); ++j) {
                    tab32_.q[small[j]] = static_cast<uint32_t>(all_[small[j]]);
                    tab32_.slot[small[j]] = static_cast<uint8_t>(j);
                }
            }
        }
    }
    host_primes_ = devs;
    d_primes_ = DeviceBuffer(devs.size() * sizeof(PrimeDev), stream_);
    LB_CUDA(cudaMemcpyAsync(d_primes_.get(), devs.data(), devs.size() * sizeof(PrimeDev), cudaMemcpyHostToDevice,
                            stream_));
    LB_CUDA(cudaStreamSynchronize(stream_));
    bfv_setup(*this);
}

Context::~Context() {
    bfv_.reset();
    d_primes_ = DeviceBuffer();
    d_tables_ = DeviceBuffer();
    d_tables32_ = DeviceBuffer();
    if (stream_) {
        cudaStreamSynchronize(stream_);
        cudaStreamDestroy(stream_);
    }
}

namespace {

template <int LOGN, class W, class St, bool MAPPED, int NT>
void launch_ntt_m(const LimbBatch& b, const PrimeDev* primes, const PrimeTab32& tab, bool inverse, cudaStream_t s) {
    using S = NttShape<LOGN>;
    const uint64_t limbs = static_cast<uint64_t>(b.polys) * b.limbs;
    if (limbs == 0) return;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid_xyz(b.limbs * S::CL, b.polys / NT);
    cfg.blockDim = dim3(S::T);
    cfg.dynamicSmemBytes = inverse ? ntt_inverse_smem<LOGN, W, NT>() : 0;
    cfg.stream = s;
    if (inverse) {
        static const bool configured = [] {
            LB_CUDA(cudaFuncSetAttribute(ntt_inverse_kernel<LOGN, W, St, MAPPED, NT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(ntt_inverse_smem<LOGN, W, NT>())));
            return true;
        }();
        (void)configured;
    }
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = S::CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (inverse)
        LB_CUDA(cudaLaunchKernelEx(&cfg, ntt_inverse_kernel<LOGN, W, St, MAPPED, NT>, b, primes, tab));
    else
        LB_CUDA(cudaLaunchKernelEx(&cfg, ntt_forward_kernel<LOGN, W, St, MAPPED, NT>, b, primes, tab));
    launch_counter().fetch_add(1, std::memory_order_relaxed);
}

// the batch's polys [first, first + count)
template <class St>
LimbBatch sub_batch(const LimbBatch& b, uint32_t first, uint32_t count) {
    LimbBatch o = b;
    o.polys = count;
    o.data = reinterpret_cast<uint64_t*>(reinterpret_cast<St*>(b.data) + uint64_t(first) * b.poly_stride);
    if (b.src) o.src = reinterpret_cast<const uint64_t*>(reinterpret_cast<const St*>(b.src) + uint64_t(first) * b.src_stride);
    return o;
}

template <int LOGN, class W, class St>
void launch_ntt(const LimbBatch& b, const PrimeDev* primes, const PrimeTab32& tab, bool inverse, cudaStream_t s) {
    if (b.prime_map) {
        launch_ntt_m<LOGN, W, St, true, 1>(b, primes, tab, inverse, s);
        return;
    }
    // 32-bit word transforms run two polys per cluster (shared twiddles);
    // an odd poly is left to the single-transform instance
    if constexpr (sizeof(W) == 4 && inv_push<LOGN>()) {
        // (small batches stay unpaired: half as many clusters under-fill the
        // GPU — single-image latency 7.07 vs 7.15 ms, two images 13.1 vs 13.9)
        if ((Context::ntt_pairs() & (inverse ? 2 : 1)) && b.polys >= Context::pair_min_count()) {
            const uint32_t even = b.polys & ~1u;
            launch_ntt_m<LOGN, W, St, false, 2>(sub_batch<St>(b, 0, even), primes, tab, inverse, s);
            if (b.polys & 1u) launch_ntt_m<LOGN, W, St, false, 1>(sub_batch<St>(b, even, 1), primes, tab, inverse, s);
            return;
        }
    }
    launch_ntt_m<LOGN, W, St, false, 1>(b, primes, tab, inverse, s);
}

template <class W, class St>
void dispatch_ntt(int logn, const LimbBatch& b, const PrimeDev* primes, const PrimeTab32& tab, bool inverse,
                  cudaStream_t s) {
    switch (logn) {
        case 12: launch_ntt<12, W, St>(b, primes, tab, inverse, s); break;
        case 13: launch_ntt<13, W, St>(b, primes, tab, inverse, s); break;
        case 14: launch_ntt<14, W, St>(b, primes, tab, inverse, s); break;
        case 15: launch_ntt<15, W, St>(b, primes, tab, inverse, s); break;
        default: throw std::invalid_argument("unsupported ring degree");
    }
}

void dispatch_ntt(bool word32, int logn, const LimbBatch& b, const PrimeDev* primes, const PrimeTab32& tab,
                  bool inverse, cudaStream_t s) {
    if (b.packed32) {
        if (!word32) throw std::invalid_argument("packed 32-bit limbs need primes below 2^30");
        dispatch_ntt<uint32_t, uint32_t>(logn, b, primes, tab, inverse, s);
    } else if (word32) {
        dispatch_ntt<uint32_t, uint64_t>(logn, b, primes, tab, inverse, s);
    } else {
        dispatch_ntt<uint64_t, uint64_t>(logn, b, primes, tab, inverse, s);
    }
}

void check_batch(const Context& cx, const LimbBatch& b) {
    if (!b.prime_map && b.first_prime + b.limbs > cx.prime_count())
        throw std::invalid_argument("limb primes out of range");
    if (b.prime_map && b.map_period == 0) throw std::invalid_argument("prime map without period");
    if (b.poly_stride < static_cast<uint64_t>(b.limbs) * cx.n())
        throw std::invalid_argument("poly stride smaller than limbs * n");
}

}  // namespace

bool Context::word32_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("LB_WORD32");
        return !(e && e[0] == '0');
    }();
    return on;
}

int Context::ntt_pairs() {
    static const int mask = [] {
        const char* e = std::getenv("LB_NTT_PAIR");
        return e ? std::atoi(e) : 3;
    }();
    return mask;
}

uint32_t Context::pair_min_count() {
    static const uint32_t v = [] {
        const char* e = std::getenv("LB_PAIR_MIN");
        return e ? static_cast<uint32_t>(std::max(2, std::atoi(e))) : 32u;
    }();
    return v;
}

bool Context::batch_word32(const LimbBatch& b) const {
    if (!word32_enabled() || !tab32_.count) return false;
    if (b.prime_map) return b.map_small;
    if (b.last_stage && !b.last_stage32) return false;
    for (uint32_t l = 0; l < b.limbs; ++l)
        if (all_[b.first_prime + l] >= kWord32Bound) return false;
    return true;
}

void Context::ntt_forward(const LimbBatch& b, cudaStream_t s) const {
    check_batch(*this, b);
    dispatch_ntt(batch_word32(b), logn_, b, dev_primes(), tab32_, false, s);
}

void Context::ntt_inverse(const LimbBatch& b, cudaStream_t s) const {
    check_batch(*this, b);
    dispatch_ntt(batch_word32(b), logn_, b, dev_primes(), tab32_, true, s);
}

}  // namespace lb
