// Stand-in for boost::multiprecision::cpp_int, written for this repo.
//
// TEST INFRASTRUCTURE ONLY. The reference (packnn, /root/reference/proj)
// includes <boost/multiprecision/cpp_int.hpp> (proj/include/packnn/bigint.hpp:3)
// but Boost is absent from this image, so oracle/Makefile compiles the
// reference sources against this header instead. It implements only what the
// reference uses: signed arbitrary-precision integers with + - * / % (truncated
// division, C++ sign rules like cpp_int), unary -, <<, >>, |, comparisons,
// explicit conversion to built-in integers, and str().
//
// Representation: sign flag + little-endian magnitude of 32-bit limbs with no
// leading zero limbs (zero is the empty vector, never negative).
#pragma once

#include <algorithm>
#include <compare>
#include <cstdint>
#include <ostream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace boost {
namespace multiprecision {

class cpp_int {
public:
    cpp_int() = default;

    template <class T, std::enable_if_t<std::is_integral_v<T>, int> = 0>
    cpp_int(T v) {  // NOLINT(google-explicit-constructor): cpp_int converts implicitly
        if constexpr (std::is_signed_v<T>) {
            if (v < 0) {
                neg_ = true;
                // Negate through unsigned arithmetic so INT64_MIN is safe.
                set_u128(static_cast<unsigned __int128>(-(static_cast<__int128>(v))));
                return;
            }
        }
        set_u128(static_cast<unsigned __int128>(v));
    }
    cpp_int(unsigned __int128 v) { set_u128(v); }
    cpp_int(__int128 v) {
        if (v < 0) {
            neg_ = true;
            set_u128(static_cast<unsigned __int128>(-v));
        } else {
            set_u128(static_cast<unsigned __int128>(v));
        }
    }
    explicit cpp_int(const char* s) { parse(s); }
    explicit cpp_int(const std::string& s) { parse(s.c_str()); }

    // ---- conversion -------------------------------------------------------
    template <class T, std::enable_if_t<std::is_integral_v<T>, int> = 0>
    explicit operator T() const {
        // Low 64 bits of the magnitude, then the sign applied modulo 2^64,
        // matching cpp_int's truncating conversion for in-range values.
        uint64_t lo = 0;
        if (!mag_.empty()) lo = mag_[0];
        if (mag_.size() > 1) lo |= static_cast<uint64_t>(mag_[1]) << 32;
        if (neg_) lo = ~lo + 1;
        return static_cast<T>(lo);
    }
    explicit operator bool() const { return !mag_.empty(); }
    explicit operator double() const {
        double r = 0;
        for (size_t i = mag_.size(); i-- > 0;) r = r * 4294967296.0 + mag_[i];
        return neg_ ? -r : r;
    }

    std::string str() const {
        if (mag_.empty()) return "0";
        std::vector<uint32_t> m = mag_;
        std::string digits;
        while (!m.empty()) {
            uint32_t rem = divmod_small_inplace(m, 1000000000u);
            for (int i = 0; i < 9; ++i) {
                digits.push_back(static_cast<char>('0' + rem % 10));
                rem /= 10;
                if (m.empty() && rem == 0) break;
            }
        }
        while (digits.size() > 1 && digits.back() == '0') digits.pop_back();
        if (neg_) digits.push_back('-');
        std::reverse(digits.begin(), digits.end());
        return digits;
    }

    // ---- arithmetic ---------------------------------------------------------
    friend cpp_int operator-(const cpp_int& a) {
        cpp_int r = a;
        if (!r.mag_.empty()) r.neg_ = !r.neg_;
        return r;
    }
    friend cpp_int operator+(const cpp_int& a, const cpp_int& b) { return add_signed(a, b, false); }
    friend cpp_int operator-(const cpp_int& a, const cpp_int& b) { return add_signed(a, b, true); }
    friend cpp_int operator*(const cpp_int& a, const cpp_int& b) {
        cpp_int r;
        if (a.mag_.empty() || b.mag_.empty()) return r;
        r.mag_.assign(a.mag_.size() + b.mag_.size(), 0);
        for (size_t i = 0; i < a.mag_.size(); ++i) {
            uint64_t carry = 0;
            const uint64_t ai = a.mag_[i];
            for (size_t j = 0; j < b.mag_.size(); ++j) {
                uint64_t cur = ai * b.mag_[j] + r.mag_[i + j] + carry;
                r.mag_[i + j] = static_cast<uint32_t>(cur);
                carry = cur >> 32;
            }
            size_t k = i + b.mag_.size();
            while (carry) {
                uint64_t cur = static_cast<uint64_t>(r.mag_[k]) + carry;
                r.mag_[k] = static_cast<uint32_t>(cur);
                carry = cur >> 32;
                ++k;
            }
        }
        r.trim();
        r.neg_ = !r.mag_.empty() && (a.neg_ != b.neg_);
        return r;
    }
    // Truncated division (quotient rounds toward zero), remainder takes the
    // dividend's sign, as for built-in integers and cpp_int.
    friend cpp_int operator/(const cpp_int& a, const cpp_int& b) {
        cpp_int q, r;
        divmod(a, b, q, r);
        return q;
    }
    friend cpp_int operator%(const cpp_int& a, const cpp_int& b) {
        cpp_int q, r;
        divmod(a, b, q, r);
        return r;
    }
    friend cpp_int operator<<(const cpp_int& a, unsigned s) {
        cpp_int r;
        if (a.mag_.empty()) return r;
        const unsigned limbs = s / 32, bits = s % 32;
        r.mag_.assign(a.mag_.size() + limbs + 1, 0);
        for (size_t i = 0; i < a.mag_.size(); ++i) {
            uint64_t v = static_cast<uint64_t>(a.mag_[i]) << bits;
            r.mag_[i + limbs] |= static_cast<uint32_t>(v);
            r.mag_[i + limbs + 1] |= static_cast<uint32_t>(v >> 32);
        }
        r.trim();
        r.neg_ = a.neg_;
        return r;
    }
    friend cpp_int operator>>(const cpp_int& a, unsigned s) {
        // Magnitude shift (only used on non-negative values in this repo).
        cpp_int r;
        const unsigned limbs = s / 32, bits = s % 32;
        if (limbs >= a.mag_.size()) return r;
        r.mag_.assign(a.mag_.size() - limbs, 0);
        for (size_t i = limbs; i < a.mag_.size(); ++i) {
            uint64_t v = a.mag_[i];
            if (i + 1 < a.mag_.size()) v |= static_cast<uint64_t>(a.mag_[i + 1]) << 32;
            r.mag_[i - limbs] = static_cast<uint32_t>(v >> bits);
        }
        r.trim();
        r.neg_ = a.neg_ && !r.mag_.empty();
        return r;
    }
    friend cpp_int operator|(const cpp_int& a, const cpp_int& b) {
        // Bitwise OR on magnitudes (the reference only ORs non-negative values).
        cpp_int r;
        r.mag_.assign(std::max(a.mag_.size(), b.mag_.size()), 0);
        for (size_t i = 0; i < a.mag_.size(); ++i) r.mag_[i] |= a.mag_[i];
        for (size_t i = 0; i < b.mag_.size(); ++i) r.mag_[i] |= b.mag_[i];
        r.trim();
        r.neg_ = (a.neg_ || b.neg_) && !r.mag_.empty();
        return r;
    }

    cpp_int& operator+=(const cpp_int& b) { return *this = *this + b; }
    cpp_int& operator-=(const cpp_int& b) { return *this = *this - b; }
    cpp_int& operator*=(const cpp_int& b) { return *this = *this * b; }
    cpp_int& operator/=(const cpp_int& b) { return *this = *this / b; }
    cpp_int& operator%=(const cpp_int& b) { return *this = *this % b; }
    cpp_int& operator<<=(unsigned s) { return *this = *this << s; }
    cpp_int& operator>>=(unsigned s) { return *this = *this >> s; }
    cpp_int& operator|=(const cpp_int& b) { return *this = *this | b; }
    cpp_int& operator++() { return *this += 1; }
    cpp_int& operator--() { return *this -= 1; }

    // ---- comparison ---------------------------------------------------------
    friend bool operator==(const cpp_int& a, const cpp_int& b) {
        return a.neg_ == b.neg_ && a.mag_ == b.mag_;
    }
    friend std::strong_ordering operator<=>(const cpp_int& a, const cpp_int& b) {
        if (a.neg_ != b.neg_) return a.neg_ ? std::strong_ordering::less : std::strong_ordering::greater;
        int c = cmp_mag(a.mag_, b.mag_);
        if (a.neg_) c = -c;
        return c < 0 ? std::strong_ordering::less
                     : (c > 0 ? std::strong_ordering::greater : std::strong_ordering::equal);
    }

    friend std::ostream& operator<<(std::ostream& os, const cpp_int& v) { return os << v.str(); }

    bool is_negative() const { return neg_; }

private:
    bool neg_ = false;
    std::vector<uint32_t> mag_;

    void set_u128(unsigned __int128 v) {
        mag_.clear();
        while (v) {
            mag_.push_back(static_cast<uint32_t>(v));
            v >>= 32;
        }
        if (mag_.empty()) neg_ = false;
    }
    void trim() {
        while (!mag_.empty() && mag_.back() == 0) mag_.pop_back();
        if (mag_.empty()) neg_ = false;
    }
    void parse(const char* s) {
        mag_.clear();
        neg_ = false;
        bool negative = false;
        if (*s == '-') {
            negative = true;
            ++s;
        } else if (*s == '+') {
            ++s;
        }
        for (; *s; ++s) {
            if (*s < '0' || *s > '9') throw std::invalid_argument("cpp_int: bad digit");
            mul_small_add(10, static_cast<uint32_t>(*s - '0'));
        }
        trim();
        neg_ = negative && !mag_.empty();
    }
    void mul_small_add(uint32_t m, uint32_t a) {
        uint64_t carry = a;
        for (auto& limb : mag_) {
            uint64_t cur = static_cast<uint64_t>(limb) * m + carry;
            limb = static_cast<uint32_t>(cur);
            carry = cur >> 32;
        }
        if (carry) mag_.push_back(static_cast<uint32_t>(carry));
    }
    static uint32_t divmod_small_inplace(std::vector<uint32_t>& m, uint32_t d) {
        uint64_t rem = 0;
        for (size_t i = m.size(); i-- > 0;) {
            uint64_t cur = (rem << 32) | m[i];
            m[i] = static_cast<uint32_t>(cur / d);
            rem = cur % d;
        }
        while (!m.empty() && m.back() == 0) m.pop_back();
        return static_cast<uint32_t>(rem);
    }
    static int cmp_mag(const std::vector<uint32_t>& a, const std::vector<uint32_t>& b) {
        if (a.size() != b.size()) return a.size() < b.size() ? -1 : 1;
        for (size_t i = a.size(); i-- > 0;) {
            if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
        }
        return 0;
    }
    static std::vector<uint32_t> add_mag(const std::vector<uint32_t>& a, const std::vector<uint32_t>& b) {
        const auto& big = a.size() >= b.size() ? a : b;
        const auto& small = a.size() >= b.size() ? b : a;
        std::vector<uint32_t> r(big.size() + 1, 0);
        uint64_t carry = 0;
        for (size_t i = 0; i < big.size(); ++i) {
            uint64_t cur = static_cast<uint64_t>(big[i]) + (i < small.size() ? small[i] : 0) + carry;
            r[i] = static_cast<uint32_t>(cur);
            carry = cur >> 32;
        }
        r[big.size()] = static_cast<uint32_t>(carry);
        while (!r.empty() && r.back() == 0) r.pop_back();
        return r;
    }
    // |a| - |b| with |a| >= |b|.
    static std::vector<uint32_t> sub_mag(const std::vector<uint32_t>& a, const std::vector<uint32_t>& b) {
        std::vector<uint32_t> r(a.size(), 0);
        int64_t borrow = 0;
        for (size_t i = 0; i < a.size(); ++i) {
            int64_t cur = static_cast<int64_t>(a[i]) - (i < b.size() ? b[i] : 0) - borrow;
            borrow = cur < 0 ? 1 : 0;
            if (cur < 0) cur += (int64_t{1} << 32);
            r[i] = static_cast<uint32_t>(cur);
        }
        while (!r.empty() && r.back() == 0) r.pop_back();
        return r;
    }
    static cpp_int add_signed(const cpp_int& a, const cpp_int& b, bool negate_b) {
        const bool bneg = negate_b ? (!b.neg_ && !b.mag_.empty()) : b.neg_;
        cpp_int r;
        if (a.neg_ == bneg) {
            r.mag_ = add_mag(a.mag_, b.mag_);
            r.neg_ = a.neg_;
        } else {
            int c = cmp_mag(a.mag_, b.mag_);
            if (c == 0) return r;
            if (c > 0) {
                r.mag_ = sub_mag(a.mag_, b.mag_);
                r.neg_ = a.neg_;
            } else {
                r.mag_ = sub_mag(b.mag_, a.mag_);
                r.neg_ = bneg;
            }
        }
        r.trim();
        return r;
    }
    // Knuth algorithm D on magnitudes; signs follow truncated division.
    static void divmod(const cpp_int& a, const cpp_int& b, cpp_int& q, cpp_int& r) {
        if (b.mag_.empty()) throw std::domain_error("cpp_int: division by zero");
        q = cpp_int();
        r = cpp_int();
        if (cmp_mag(a.mag_, b.mag_) < 0) {
            r = a;
            return;
        }
        if (b.mag_.size() == 1) {
            std::vector<uint32_t> m = a.mag_;
            uint32_t rem = divmod_small_inplace(m, b.mag_[0]);
            q.mag_ = std::move(m);
            r.set_u128(rem);
        } else {
            const std::vector<uint32_t>& u0 = a.mag_;
            const std::vector<uint32_t>& v0 = b.mag_;
            const size_t n = v0.size(), m = u0.size() - n;
            int s = __builtin_clz(v0.back());
            std::vector<uint32_t> v(n), u(u0.size() + 1);
            for (size_t i = n; i-- > 0;) {
                uint64_t hi = static_cast<uint64_t>(v0[i]) << s;
                uint32_t lo = (i > 0 && s) ? static_cast<uint32_t>(static_cast<uint64_t>(v0[i - 1]) >> (32 - s)) : 0;
                v[i] = static_cast<uint32_t>(hi) | lo;
            }
            u[u0.size()] = s ? static_cast<uint32_t>(static_cast<uint64_t>(u0.back()) >> (32 - s)) : 0;
            for (size_t i = u0.size(); i-- > 0;) {
                uint64_t hi = static_cast<uint64_t>(u0[i]) << s;
                uint32_t lo = (i > 0 && s) ? static_cast<uint32_t>(static_cast<uint64_t>(u0[i - 1]) >> (32 - s)) : 0;
                u[i] = static_cast<uint32_t>(hi) | lo;
            }
            std::vector<uint32_t> qq(m + 1, 0);
            const uint64_t base = uint64_t{1} << 32;
            for (size_t j = m + 1; j-- > 0;) {
                uint64_t num = (static_cast<uint64_t>(u[j + n]) << 32) | u[j + n - 1];
                uint64_t qhat = num / v[n - 1];
                uint64_t rhat = num % v[n - 1];
                while (qhat >= base || qhat * v[n - 2] > ((rhat << 32) | u[j + n - 2])) {
                    --qhat;
                    rhat += v[n - 1];
                    if (rhat >= base) break;
                }
                int64_t borrow = 0;
                uint64_t carry = 0;
                for (size_t i = 0; i < n; ++i) {
                    uint64_t p = qhat * v[i] + carry;
                    carry = p >> 32;
                    int64_t t = static_cast<int64_t>(u[i + j]) - borrow - static_cast<int64_t>(p & 0xffffffffu);
                    u[i + j] = static_cast<uint32_t>(t);
                    borrow = t < 0 ? 1 : 0;
                }
                int64_t t = static_cast<int64_t>(u[j + n]) - borrow - static_cast<int64_t>(carry);
                u[j + n] = static_cast<uint32_t>(t);
                if (t < 0) {
                    --qhat;
                    uint64_t c = 0;
                    for (size_t i = 0; i < n; ++i) {
                        uint64_t sum = static_cast<uint64_t>(u[i + j]) + v[i] + c;
                        u[i + j] = static_cast<uint32_t>(sum);
                        c = sum >> 32;
                    }
                    u[j + n] = static_cast<uint32_t>(static_cast<uint64_t>(u[j + n]) + c);
                }
                qq[j] = static_cast<uint32_t>(qhat);
            }
            q.mag_ = std::move(qq);
            q.trim();
            std::vector<uint32_t> rem(n, 0);
            for (size_t i = 0; i < n; ++i) {
                uint64_t lo = static_cast<uint64_t>(u[i]) >> s;
                uint64_t hi = (s && i + 1 <= n) ? (static_cast<uint64_t>(u[i + 1]) << (32 - s)) : 0;
                rem[i] = static_cast<uint32_t>(lo | hi);
            }
            r.mag_ = std::move(rem);
            r.trim();
        }
        q.neg_ = !q.mag_.empty() && (a.neg_ != b.neg_);
        r.neg_ = !r.mag_.empty() && a.neg_;
    }
};

}  // namespace multiprecision
}  // namespace boost
