// ORACLE TEST INFRASTRUCTURE — not product code.
//
// Minimal stand-in for boost::multiprecision::cpp_int, covering exactly the
// surface the reference simulator uses (rational.cpp:16-37,
// bufpool.cpp:24-26, engine_internal.hpp:56-135). Boost is not installed in
// this image; the reference needs an arbitrary-precision integer because its
// exact model clock reaches ~224-bit intermediates.
//
// Representation: sign + magnitude as little-endian base-2^32 limbs, no
// leading zero limbs (zero == empty magnitude, non-negative).
#pragma once

#include <algorithm>
#include <cmath>
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
  using limb = std::uint32_t;

  cpp_int() = default;
  template <typename T, typename = std::enable_if_t<std::is_integral_v<T>>>
  cpp_int(T v) {  // NOLINT(google-explicit-constructor): boost allows implicit
    if constexpr (std::is_signed_v<T>) {
      if (v < 0) {
        neg_ = true;
        // two's complement safe magnitude
        std::uint64_t m = static_cast<std::uint64_t>(-(static_cast<__int128>(v)));
        set_mag(m);
        return;
      }
    }
    set_mag(static_cast<std::uint64_t>(v));
  }

  bool is_zero() const { return mag_.empty(); }
  int sign() const { return is_zero() ? 0 : (neg_ ? -1 : 1); }

  template <typename T>
  T convert_to() const {
    if constexpr (std::is_floating_point_v<T>) {
      return static_cast<T>(to_double_rne());
    } else {
      // integral: low 64 bits of magnitude, sign applied (values used are small)
      std::uint64_t m = 0;
      if (mag_.size() > 0) m |= mag_[0];
      if (mag_.size() > 1) m |= static_cast<std::uint64_t>(mag_[1]) << 32;
      if (neg_) return static_cast<T>(-static_cast<__int128>(m));
      return static_cast<T>(m);
    }
  }

  // --- arithmetic -----------------------------------------------------------
  friend cpp_int operator+(const cpp_int& a, const cpp_int& b) {
    if (a.neg_ == b.neg_) {
      cpp_int r;
      r.mag_ = add_mag(a.mag_, b.mag_);
      r.neg_ = a.neg_;
      r.fix();
      return r;
    }
    int c = cmp_mag(a.mag_, b.mag_);
    cpp_int r;
    if (c == 0) return r;
    if (c > 0) {
      r.mag_ = sub_mag(a.mag_, b.mag_);
      r.neg_ = a.neg_;
    } else {
      r.mag_ = sub_mag(b.mag_, a.mag_);
      r.neg_ = b.neg_;
    }
    r.fix();
    return r;
  }
  friend cpp_int operator-(const cpp_int& a) {
    cpp_int r = a;
    if (!r.is_zero()) r.neg_ = !r.neg_;
    return r;
  }
  friend cpp_int operator-(const cpp_int& a, const cpp_int& b) { return a + (-b); }
  friend cpp_int operator*(const cpp_int& a, const cpp_int& b) {
    cpp_int r;
    if (a.is_zero() || b.is_zero()) return r;
    r.mag_.assign(a.mag_.size() + b.mag_.size(), 0);
    for (std::size_t i = 0; i < a.mag_.size(); ++i) {
      std::uint64_t carry = 0;
      for (std::size_t j = 0; j < b.mag_.size(); ++j) {
        std::uint64_t cur = static_cast<std::uint64_t>(a.mag_[i]) * b.mag_[j] + r.mag_[i + j] + carry;
        r.mag_[i + j] = static_cast<limb>(cur);
        carry = cur >> 32;
      }
      std::size_t k = i + b.mag_.size();
      while (carry) {
        std::uint64_t cur = static_cast<std::uint64_t>(r.mag_[k]) + carry;
        r.mag_[k] = static_cast<limb>(cur);
        carry = cur >> 32;
        ++k;
      }
    }
    r.neg_ = a.neg_ != b.neg_;
    r.fix();
    return r;
  }
  // Truncating division (C++ semantics), as boost::multiprecision does.
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
  friend cpp_int operator<<(const cpp_int& a, int s) {
    if (s < 0) throw std::domain_error("negative shift");
    cpp_int r;
    if (a.is_zero()) return r;
    std::size_t limbs = static_cast<std::size_t>(s) / 32;
    int bits = s % 32;
    r.mag_.assign(limbs, 0);
    limb carry = 0;
    for (limb x : a.mag_) {
      if (bits == 0) {
        r.mag_.push_back(x);
      } else {
        r.mag_.push_back((x << bits) | carry);
        carry = x >> (32 - bits);
      }
    }
    if (carry) r.mag_.push_back(carry);
    r.neg_ = a.neg_;
    r.fix();
    return r;
  }
  cpp_int& operator+=(const cpp_int& b) { return *this = *this + b; }
  cpp_int& operator-=(const cpp_int& b) { return *this = *this - b; }
  cpp_int& operator*=(const cpp_int& b) { return *this = *this * b; }
  cpp_int& operator/=(const cpp_int& b) { return *this = *this / b; }
  cpp_int& operator%=(const cpp_int& b) { return *this = *this % b; }

  // --- comparison -------------------------------------------------------------
  friend int compare(const cpp_int& a, const cpp_int& b) {
    if (a.neg_ != b.neg_) return a.neg_ ? -1 : 1;
    int c = cmp_mag(a.mag_, b.mag_);
    return a.neg_ ? -c : c;
  }
  friend bool operator==(const cpp_int& a, const cpp_int& b) { return compare(a, b) == 0; }
  friend bool operator!=(const cpp_int& a, const cpp_int& b) { return compare(a, b) != 0; }
  friend bool operator<(const cpp_int& a, const cpp_int& b) { return compare(a, b) < 0; }
  friend bool operator>(const cpp_int& a, const cpp_int& b) { return compare(a, b) > 0; }
  friend bool operator<=(const cpp_int& a, const cpp_int& b) { return compare(a, b) <= 0; }
  friend bool operator>=(const cpp_int& a, const cpp_int& b) { return compare(a, b) >= 0; }

  friend std::ostream& operator<<(std::ostream& os, const cpp_int& a) { return os << a.str(); }

  std::string str() const {
    if (is_zero()) return "0";
    std::vector<limb> m = mag_;
    std::string digits;
    while (!m.empty()) {
      std::uint64_t rem = 0;
      for (std::size_t i = m.size(); i-- > 0;) {
        std::uint64_t cur = (rem << 32) | m[i];
        m[i] = static_cast<limb>(cur / 1000000000u);
        rem = cur % 1000000000u;
      }
      while (!m.empty() && m.back() == 0) m.pop_back();
      for (int k = 0; k < 9; ++k) {
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

  const std::vector<limb>& magnitude() const { return mag_; }
  bool negative() const { return neg_; }

 private:
  void set_mag(std::uint64_t m) {
    mag_.clear();
    while (m) {
      mag_.push_back(static_cast<limb>(m));
      m >>= 32;
    }
    if (mag_.empty()) neg_ = false;
  }
  void fix() {
    while (!mag_.empty() && mag_.back() == 0) mag_.pop_back();
    if (mag_.empty()) neg_ = false;
  }
  static int cmp_mag(const std::vector<limb>& a, const std::vector<limb>& b) {
    if (a.size() != b.size()) return a.size() < b.size() ? -1 : 1;
    for (std::size_t i = a.size(); i-- > 0;)
      if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
    return 0;
  }
  static std::vector<limb> add_mag(const std::vector<limb>& a, const std::vector<limb>& b) {
    const auto& x = a.size() >= b.size() ? a : b;
    const auto& y = a.size() >= b.size() ? b : a;
    std::vector<limb> r(x.size() + 1, 0);
    std::uint64_t carry = 0;
    for (std::size_t i = 0; i < x.size(); ++i) {
      std::uint64_t cur = static_cast<std::uint64_t>(x[i]) + (i < y.size() ? y[i] : 0) + carry;
      r[i] = static_cast<limb>(cur);
      carry = cur >> 32;
    }
    r[x.size()] = static_cast<limb>(carry);
    return r;
  }
  // requires |a| >= |b|
  static std::vector<limb> sub_mag(const std::vector<limb>& a, const std::vector<limb>& b) {
    std::vector<limb> r(a.size(), 0);
    std::int64_t borrow = 0;
    for (std::size_t i = 0; i < a.size(); ++i) {
      std::int64_t cur = static_cast<std::int64_t>(a[i]) - (i < b.size() ? b[i] : 0) - borrow;
      borrow = cur < 0 ? 1 : 0;
      if (cur < 0) cur += (static_cast<std::int64_t>(1) << 32);
      r[i] = static_cast<limb>(cur);
    }
    return r;
  }
  static int bitlen(const std::vector<limb>& m) {
    if (m.empty()) return 0;
    return static_cast<int>((m.size() - 1) * 32) + (32 - __builtin_clz(m.back()));
  }
  static bool test_bit(const std::vector<limb>& m, int i) {
    std::size_t w = static_cast<std::size_t>(i) / 32;
    return w < m.size() && ((m[w] >> (i % 32)) & 1u);
  }
  // Shift-subtract long division on magnitudes (operand widths here are a few
  // hundred bits at most, so the simple algorithm is adequate).
  static void divmod(const cpp_int& a, const cpp_int& b, cpp_int& q, cpp_int& r) {
    if (b.is_zero()) throw std::overflow_error("cpp_int: division by zero");
    q = cpp_int();
    r = cpp_int();
    if (cmp_mag(a.mag_, b.mag_) < 0) {
      r = a;
      return;
    }
    if (b.mag_.size() == 1) {
      std::uint64_t d = b.mag_[0], rem = 0;
      q.mag_.assign(a.mag_.size(), 0);
      for (std::size_t i = a.mag_.size(); i-- > 0;) {
        std::uint64_t cur = (rem << 32) | a.mag_[i];
        q.mag_[i] = static_cast<limb>(cur / d);
        rem = cur % d;
      }
      r.set_mag(rem);
    } else {
      int n = bitlen(a.mag_);
      q.mag_.assign(a.mag_.size(), 0);
      cpp_int bb;
      bb.mag_ = b.mag_;
      for (int i = n - 1; i >= 0; --i) {
        r = r << 1;
        if (test_bit(a.mag_, i)) {
          if (r.mag_.empty()) r.mag_.push_back(0);
          r.mag_[0] |= 1u;
        }
        if (cmp_mag(r.mag_, bb.mag_) >= 0) {
          r.mag_ = sub_mag(r.mag_, bb.mag_);
          r.fix();
          q.mag_[static_cast<std::size_t>(i) / 32] |= (1u << (i % 32));
        }
      }
    }
    q.neg_ = a.neg_ != b.neg_;
    q.fix();
    r.neg_ = a.neg_;
    r.fix();
  }
  // Round-to-nearest-even conversion of the magnitude.
  double to_double_rne() const {
    if (is_zero()) return 0.0;
    int n = bitlen(mag_);
    double out;
    if (n <= 64) {
      std::uint64_t m = 0;
      for (std::size_t i = 0; i < mag_.size(); ++i) m |= static_cast<std::uint64_t>(mag_[i]) << (32 * i);
      out = static_cast<double>(m);  // hardware RNE
    } else {
      // top 64 bits + sticky bit, then let hardware round the 64-bit value
      int shift = n - 64;
      std::uint64_t top = 0;
      for (int i = 0; i < 64; ++i)
        if (test_bit(mag_, shift + i)) top |= (static_cast<std::uint64_t>(1) << i);
      bool sticky = false;
      for (int i = 0; i < shift && !sticky; ++i) sticky = test_bit(mag_, i);
      // fold sticky into the lowest bit (below the 53-bit rounding point)
      if (sticky) top |= 1u;
      out = std::ldexp(static_cast<double>(top), shift);
    }
    return neg_ ? -out : out;
  }

  bool neg_ = false;
  std::vector<limb> mag_;
};

}  // namespace multiprecision
}  // namespace boost
