// Exact arithmetic for the model clock (reference counterpart: rational.hpp /
// rational.cpp, which use boost::rational<cpp_int>). Our own implementation:
// 32-bit limb magnitudes, Knuth long division, binary gcd, 64-bit fast paths.
#include <algorithm>
#include <bit>
#include <cmath>
#include <cstring>

#include "tencache/tencache.hpp"

namespace tencache {

namespace {

using Limbs = std::vector<std::uint32_t>;

void trim_limbs(Limbs& w) {
  while (!w.empty() && w.back() == 0) w.pop_back();
}

int cmp_mag(const Limbs& a, const Limbs& b) {
  if (a.size() != b.size()) return a.size() < b.size() ? -1 : 1;
  for (std::size_t i = a.size(); i-- > 0;)
    if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
  return 0;
}

Limbs add_mag(const Limbs& a, const Limbs& b) {
  const Limbs& x = a.size() >= b.size() ? a : b;
  const Limbs& y = a.size() >= b.size() ? b : a;
  Limbs r(x.size() + 1);
  std::uint64_t c = 0;
  for (std::size_t i = 0; i < x.size(); ++i) {
    c += static_cast<std::uint64_t>(x[i]) + (i < y.size() ? y[i] : 0u);
    r[i] = static_cast<std::uint32_t>(c);
    c >>= 32;
  }
  r[x.size()] = static_cast<std::uint32_t>(c);
  trim_limbs(r);
  return r;
}

// |a| >= |b|
Limbs sub_mag(const Limbs& a, const Limbs& b) {
  Limbs r(a.size());
  std::uint64_t borrow = 0;
  for (std::size_t i = 0; i < a.size(); ++i) {
    std::uint64_t sub = static_cast<std::uint64_t>(i < b.size() ? b[i] : 0u) + borrow;
    std::uint64_t ai = a[i];
    r[i] = static_cast<std::uint32_t>(ai - sub);
    borrow = ai < sub ? 1 : 0;
  }
  trim_limbs(r);
  return r;
}

Limbs mul_mag(const Limbs& a, const Limbs& b) {
  if (a.empty() || b.empty()) return {};
  Limbs r(a.size() + b.size(), 0);
  for (std::size_t i = 0; i < a.size(); ++i) {
    std::uint64_t carry = 0;
    const std::uint64_t ai = a[i];
    for (std::size_t j = 0; j < b.size(); ++j) {
      std::uint64_t t = ai * b[j] + r[i + j] + carry;
      r[i + j] = static_cast<std::uint32_t>(t);
      carry = t >> 32;
    }
    r[i + b.size()] = static_cast<std::uint32_t>(carry);
  }
  trim_limbs(r);
  return r;
}

// Knuth, TAOCP vol.2 §4.3.1 Algorithm D, base 2^32. Requires v non-empty.
void divmod_mag(const Limbs& u, const Limbs& v, Limbs& q, Limbs& r) {
  if (cmp_mag(u, v) < 0) {
    q.clear();
    r = u;
    return;
  }
  const std::size_t n = v.size(), m = u.size() - v.size();
  if (n == 1) {
    q.assign(u.size(), 0);
    std::uint64_t rem = 0, d = v[0];
    for (std::size_t i = u.size(); i-- > 0;) {
      std::uint64_t cur = (rem << 32) | u[i];
      q[i] = static_cast<std::uint32_t>(cur / d);
      rem = cur % d;
    }
    trim_limbs(q);
    r.clear();
    if (rem) r.push_back(static_cast<std::uint32_t>(rem));
    return;
  }
  const int s = std::countl_zero(v.back());
  Limbs vn(n), un(u.size() + 1);
  for (std::size_t i = n - 1; i > 0; --i)
    vn[i] = (v[i] << s) | (s ? static_cast<std::uint32_t>(static_cast<std::uint64_t>(v[i - 1]) >> (32 - s)) : 0u);
  vn[0] = v[0] << s;
  un[u.size()] = s ? static_cast<std::uint32_t>(static_cast<std::uint64_t>(u.back()) >> (32 - s)) : 0u;
  for (std::size_t i = u.size() - 1; i > 0; --i)
    un[i] = (u[i] << s) | (s ? static_cast<std::uint32_t>(static_cast<std::uint64_t>(u[i - 1]) >> (32 - s)) : 0u);
  un[0] = u[0] << s;

  q.assign(m + 1, 0);
  const std::uint64_t B = 1ull << 32;
  for (std::size_t j = m + 1; j-- > 0;) {
    std::uint64_t top = (static_cast<std::uint64_t>(un[j + n]) << 32) | un[j + n - 1];
    std::uint64_t qhat = top / vn[n - 1];
    std::uint64_t rhat = top % vn[n - 1];
    while (qhat >= B || qhat * vn[n - 2] > ((rhat << 32) | un[j + n - 2])) {
      --qhat;
      rhat += vn[n - 1];
      if (rhat >= B) break;
    }
    // un[j..j+n] -= qhat * vn
    std::int64_t borrow = 0;
    std::uint64_t carry = 0;
    for (std::size_t i = 0; i < n; ++i) {
      std::uint64_t p = qhat * vn[i] + carry;
      carry = p >> 32;
      std::int64_t t = static_cast<std::int64_t>(un[i + j]) - borrow - static_cast<std::int64_t>(p & 0xffffffffu);
      un[i + j] = static_cast<std::uint32_t>(t);
      borrow = t < 0 ? 1 : 0;
    }
    std::int64_t t = static_cast<std::int64_t>(un[j + n]) - borrow - static_cast<std::int64_t>(carry);
    un[j + n] = static_cast<std::uint32_t>(t);
    if (t < 0) {  // add back
      --qhat;
      std::uint64_t c = 0;
      for (std::size_t i = 0; i < n; ++i) {
        c += static_cast<std::uint64_t>(un[i + j]) + vn[i];
        un[i + j] = static_cast<std::uint32_t>(c);
        c >>= 32;
      }
      un[j + n] = static_cast<std::uint32_t>(static_cast<std::uint64_t>(un[j + n]) + c);
    }
    q[j] = static_cast<std::uint32_t>(qhat);
  }
  trim_limbs(q);
  r.assign(n, 0);
  for (std::size_t i = 0; i < n; ++i)
    r[i] = (un[i] >> s) | (s ? static_cast<std::uint32_t>(static_cast<std::uint64_t>(un[i + 1]) << (32 - s)) : 0u);
  trim_limbs(r);
}

bool fits_u64(const Limbs& w) { return w.size() <= 2; }
std::uint64_t as_u64(const Limbs& w) {
  std::uint64_t v = 0;
  if (!w.empty()) v = w[0];
  if (w.size() > 1) v |= static_cast<std::uint64_t>(w[1]) << 32;
  return v;
}
Limbs from_u64(std::uint64_t v) {
  Limbs w;
  while (v) {
    w.push_back(static_cast<std::uint32_t>(v));
    v >>= 32;
  }
  return w;
}

unsigned ctz_mag(const Limbs& w) {
  unsigned z = 0;
  for (std::uint32_t x : w) {
    if (x) return z + static_cast<unsigned>(std::countr_zero(x));
    z += 32;
  }
  return z;
}

void shr_mag(Limbs& w, unsigned bits) {
  std::size_t limbs = bits / 32;
  unsigned b = bits % 32;
  if (limbs >= w.size()) {
    w.clear();
    return;
  }
  w.erase(w.begin(), w.begin() + static_cast<std::ptrdiff_t>(limbs));
  if (b) {
    for (std::size_t i = 0; i + 1 < w.size(); ++i) w[i] = (w[i] >> b) | (w[i + 1] << (32 - b));
    w.back() >>= b;
  }
  trim_limbs(w);
}

Limbs shl_mag(const Limbs& a, unsigned bits) {
  if (a.empty()) return {};
  Limbs r(bits / 32, 0);
  unsigned b = bits % 32;
  std::uint32_t carry = 0;
  for (std::uint32_t x : a) {
    r.push_back(b ? ((x << b) | carry) : x);
    carry = b ? static_cast<std::uint32_t>(static_cast<std::uint64_t>(x) >> (32 - b)) : 0u;
  }
  if (carry) r.push_back(carry);
  return r;
}

}  // namespace

// ----------------------------------------------------------------- BigInt
void BigInt::set_u64(std::uint64_t m) {
  w_ = from_u64(m);
  if (w_.empty()) neg_ = false;
}

std::uint64_t BigInt::low_u64() const { return as_u64(w_); }

void BigInt::trim() {
  trim_limbs(w_);
  if (w_.empty()) neg_ = false;
}

std::size_t BigInt::bit_length() const {
  if (w_.empty()) return 0;
  return (w_.size() - 1) * 32 + (32 - static_cast<std::size_t>(std::countl_zero(w_.back())));
}

BigInt operator+(const BigInt& a, const BigInt& b) {
  BigInt r;
  if (a.neg_ == b.neg_) {
    r.w_ = add_mag(a.w_, b.w_);
    r.neg_ = a.neg_;
  } else {
    int c = cmp_mag(a.w_, b.w_);
    if (c == 0) return r;
    if (c > 0) {
      r.w_ = sub_mag(a.w_, b.w_);
      r.neg_ = a.neg_;
    } else {
      r.w_ = sub_mag(b.w_, a.w_);
      r.neg_ = b.neg_;
    }
  }
  r.trim();
  return r;
}

BigInt operator-(const BigInt& a) {
  BigInt r = a;
  if (!r.w_.empty()) r.neg_ = !r.neg_;
  return r;
}

BigInt operator-(const BigInt& a, const BigInt& b) { return a + (-b); }

BigInt operator*(const BigInt& a, const BigInt& b) {
  BigInt r;
  r.w_ = mul_mag(a.w_, b.w_);
  r.neg_ = a.neg_ != b.neg_;
  r.trim();
  return r;
}

void BigInt::divmod(const BigInt& a, const BigInt& b, BigInt& q, BigInt& r) {
  if (b.w_.empty()) throw std::domain_error("BigInt: division by zero");
  divmod_mag(a.w_, b.w_, q.w_, r.w_);
  q.neg_ = a.neg_ != b.neg_;
  r.neg_ = a.neg_;
  q.trim();
  r.trim();
}

BigInt operator/(const BigInt& a, const BigInt& b) {
  BigInt q, r;
  BigInt::divmod(a, b, q, r);
  return q;
}

BigInt operator%(const BigInt& a, const BigInt& b) {
  BigInt q, r;
  BigInt::divmod(a, b, q, r);
  return r;
}

BigInt operator<<(const BigInt& a, int bits) {
  if (bits < 0) throw std::domain_error("BigInt: negative shift");
  BigInt r;
  r.w_ = shl_mag(a.w_, static_cast<unsigned>(bits));
  r.neg_ = a.neg_;
  r.trim();
  return r;
}

int compare(const BigInt& a, const BigInt& b) {
  if (a.neg_ != b.neg_) return a.neg_ ? -1 : 1;
  int c = cmp_mag(a.w_, b.w_);
  return a.neg_ ? -c : c;
}

// Binary gcd on magnitudes; result non-negative.
BigInt BigInt::gcd(BigInt a, BigInt b) {
  a.neg_ = b.neg_ = false;
  if (a.w_.empty()) return b;
  if (b.w_.empty()) return a;
  if (fits_u64(a.w_) && fits_u64(b.w_)) {
    std::uint64_t x = as_u64(a.w_), y = as_u64(b.w_);
    int sh = std::countr_zero(x | y);
    x >>= std::countr_zero(x);
    while (y) {
      y >>= std::countr_zero(y);
      if (x > y) std::swap(x, y);
      y -= x;
    }
    BigInt g;
    g.set_u64(x << sh);
    return g;
  }
  unsigned za = ctz_mag(a.w_), zb = ctz_mag(b.w_);
  unsigned sh = std::min(za, zb);
  shr_mag(a.w_, za);
  shr_mag(b.w_, zb);
  // Mix Euclid steps (cheap when sizes differ a lot) with binary steps.
  while (!b.w_.empty()) {
    if (a.w_.size() > b.w_.size() + 1 || b.w_.size() > a.w_.size() + 1) {
      Limbs q, r;
      if (cmp_mag(a.w_, b.w_) > 0) {
        divmod_mag(a.w_, b.w_, q, r);
        a.w_ = std::move(b.w_);
        b.w_ = std::move(r);
      } else {
        divmod_mag(b.w_, a.w_, q, r);
        b.w_ = std::move(r);
      }
      if (b.w_.empty()) break;
      shr_mag(a.w_, ctz_mag(a.w_));
      shr_mag(b.w_, ctz_mag(b.w_));
      continue;
    }
    if (fits_u64(a.w_) && fits_u64(b.w_)) {
      std::uint64_t x = as_u64(a.w_), y = as_u64(b.w_);
      while (y) {
        y >>= std::countr_zero(y);
        if (x > y) std::swap(x, y);
        y -= x;
      }
      a.w_ = from_u64(x);
      break;
    }
    int c = cmp_mag(a.w_, b.w_);
    if (c == 0) break;
    if (c > 0) std::swap(a.w_, b.w_);
    b.w_ = sub_mag(b.w_, a.w_);
    shr_mag(b.w_, ctz_mag(b.w_));
  }
  a.w_ = shl_mag(a.w_, sh);
  a.trim();
  return a;
}

std::string BigInt::str() const {
  if (w_.empty()) return "0";
  Limbs m = w_;
  std::string out;
  while (!m.empty()) {
    std::uint64_t rem = 0;
    for (std::size_t i = m.size(); i-- > 0;) {
      std::uint64_t cur = (rem << 32) | m[i];
      m[i] = static_cast<std::uint32_t>(cur / 1000000000u);
      rem = cur % 1000000000u;
    }
    trim_limbs(m);
    for (int k = 0; k < 9; ++k) {
      out.push_back(static_cast<char>('0' + rem % 10));
      rem /= 10;
      if (m.empty() && rem == 0) break;
    }
  }
  while (out.size() > 1 && out.back() == '0') out.pop_back();
  if (neg_) out.push_back('-');
  std::reverse(out.begin(), out.end());
  return out;
}

double BigInt::to_double() const {
  if (w_.empty()) return 0.0;
  std::size_t n = bit_length();
  double mag;
  if (n <= 64) {
    mag = static_cast<double>(as_u64(w_));
  } else {
    // keep the top 64 bits and fold everything below into a sticky bit, so
    // the hardware's single u64->double rounding is round-to-nearest-even.
    unsigned shift = static_cast<unsigned>(n - 64);
    Limbs t = w_;
    bool sticky = ctz_mag(t) < shift;
    shr_mag(t, shift);
    std::uint64_t top = as_u64(t) | (sticky ? 1u : 0u);
    mag = std::ldexp(static_cast<double>(top), static_cast<int>(shift));
  }
  return neg_ ? -mag : mag;
}

// -------------------------------------------------------------------- Rat
Rat::Rat(const BigInt& n, const BigInt& d) : num_(n), den_(d) {
  if (den_.is_zero()) throw std::domain_error("Rat: zero denominator");
  reduce();
}

void Rat::reduce() {
  if (num_.is_zero()) {
    den_ = BigInt(1);
    return;
  }
  if (den_.is_negative()) {
    num_ = -num_;
    den_ = -den_;
  }
  BigInt g = BigInt::gcd(num_, den_);
  if (!(g == BigInt(1))) {
    num_ = num_ / g;
    den_ = den_ / g;
  }
}

Rat operator+(const Rat& a, const Rat& b) {
  if (a.num_.is_zero()) return b;
  if (b.num_.is_zero()) return a;
  if (a.den_ == b.den_) {
    Rat r(a.num_ + b.num_, a.den_, Rat::Raw{});
    r.reduce();
    return r;
  }
  // Henrici: g = gcd(b1, b2) keeps intermediates small.
  BigInt g = BigInt::gcd(a.den_, b.den_);
  if (g == BigInt(1)) {
    Rat r(a.num_ * b.den_ + b.num_ * a.den_, a.den_ * b.den_, Rat::Raw{});
    // already reduced: gcd(a1 b2 + a2 b1, b1 b2) = 1 when gcd(b1,b2)=1
    if (r.num_.is_zero()) r.den_ = BigInt(1);
    return r;
  }
  BigInt ad = a.den_ / g, bd = b.den_ / g;
  Rat r(a.num_ * bd + b.num_ * ad, ad * b.den_, Rat::Raw{});
  r.reduce();
  return r;
}

Rat operator-(const Rat& a, const Rat& b) { return a + Rat(-b.num_, b.den_, Rat::Raw{}); }

Rat operator*(const Rat& a, const Rat& b) {
  if (a.num_.is_zero() || b.num_.is_zero()) return Rat();
  Rat r(a.num_ * b.num_, a.den_ * b.den_, Rat::Raw{});
  r.reduce();
  return r;
}

Rat operator/(const Rat& a, const Rat& b) {
  if (b.num_.is_zero()) throw std::domain_error("Rat: division by zero");
  Rat r(a.num_ * b.den_, a.den_ * b.num_, Rat::Raw{});
  r.reduce();
  return r;
}

bool operator<(const Rat& a, const Rat& b) {
  int sa = a.num_.sign(), sb = b.num_.sign();
  if (sa != sb) return sa < sb;
  if (a.den_ == b.den_) return a.num_ < b.num_;
  return a.num_ * b.den_ < b.num_ * a.den_;
}

Rat rat_from_double(double v) {
  if (!std::isfinite(v)) throw std::domain_error("rat_from_double: non-finite value");
  if (v == 0.0) return Rat(0);
  std::uint64_t bits;
  std::memcpy(&bits, &v, sizeof bits);
  bool neg = bits >> 63;
  int e = static_cast<int>((bits >> 52) & 0x7ff);
  std::uint64_t frac = bits & ((1ull << 52) - 1);
  std::uint64_t mant;
  int exp2;
  if (e == 0) {  // subnormal
    mant = frac;
    exp2 = -1074;
  } else {
    mant = frac | (1ull << 52);
    exp2 = e - 1075;
  }
  int tz = std::countr_zero(mant);
  mant >>= tz;
  exp2 += tz;
  BigInt n = neg ? -BigInt(mant) : BigInt(mant);
  if (exp2 >= 0) return Rat(n << exp2);
  return Rat(n, BigInt(1) << -exp2);
}

double to_double(const Rat& r) {
  if (r.numerator().is_zero()) return 0.0;
  return r.numerator().to_double() / r.denominator().to_double();
}

Rat rat_decimal(std::int64_t mantissa, int exp10) {
  BigInt scale(1);
  for (int i = 0; i < std::abs(exp10); ++i) scale = scale * BigInt(10);
  if (exp10 >= 0) return Rat(BigInt(mantissa) * scale);
  return Rat(BigInt(mantissa), scale);
}

std::string rat_to_string(const Rat& r) {
  std::string s = r.numerator().str();
  if (!(r.denominator() == BigInt(1))) s += "/" + r.denominator().str();
  return s;
}

}  // namespace tencache
