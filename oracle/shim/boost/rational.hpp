// ORACLE TEST INFRASTRUCTURE — not product code.
//
// Minimal stand-in for boost::rational<T> (always normalised: gcd-reduced,
// positive denominator), covering the surface the reference simulator uses.
#pragma once

#include <stdexcept>

#include <boost/multiprecision/cpp_int.hpp>

namespace boost {

template <typename T>
class rational {
 public:
  rational() : num_(0), den_(1) {}
  template <typename U>
  rational(const U& n) : num_(n), den_(1) {}  // NOLINT: implicit as in boost
  rational(const T& n, const T& d) : num_(n), den_(d) { normalize(); }

  const T& numerator() const { return num_; }
  const T& denominator() const { return den_; }

  friend rational operator+(const rational& a, const rational& b) {
    return rational(a.num_ * b.den_ + b.num_ * a.den_, a.den_ * b.den_);
  }
  friend rational operator-(const rational& a, const rational& b) {
    return rational(a.num_ * b.den_ - b.num_ * a.den_, a.den_ * b.den_);
  }
  friend rational operator*(const rational& a, const rational& b) {
    return rational(a.num_ * b.num_, a.den_ * b.den_);
  }
  friend rational operator/(const rational& a, const rational& b) {
    if (b.num_ == T(0)) throw std::domain_error("rational: division by zero");
    return rational(a.num_ * b.den_, a.den_ * b.num_);
  }
  rational& operator+=(const rational& b) { return *this = *this + b; }
  rational& operator-=(const rational& b) { return *this = *this - b; }
  rational& operator*=(const rational& b) { return *this = *this * b; }
  rational& operator/=(const rational& b) { return *this = *this / b; }

  friend bool operator==(const rational& a, const rational& b) {
    return a.num_ == b.num_ && a.den_ == b.den_;
  }
  friend bool operator!=(const rational& a, const rational& b) { return !(a == b); }
  friend bool operator<(const rational& a, const rational& b) {
    return a.num_ * b.den_ < b.num_ * a.den_;
  }
  friend bool operator>(const rational& a, const rational& b) { return b < a; }
  friend bool operator<=(const rational& a, const rational& b) { return !(b < a); }
  friend bool operator>=(const rational& a, const rational& b) { return !(a < b); }

 private:
  static T gcd(T a, T b) {
    if (a < T(0)) a = -a;
    if (b < T(0)) b = -b;
    while (!(b == T(0))) {
      T t = a % b;
      a = b;
      b = t;
    }
    return a;
  }
  void normalize() {
    if (den_ == T(0)) throw std::domain_error("rational: zero denominator");
    if (num_ == T(0)) {
      den_ = T(1);
      return;
    }
    T g = gcd(num_, den_);
    num_ = num_ / g;
    den_ = den_ / g;
    if (den_ < T(0)) {
      num_ = -num_;
      den_ = -den_;
    }
  }

  T num_;
  T den_;
};

}  // namespace boost
