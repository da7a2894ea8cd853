// Exact integer and rational arithmetic for symbolic counts.
//
// The reference keeps counts exact with Boost.Multiprecision cpp_int /
// cpp_rational (reference include/perfseer/poly.hpp:8,14-15). This port has
// no Boost: BigInt is a checked signed 128-bit integer and Rational a
// normalised fraction of two of them. Every operation that would leave the
// 128-bit range throws std::overflow_error, so an exact count is either
// right or loudly absent — never silently wrong. Counts in this path are
// bounded by products of problem sizes (< 2^80 at the largest configs).
//
// The member/free-function surface (numerator, denominator, convert_to<T>,
// str, lcm) matches the subset the reference API exposes to its callers.
#pragma once

#include <cstdint>
#include <limits>
#include <stdexcept>
#include <string>
#include <type_traits>

namespace perfseer {

namespace exact_detail {
using i128 = __int128;
inline i128 add(i128 a, i128 b) {
  i128 r;
  if (__builtin_add_overflow(a, b, &r)) throw std::overflow_error("exact arithmetic overflow (+)");
  return r;
}
inline i128 sub(i128 a, i128 b) {
  i128 r;
  if (__builtin_sub_overflow(a, b, &r)) throw std::overflow_error("exact arithmetic overflow (-)");
  return r;
}
inline i128 mul(i128 a, i128 b) {
  i128 r;
  if (__builtin_mul_overflow(a, b, &r)) throw std::overflow_error("exact arithmetic overflow (*)");
  return r;
}
inline i128 gcd(i128 a, i128 b) {
  if (a < 0) a = -a;
  if (b < 0) b = -b;
  while (b) {
    i128 t = a % b;
    a = b;
    b = t;
  }
  return a;
}
std::string to_string(i128 v);
i128 parse(const std::string& s);
}  // namespace exact_detail

class BigInt {
 public:
  BigInt() = default;
  template <class T, class = std::enable_if_t<std::is_integral_v<T>>>
  BigInt(T v) : v_(static_cast<exact_detail::i128>(v)) {}
  explicit BigInt(const std::string& s) : v_(exact_detail::parse(s)) {}
  explicit BigInt(const char* s) : v_(exact_detail::parse(s)) {}

  static BigInt raw(exact_detail::i128 v) {
    BigInt b;
    b.v_ = v;
    return b;
  }
  exact_detail::i128 value() const { return v_; }
  std::string str() const { return exact_detail::to_string(v_); }

  template <class T>
  T convert_to() const {
    if constexpr (std::is_floating_point_v<T>) {
      return static_cast<T>(v_);
    } else {
      if (v_ > static_cast<exact_detail::i128>(std::numeric_limits<T>::max()) ||
          v_ < static_cast<exact_detail::i128>(std::numeric_limits<T>::min()))
        throw std::overflow_error("integer does not fit the requested type");
      return static_cast<T>(v_);
    }
  }

  friend BigInt operator+(const BigInt& a, const BigInt& b) { return raw(exact_detail::add(a.v_, b.v_)); }
  friend BigInt operator-(const BigInt& a, const BigInt& b) { return raw(exact_detail::sub(a.v_, b.v_)); }
  friend BigInt operator*(const BigInt& a, const BigInt& b) { return raw(exact_detail::mul(a.v_, b.v_)); }
  friend BigInt operator/(const BigInt& a, const BigInt& b) {
    if (b.v_ == 0) throw std::domain_error("integer division by zero");
    return raw(a.v_ / b.v_);
  }
  friend BigInt operator%(const BigInt& a, const BigInt& b) {
    if (b.v_ == 0) throw std::domain_error("integer division by zero");
    return raw(a.v_ % b.v_);
  }
  BigInt operator-() const { return raw(exact_detail::sub(0, v_)); }
  BigInt& operator+=(const BigInt& o) { return *this = *this + o; }
  BigInt& operator-=(const BigInt& o) { return *this = *this - o; }
  BigInt& operator*=(const BigInt& o) { return *this = *this * o; }
  BigInt& operator/=(const BigInt& o) { return *this = *this / o; }
  friend bool operator==(const BigInt& a, const BigInt& b) { return a.v_ == b.v_; }
  friend bool operator!=(const BigInt& a, const BigInt& b) { return a.v_ != b.v_; }
  friend bool operator<(const BigInt& a, const BigInt& b) { return a.v_ < b.v_; }
  friend bool operator>(const BigInt& a, const BigInt& b) { return a.v_ > b.v_; }
  friend bool operator<=(const BigInt& a, const BigInt& b) { return a.v_ <= b.v_; }
  friend bool operator>=(const BigInt& a, const BigInt& b) { return a.v_ >= b.v_; }
  friend BigInt gcd(const BigInt& a, const BigInt& b) { return raw(exact_detail::gcd(a.v_, b.v_)); }
  friend BigInt lcm(const BigInt& a, const BigInt& b) {
    if (a.v_ == 0 || b.v_ == 0) return BigInt(0);
    exact_detail::i128 r = exact_detail::mul(a.v_ / exact_detail::gcd(a.v_, b.v_), b.v_);
    return raw(r < 0 ? -r : r);
  }

 private:
  exact_detail::i128 v_ = 0;
};

/// p/q in lowest terms with q > 0.
class Rational {
 public:
  Rational() = default;
  template <class T, class = std::enable_if_t<std::is_integral_v<T>>>
  Rational(T v) : p_(static_cast<exact_detail::i128>(v)) {}
  Rational(const BigInt& v) : p_(v.value()) {}
  template <class A, class B,
            class = std::enable_if_t<(std::is_integral_v<A> || std::is_same_v<A, BigInt>) &&
                                     (std::is_integral_v<B> || std::is_same_v<B, BigInt>)>>
  Rational(const A& num, const B& den) {
    assign(BigInt(num).value(), BigInt(den).value());
  }

  friend BigInt numerator(const Rational& r) { return BigInt::raw(r.p_); }
  friend BigInt denominator(const Rational& r) { return BigInt::raw(r.q_); }

  std::string str() const {
    std::string s = exact_detail::to_string(p_);
    return q_ == 1 ? s : s + "/" + exact_detail::to_string(q_);
  }
  template <class T>
  T convert_to() const {
    if constexpr (std::is_floating_point_v<T>)
      return static_cast<T>(p_) / static_cast<T>(q_);
    else
      return BigInt::raw(p_ / q_).convert_to<T>();
  }

  friend Rational operator+(const Rational& a, const Rational& b) {
    using namespace exact_detail;
    i128 g = gcd(a.q_, b.q_);
    return make(add(mul(a.p_, b.q_ / g), mul(b.p_, a.q_ / g)), mul(a.q_, b.q_ / g));
  }
  friend Rational operator-(const Rational& a, const Rational& b) { return a + (-b); }
  friend Rational operator*(const Rational& a, const Rational& b) {
    using namespace exact_detail;
    i128 g1 = gcd(a.p_, b.q_), g2 = gcd(b.p_, a.q_);
    if (!g1) g1 = 1;
    if (!g2) g2 = 1;
    return make(mul(a.p_ / g1, b.p_ / g2), mul(a.q_ / g2, b.q_ / g1));
  }
  friend Rational operator/(const Rational& a, const Rational& b) {
    if (b.p_ == 0) throw std::domain_error("rational division by zero");
    Rational inv;
    inv.p_ = b.p_ < 0 ? -b.q_ : b.q_;
    inv.q_ = b.p_ < 0 ? -b.p_ : b.p_;
    return a * inv;
  }
  Rational operator-() const {
    Rational r = *this;
    r.p_ = exact_detail::sub(0, p_);
    return r;
  }
  Rational& operator+=(const Rational& o) { return *this = *this + o; }
  Rational& operator-=(const Rational& o) { return *this = *this - o; }
  Rational& operator*=(const Rational& o) { return *this = *this * o; }
  Rational& operator/=(const Rational& o) { return *this = *this / o; }
  friend bool operator==(const Rational& a, const Rational& b) { return a.p_ == b.p_ && a.q_ == b.q_; }
  friend bool operator!=(const Rational& a, const Rational& b) { return !(a == b); }
  friend bool operator<(const Rational& a, const Rational& b) { return (a - b).signum() < 0; }
  friend bool operator>(const Rational& a, const Rational& b) { return (a - b).signum() > 0; }
  friend bool operator<=(const Rational& a, const Rational& b) { return (a - b).signum() <= 0; }
  friend bool operator>=(const Rational& a, const Rational& b) { return (a - b).signum() >= 0; }

  bool is_integer() const { return q_ == 1; }
  int signum() const { return p_ < 0 ? -1 : (p_ > 0 ? 1 : 0); }

 private:
  static Rational make(exact_detail::i128 p, exact_detail::i128 q) {
    Rational r;
    r.assign(p, q);
    return r;
  }
  void assign(exact_detail::i128 p, exact_detail::i128 q) {
    if (q == 0) throw std::domain_error("rational with zero denominator");
    if (q < 0) {
      p = exact_detail::sub(0, p);
      q = exact_detail::sub(0, q);
    }
    exact_detail::i128 g = exact_detail::gcd(p, q);
    if (g > 1) {
      p /= g;
      q /= g;
    }
    p_ = p;
    q_ = q;
  }
  exact_detail::i128 p_ = 0, q_ = 1;
};

inline double to_double(const Rational& r) { return r.convert_to<double>(); }
inline bool is_integer(const Rational& r) { return r.is_integer(); }

}  // namespace perfseer
