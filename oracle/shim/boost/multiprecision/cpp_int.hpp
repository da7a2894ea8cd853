// TEST INFRASTRUCTURE ONLY (oracle/): a restatement of the subset of
// Boost.Multiprecision (third-party, unpinned: the reference's vendor/ tree is
// gitignored upstream, /root/reference/proj/.gitignore:2) that the reference
// library uses: `cpp_int` and `cpp_rational` as exact integers and
// normalised fractions. It exists only so the UNMODIFIED reference sources
// under /root/reference/proj/src can be compiled into oracle/_ref and used as
// the parity oracle. Call sites it serves: poly.hpp:14-18,45-66,138-151,
// poly.cpp:43-59,105-167, lang.cpp:158,186-188,402-419, kernel_json.cpp:9-18,
// oracle.cpp:44-66, counting.cpp:90-133, features.cpp:253-338.
//
// Representation: a checked signed 128-bit integer. Every operation that
// would leave the 128-bit range throws std::overflow_error, so the oracle can
// never silently return a wrong exact count (Boost would have promoted to a
// wider limb vector; no reference path at the configured sizes needs more).
#pragma once

#include <cstdint>
#include <limits>
#include <stdexcept>
#include <string>
#include <type_traits>

namespace boost {
namespace multiprecision {

class cpp_int {
 public:
  using rep = __int128;
  cpp_int() : v_(0) {}
  template <class T, class = std::enable_if_t<std::is_integral_v<T>>>
  cpp_int(T x) : v_(static_cast<rep>(x)) {}
  explicit cpp_int(const std::string& s) : v_(parse(s)) {}
  explicit cpp_int(const char* s) : v_(parse(s)) {}
  static cpp_int from_rep(rep r) {
    cpp_int c;
    c.v_ = r;
    return c;
  }
  rep raw() const { return v_; }

  std::string str() const {
    if (v_ == 0) return "0";
    bool neg = v_ < 0;
    unsigned __int128 m = neg ? static_cast<unsigned __int128>(-(v_ + 1)) + 1
                              : static_cast<unsigned __int128>(v_);
    std::string digits;
    while (m) {
      digits.insert(digits.begin(), static_cast<char>('0' + static_cast<int>(m % 10)));
      m /= 10;
    }
    return neg ? "-" + digits : digits;
  }
  template <class T>
  T convert_to() const {
    if constexpr (std::is_floating_point_v<T>) {
      return static_cast<T>(v_);
    } else {
      if (v_ > static_cast<rep>(std::numeric_limits<T>::max()) ||
          v_ < static_cast<rep>(std::numeric_limits<T>::min()))
        throw std::overflow_error("cpp_int shim: value does not fit the target type");
      return static_cast<T>(v_);
    }
  }

  static rep add(rep a, rep b) {
    rep r;
    if (__builtin_add_overflow(a, b, &r)) throw std::overflow_error("cpp_int shim: add overflow");
    return r;
  }
  static rep sub(rep a, rep b) {
    rep r;
    if (__builtin_sub_overflow(a, b, &r)) throw std::overflow_error("cpp_int shim: sub overflow");
    return r;
  }
  static rep mul(rep a, rep b) {
    rep r;
    if (__builtin_mul_overflow(a, b, &r)) throw std::overflow_error("cpp_int shim: mul overflow");
    return r;
  }
  static rep div(rep a, rep b) {
    if (b == 0) throw std::overflow_error("Division by zero.");
    return a / b;  // truncation, as Boost
  }

  friend cpp_int operator+(const cpp_int& a, const cpp_int& b) { return from_rep(add(a.v_, b.v_)); }
  friend cpp_int operator-(const cpp_int& a, const cpp_int& b) { return from_rep(sub(a.v_, b.v_)); }
  friend cpp_int operator*(const cpp_int& a, const cpp_int& b) { return from_rep(mul(a.v_, b.v_)); }
  friend cpp_int operator/(const cpp_int& a, const cpp_int& b) { return from_rep(div(a.v_, b.v_)); }
  friend cpp_int operator%(const cpp_int& a, const cpp_int& b) {
    if (b.v_ == 0) throw std::overflow_error("Division by zero.");
    return from_rep(a.v_ % b.v_);
  }
  cpp_int operator-() const { return from_rep(sub(0, v_)); }
  cpp_int& operator+=(const cpp_int& o) { return *this = *this + o; }
  cpp_int& operator-=(const cpp_int& o) { return *this = *this - o; }
  cpp_int& operator*=(const cpp_int& o) { return *this = *this * o; }
  cpp_int& operator/=(const cpp_int& o) { return *this = *this / o; }
  friend bool operator==(const cpp_int& a, const cpp_int& b) { return a.v_ == b.v_; }
  friend bool operator!=(const cpp_int& a, const cpp_int& b) { return a.v_ != b.v_; }
  friend bool operator<(const cpp_int& a, const cpp_int& b) { return a.v_ < b.v_; }
  friend bool operator>(const cpp_int& a, const cpp_int& b) { return a.v_ > b.v_; }
  friend bool operator<=(const cpp_int& a, const cpp_int& b) { return a.v_ <= b.v_; }
  friend bool operator>=(const cpp_int& a, const cpp_int& b) { return a.v_ >= b.v_; }

  friend cpp_int gcd(const cpp_int& a, const cpp_int& b) { return from_rep(gcd_rep(a.v_, b.v_)); }
  friend cpp_int lcm(const cpp_int& a, const cpp_int& b) {
    if (a.v_ == 0 || b.v_ == 0) return cpp_int(0);
    rep g = gcd_rep(a.v_, b.v_);
    rep r = mul(a.v_ / g, b.v_);
    return from_rep(r < 0 ? -r : r);
  }
  friend cpp_int abs(const cpp_int& a) { return a.v_ < 0 ? -a : a; }

  static rep gcd_rep(rep a, rep b) {
    if (a < 0) a = -a;
    if (b < 0) b = -b;
    while (b != 0) {
      rep t = a % b;
      a = b;
      b = t;
    }
    return a;
  }

 private:
  static rep parse(const std::string& s) {
    size_t i = 0;
    bool neg = false;
    if (i < s.size() && (s[i] == '-' || s[i] == '+')) neg = s[i++] == '-';
    if (i == s.size()) throw std::runtime_error("cpp_int shim: malformed integer '" + s + "'");
    rep v = 0;
    for (; i < s.size(); ++i) {
      if (s[i] < '0' || s[i] > '9')
        throw std::runtime_error("cpp_int shim: malformed integer '" + s + "'");
      v = add(mul(v, 10), s[i] - '0');
    }
    return neg ? -v : v;
  }
  rep v_;
};

/// Normalised fraction num/den with den > 0 and gcd(num, den) == 1.
class cpp_rational {
 public:
  using rep = cpp_int::rep;
  cpp_rational() : n_(0), d_(1) {}
  template <class T, class = std::enable_if_t<std::is_integral_v<T>>>
  cpp_rational(T x) : n_(static_cast<rep>(x)), d_(1) {}
  cpp_rational(const cpp_int& x) : n_(x.raw()), d_(1) {}
  template <class A, class B,
            class = std::enable_if_t<(std::is_integral_v<A> || std::is_same_v<A, cpp_int>) &&
                                     (std::is_integral_v<B> || std::is_same_v<B, cpp_int>)>>
  cpp_rational(const A& num, const B& den) {
    set(cpp_int(num).raw(), cpp_int(den).raw());
  }

  friend cpp_int numerator(const cpp_rational& r) { return cpp_int::from_rep(r.n_); }
  friend cpp_int denominator(const cpp_rational& r) { return cpp_int::from_rep(r.d_); }

  std::string str() const {
    std::string s = cpp_int::from_rep(n_).str();
    if (d_ != 1) s += "/" + cpp_int::from_rep(d_).str();
    return s;
  }
  template <class T>
  T convert_to() const {
    if constexpr (std::is_floating_point_v<T>) {
      return static_cast<T>(n_) / static_cast<T>(d_);
    } else {
      return cpp_int::from_rep(n_ / d_).convert_to<T>();  // truncation toward zero
    }
  }

  friend cpp_rational operator+(const cpp_rational& a, const cpp_rational& b) {
    rep g = cpp_int::gcd_rep(a.d_, b.d_);
    rep da = a.d_ / g, db = b.d_ / g;
    rep num = cpp_int::add(cpp_int::mul(a.n_, db), cpp_int::mul(b.n_, da));
    rep den = cpp_int::mul(a.d_, db);
    return make(num, den);
  }
  friend cpp_rational operator-(const cpp_rational& a, const cpp_rational& b) { return a + (-b); }
  friend cpp_rational operator*(const cpp_rational& a, const cpp_rational& b) {
    rep g1 = cpp_int::gcd_rep(a.n_, b.d_), g2 = cpp_int::gcd_rep(b.n_, a.d_);
    if (g1 == 0) g1 = 1;
    if (g2 == 0) g2 = 1;
    return make(cpp_int::mul(a.n_ / g1, b.n_ / g2), cpp_int::mul(a.d_ / g2, b.d_ / g1));
  }
  friend cpp_rational operator/(const cpp_rational& a, const cpp_rational& b) {
    if (b.n_ == 0) throw std::overflow_error("Division by zero.");
    cpp_rational inv;
    inv.n_ = b.n_ < 0 ? -b.d_ : b.d_;
    inv.d_ = b.n_ < 0 ? -b.n_ : b.n_;
    return a * inv;
  }
  cpp_rational operator-() const {
    cpp_rational r = *this;
    r.n_ = cpp_int::sub(0, n_);
    return r;
  }
  cpp_rational& operator+=(const cpp_rational& o) { return *this = *this + o; }
  cpp_rational& operator-=(const cpp_rational& o) { return *this = *this - o; }
  cpp_rational& operator*=(const cpp_rational& o) { return *this = *this * o; }
  cpp_rational& operator/=(const cpp_rational& o) { return *this = *this / o; }

  friend bool operator==(const cpp_rational& a, const cpp_rational& b) {
    return a.n_ == b.n_ && a.d_ == b.d_;
  }
  friend bool operator!=(const cpp_rational& a, const cpp_rational& b) { return !(a == b); }
  friend bool operator<(const cpp_rational& a, const cpp_rational& b) { return cmp(a, b) < 0; }
  friend bool operator>(const cpp_rational& a, const cpp_rational& b) { return cmp(a, b) > 0; }
  friend bool operator<=(const cpp_rational& a, const cpp_rational& b) { return cmp(a, b) <= 0; }
  friend bool operator>=(const cpp_rational& a, const cpp_rational& b) { return cmp(a, b) >= 0; }

 private:
  static int cmp(const cpp_rational& a, const cpp_rational& b) {
    cpp_rational d = a - b;
    return d.n_ < 0 ? -1 : (d.n_ > 0 ? 1 : 0);
  }
  static cpp_rational make(rep num, rep den) {
    cpp_rational r;
    r.set(num, den);
    return r;
  }
  void set(rep num, rep den) {
    if (den == 0) throw std::overflow_error("Division by zero.");
    if (den < 0) {
      num = cpp_int::sub(0, num);
      den = cpp_int::sub(0, den);
    }
    rep g = cpp_int::gcd_rep(num, den);
    if (g == 0) g = 1;
    n_ = num / g;
    d_ = den / g;
  }
  rep n_, d_;
};

}  // namespace multiprecision
}  // namespace boost
