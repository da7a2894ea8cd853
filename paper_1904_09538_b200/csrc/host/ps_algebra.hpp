// Symbolic algebra for counts: monomials, exact-coefficient polynomials over
// size parameters and loop indices, ratios, and affine index expressions.
//
// API-compatible with the reference's Poly / PolyRatio / PiecewisePoly /
// AffineExpr (reference include/perfseer/poly.hpp:20-226, affine.hpp:17-142):
// the same constructors, operators, canonical printing and evaluation, so
// count keys such as "mem:global:load:4:...:ls={0:1;1:n}..." are
// byte-identical to the reference's.
#pragma once

#include <map>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include "ps_errors.hpp"
#include "ps_exact.hpp"

namespace perfseer {

/// A product of symbol powers; exponents are >= 1 and keyed by symbol name.
struct Monomial {
  std::map<std::string, int> exps;

  int degree() const {
    int d = 0;
    for (const auto& kv : exps) d += kv.second;
    return d;
  }
  Monomial operator*(const Monomial& o) const {
    Monomial r = *this;
    for (const auto& [sym, e] : o.exps) r.exps[sym] += e;
    return r;
  }
  bool operator<(const Monomial& o) const { return exps < o.exps; }
  bool operator==(const Monomial& o) const { return exps == o.exps; }
};

/// Multivariate polynomial with exact rational coefficients. Zero
/// coefficients are never stored, so structural equality is value equality.
class Poly {
 public:
  using TermMap = std::map<Monomial, Rational>;

  Poly() = default;
  static Poly constant(const Rational& c);
  static Poly constant(long long c) { return constant(Rational(c)); }
  static Poly symbol(const std::string& name);

  bool is_zero() const { return t_.empty(); }
  bool is_constant() const { return t_.empty() || (t_.size() == 1 && t_.begin()->first.exps.empty()); }
  Rational constant_value() const;
  int degree() const;
  std::set<std::string> symbols() const;

  Poly operator+(const Poly& o) const;
  Poly operator-(const Poly& o) const;
  Poly operator-() const;
  Poly operator*(const Poly& o) const;
  Poly operator*(const Rational& c) const;
  Poly& operator+=(const Poly& o) { return *this = *this + o; }
  Poly& operator-=(const Poly& o) { return *this = *this - o; }
  Poly& operator*=(const Poly& o) { return *this = *this * o; }
  Poly pow(unsigned e) const;
  bool operator==(const Poly& o) const { return t_ == o.t_; }
  bool operator!=(const Poly& o) const { return !(t_ == o.t_); }

  /// Replaces every occurrence of `name` by `value`.
  Poly substitute(const std::string& name, const Poly& value) const;
  /// Exact value at integer bindings; unbound symbols are an EvalError.
  Rational eval(const std::map<std::string, long long>& env) const;
  /// Canonical text: terms by total degree (high first) then exponents over
  /// the sorted symbol set (high first); a common denominator is factored
  /// out, e.g. "(n^2 - 2*n*p + p^2 + n - p)/2".
  std::string str() const;

  const TermMap& terms() const { return t_; }
  void accumulate(const Monomial& m, const Rational& c);

 private:
  TermMap t_;
};

inline Poly operator*(const Rational& c, const Poly& p) { return p * c; }

/// Exact division num/den when possible (multivariate, leading-term
/// elimination in lexicographic order); false when den does not divide num.
bool try_divide(const Poly& num, const Poly& den, Poly& quotient);

/// Sum of p over integer `iname` in [lo, hi] by closed-form power sums
/// (Faulhaber); exact whenever hi >= lo - 1.
Poly sum_over_range(const Poly& p, const std::string& iname, const Poly& lo, const Poly& hi);

/// Exact num/den, reduced to a polynomial when the division is exact
/// (access-to-footprint ratios).
struct PolyRatio {
  Poly num;
  Poly den = Poly::constant(1);

  static PolyRatio exact(const Poly& p) { return PolyRatio{p, Poly::constant(1)}; }
  static PolyRatio of(const Poly& n, const Poly& d);
  bool is_poly() const { return den == Poly::constant(1); }
  Rational eval(const std::map<std::string, long long>& env) const;
  bool operator==(const PolyRatio& o) const { return num == o.num && den == o.den; }
  std::string str() const;
};

struct PolyPiece {
  std::vector<std::string> guards;
  Poly poly;
};

/// Guarded polynomial pieces; the counting engine emits single pieces valid
/// on the kernel's assumption region.
struct PiecewisePoly {
  std::vector<PolyPiece> pieces;

  static PiecewisePoly single(const Poly& p, std::vector<std::string> guards = {}) {
    return PiecewisePoly{{PolyPiece{std::move(guards), p}}};
  }
  const Poly& poly() const {
    if (pieces.size() != 1) throw EvalError("expected single-piece polynomial");
    return pieces.front().poly;
  }
  Rational eval(const std::map<std::string, long long>& env) const { return poly().eval(env); }
  std::string str() const { return poly().str(); }
};

/// Linear in loop indices, coefficients polynomial in size parameters:
/// sum_i lin[i] * i + off.
struct AffineExpr {
  std::map<std::string, Poly> lin;  // index -> nonzero coefficient
  Poly off;

  static AffineExpr constant(const Rational& c) { return AffineExpr{{}, Poly::constant(c)}; }
  static AffineExpr constant(long long c) { return constant(Rational(c)); }
  static AffineExpr index(const std::string& name) {
    AffineExpr a;
    a.lin.emplace(name, Poly::constant(1));
    return a;
  }
  static AffineExpr param(const std::string& name) { return AffineExpr{{}, Poly::symbol(name)}; }

  bool is_index_free() const { return lin.empty(); }
  bool is_constant() const { return lin.empty() && off.is_constant(); }

  AffineExpr operator+(const AffineExpr& o) const;
  AffineExpr operator-() const;
  AffineExpr operator-(const AffineExpr& o) const { return *this + (-o); }
  AffineExpr scaled(const Rational& k) const { return scaled(Poly::constant(k)); }
  AffineExpr scaled(const Poly& k) const;
  /// Product with an index-free factor (SemanticError otherwise).
  AffineExpr times(const AffineExpr& o) const;
  AffineExpr substitute_index(const std::string& name, const AffineExpr& value) const;
  AffineExpr substitute_param(const std::string& name, const Rational& value) const;
  Poly to_poly() const;
  Rational eval(const std::map<std::string, long long>& env) const { return to_poly().eval(env); }
  std::set<std::string> index_symbols() const;
  std::set<std::string> all_symbols() const;
  /// Constant index coefficients and an offset of degree <= 1.
  bool strictly_affine() const;
  /// Integer index coefficients and integer offset coefficients.
  bool integer_coefficients() const;
  bool operator==(const AffineExpr& o) const { return lin == o.lin && off == o.off; }
  bool operator!=(const AffineExpr& o) const { return !(*this == o); }
  std::string str() const { return to_poly().str(); }
};

}  // namespace perfseer
