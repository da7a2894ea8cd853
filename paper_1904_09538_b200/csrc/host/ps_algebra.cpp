// Polynomial / affine algebra (see ps_algebra.hpp).
#include "ps_algebra.hpp"

#include <algorithm>
#include <mutex>

namespace perfseer {

namespace exact_detail {

std::string to_string(i128 v) {
  if (v == 0) return "0";
  const bool neg = v < 0;
  unsigned __int128 m = neg ? (unsigned __int128)(-(v + 1)) + 1u : (unsigned __int128)v;
  char buf[48];
  int pos = 47;
  buf[pos] = '\0';
  while (m) {
    buf[--pos] = char('0' + int(m % 10));
    m /= 10;
  }
  if (neg) buf[--pos] = '-';
  return std::string(buf + pos);
}

i128 parse(const std::string& s) {
  size_t i = 0;
  bool neg = false;
  if (i < s.size() && (s[i] == '+' || s[i] == '-')) neg = s[i++] == '-';
  if (i >= s.size()) throw std::invalid_argument("malformed integer literal '" + s + "'");
  i128 v = 0;
  for (; i < s.size(); ++i) {
    if (s[i] < '0' || s[i] > '9') throw std::invalid_argument("malformed integer literal '" + s + "'");
    v = add(mul(v, 10), s[i] - '0');
  }
  return neg ? -v : v;
}

}  // namespace exact_detail

// ---------------------------------------------------------------------------
// Poly

Poly Poly::constant(const Rational& c) {
  Poly p;
  if (c != 0) p.t_.emplace(Monomial{}, c);
  return p;
}

Poly Poly::symbol(const std::string& name) {
  Poly p;
  Monomial m;
  m.exps.emplace(name, 1);
  p.t_.emplace(std::move(m), Rational(1));
  return p;
}

void Poly::accumulate(const Monomial& m, const Rational& c) {
  if (c == 0) return;
  auto it = t_.find(m);
  if (it == t_.end()) {
    t_.emplace(m, c);
    return;
  }
  it->second += c;
  if (it->second == 0) t_.erase(it);
}

Rational Poly::constant_value() const {
  if (t_.empty()) return Rational(0);
  if (!is_constant()) throw EvalError("polynomial is not constant: " + str());
  return t_.begin()->second;
}

int Poly::degree() const {
  int d = 0;
  for (const auto& kv : t_) d = std::max(d, kv.first.degree());
  return d;
}

std::set<std::string> Poly::symbols() const {
  std::set<std::string> s;
  for (const auto& kv : t_)
    for (const auto& e : kv.first.exps) s.insert(e.first);
  return s;
}

Poly Poly::operator+(const Poly& o) const {
  Poly r = *this;
  for (const auto& [m, c] : o.t_) r.accumulate(m, c);
  return r;
}

Poly Poly::operator-(const Poly& o) const {
  Poly r = *this;
  for (const auto& [m, c] : o.t_) r.accumulate(m, -c);
  return r;
}

Poly Poly::operator-() const {
  Poly r;
  for (const auto& [m, c] : t_) r.t_.emplace(m, -c);
  return r;
}

Poly Poly::operator*(const Poly& o) const {
  Poly r;
  for (const auto& [ma, ca] : t_)
    for (const auto& [mb, cb] : o.t_) r.accumulate(ma * mb, ca * cb);
  return r;
}

Poly Poly::operator*(const Rational& c) const {
  Poly r;
  if (c == 0) return r;
  for (const auto& [m, k] : t_) r.t_.emplace(m, k * c);
  return r;
}

Poly Poly::pow(unsigned e) const {
  Poly r = constant(1), base = *this;
  while (e) {  // square-and-multiply; exact, so the order is immaterial
    if (e & 1u) r = r * base;
    e >>= 1u;
    if (e) base = base * base;
  }
  return r;
}

Poly Poly::substitute(const std::string& name, const Poly& value) const {
  Poly r;
  for (const auto& [m, c] : t_) {
    auto hit = m.exps.find(name);
    if (hit == m.exps.end()) {
      r.accumulate(m, c);
      continue;
    }
    Monomial rest = m;
    rest.exps.erase(name);
    Poly term;
    term.t_.emplace(rest, c);
    r += term * value.pow(static_cast<unsigned>(hit->second));
  }
  return r;
}

Rational Poly::eval(const std::map<std::string, long long>& env) const {
  Rational acc(0);
  for (const auto& [m, c] : t_) {
    Rational v = c;
    for (const auto& [sym, e] : m.exps) {
      auto b = env.find(sym);
      if (b == env.end()) throw EvalError("unbound symbol '" + sym + "' in " + str());
      for (int i = 0; i < e; ++i) v *= Rational(b->second);
    }
    acc += v;
  }
  return acc;
}

namespace {

std::string monomial_text(const Monomial& m) {
  std::string s;
  for (const auto& [sym, e] : m.exps) {
    if (!s.empty()) s.push_back('*');
    s += sym;
    if (e > 1) s += "^" + std::to_string(e);
  }
  return s;
}

int exponent_of(const Monomial& m, const std::string& sym) {
  auto it = m.exps.find(sym);
  return it == m.exps.end() ? 0 : it->second;
}

}  // namespace

std::string Poly::str() const {
  if (t_.empty()) return "0";
  BigInt den(1);
  for (const auto& kv : t_) den = lcm(den, denominator(kv.second));

  std::vector<std::string> universe;
  for (const auto& s : symbols()) universe.push_back(s);
  std::vector<const TermMap::value_type*> order;
  for (const auto& kv : t_) order.push_back(&kv);
  std::stable_sort(order.begin(), order.end(), [&](const auto* a, const auto* b) {
    int da = a->first.degree(), db = b->first.degree();
    if (da != db) return da > db;
    for (const auto& s : universe) {
      int ea = exponent_of(a->first, s), eb = exponent_of(b->first, s);
      if (ea != eb) return ea > eb;
    }
    return false;
  });

  std::string out;
  for (size_t i = 0; i < order.size(); ++i) {
    BigInt k = numerator(order[i]->second * Rational(den));
    const bool negative = k < 0;
    if (negative) k = -k;
    if (i == 0)
      out += negative ? "-" : "";
    else
      out += negative ? " - " : " + ";
    std::string mono = monomial_text(order[i]->first);
    if (mono.empty())
      out += k.str();
    else if (k == 1)
      out += mono;
    else
      out += k.str() + "*" + mono;
  }
  return den == 1 ? out : "(" + out + ")/" + den.str();
}

// ---------------------------------------------------------------------------
// Division

namespace {

// Lexicographic comparison over alphabetically ordered symbols: the first
// symbol where the monomials differ decides, larger exponent wins.
bool lex_before(const Monomial& a, const Monomial& b) {
  auto ia = a.exps.begin(), ib = b.exps.begin();
  for (; ia != a.exps.end() && ib != b.exps.end(); ++ia, ++ib) {
    if (ia->first != ib->first) return ia->first < ib->first;
    if (ia->second != ib->second) return ia->second > ib->second;
  }
  return ia != a.exps.end();
}

const Poly::TermMap::value_type& leading(const Poly& p) {
  const Poly::TermMap::value_type* best = nullptr;
  for (const auto& kv : p.terms())
    if (!best || lex_before(kv.first, best->first)) best = &kv;
  return *best;
}

}  // namespace

bool try_divide(const Poly& num, const Poly& den, Poly& quotient) {
  if (den.is_zero()) return false;
  if (num.is_zero()) {
    quotient = Poly();
    return true;
  }
  if (den.is_constant()) {
    quotient = num * (Rational(1) / den.constant_value());
    return true;
  }
  const auto& dlead = leading(den);
  Poly rem = num, q;
  while (!rem.is_zero()) {
    const auto& rlead = leading(rem);
    Monomial factor;
    for (const auto& [sym, e] : rlead.first.exps) {
      int need = exponent_of(dlead.first, sym);
      if (e > need) factor.exps.emplace(sym, e - need);
    }
    for (const auto& [sym, e] : dlead.first.exps)
      if (exponent_of(rlead.first, sym) < e) return false;
    Poly t;
    t.accumulate(factor, rlead.second / dlead.second);
    q += t;
    rem -= t * den;
  }
  quotient = q;
  return true;
}

// ---------------------------------------------------------------------------
// Range sums

namespace {

// F_k(x) = sum_{i=0}^{x} i^k as a polynomial in the reserved symbol "x",
// from (k+1) F_k = (x+1)^{k+1} - sum_{j<k} C(k+1, j) F_j.
const Poly& faulhaber(int k) {
  static std::mutex mu;
  static std::vector<Poly> table;
  std::lock_guard<std::mutex> lock(mu);
  const Poly x1 = Poly::symbol("x") + Poly::constant(1);
  while ((int)table.size() <= k) {
    const int j = (int)table.size();
    Poly acc = x1.pow((unsigned)(j + 1));
    Rational binom(1);  // C(j+1, i)
    for (int i = 0; i < j; ++i) {
      acc -= table[(size_t)i] * binom;
      binom = binom * Rational(j + 1 - i) / Rational(i + 1);
    }
    table.push_back(acc * Rational(1, j + 1));
  }
  return table[(size_t)k];
}

}  // namespace

Poly sum_over_range(const Poly& p, const std::string& iname, const Poly& lo, const Poly& hi) {
  // Group p by the power of iname: p = sum_k c_k(other symbols) * iname^k.
  std::map<int, Poly> by_power;
  for (const auto& [m, c] : p.terms()) {
    Monomial rest = m;
    int k = 0;
    auto it = rest.exps.find(iname);
    if (it != rest.exps.end()) {
      k = it->second;
      rest.exps.erase(it);
    }
    by_power[k].accumulate(rest, c);
  }
  const Poly below = lo - Poly::constant(1);
  Poly total;
  for (const auto& [k, coeff] : by_power) {
    const Poly& f = faulhaber(k);
    total += coeff * (f.substitute("x", hi) - f.substitute("x", below));
  }
  return total;
}

// ---------------------------------------------------------------------------
// PolyRatio

PolyRatio PolyRatio::of(const Poly& n, const Poly& d) {
  Poly q;
  if (try_divide(n, d, q)) return exact(q);
  return PolyRatio{n, d};
}

Rational PolyRatio::eval(const std::map<std::string, long long>& env) const {
  Rational d = den.eval(env);
  if (d == 0) throw EvalError("footprint evaluates to zero in ratio " + str());
  return num.eval(env) / d;
}

std::string PolyRatio::str() const {
  if (is_poly()) return num.str();
  return "(" + num.str() + ")/(" + den.str() + ")";
}

// ---------------------------------------------------------------------------
// AffineExpr

AffineExpr AffineExpr::operator+(const AffineExpr& o) const {
  AffineExpr r = *this;
  for (const auto& [s, c] : o.lin) {
    Poly sum = r.lin.count(s) ? r.lin[s] + c : c;
    if (sum.is_zero())
      r.lin.erase(s);
    else
      r.lin[s] = sum;
  }
  r.off += o.off;
  return r;
}

AffineExpr AffineExpr::operator-() const {
  AffineExpr r;
  for (const auto& [s, c] : lin) r.lin.emplace(s, -c);
  r.off = -off;
  return r;
}

AffineExpr AffineExpr::scaled(const Poly& k) const {
  AffineExpr r;
  if (k.is_zero()) return r;
  for (const auto& [s, c] : lin) r.lin.emplace(s, c * k);
  r.off = off * k;
  return r;
}

AffineExpr AffineExpr::times(const AffineExpr& o) const {
  if (o.is_index_free()) return scaled(o.off);
  if (is_index_free()) return o.scaled(off);
  throw SemanticError("non-affine product of index expressions");
}

AffineExpr AffineExpr::substitute_index(const std::string& name, const AffineExpr& value) const {
  auto it = lin.find(name);
  if (it == lin.end()) return *this;
  AffineExpr base = *this;
  Poly coeff = it->second;
  base.lin.erase(name);
  return base + value.scaled(coeff);
}

AffineExpr AffineExpr::substitute_param(const std::string& name, const Rational& value) const {
  const Poly v = Poly::constant(value);
  AffineExpr r;
  for (const auto& [s, c] : lin) {
    Poly nc = c.substitute(name, v);
    if (!nc.is_zero()) r.lin.emplace(s, nc);
  }
  r.off = off.substitute(name, v);
  return r;
}

Poly AffineExpr::to_poly() const {
  Poly p = off;
  for (const auto& [s, c] : lin) p += c * Poly::symbol(s);
  return p;
}

std::set<std::string> AffineExpr::index_symbols() const {
  std::set<std::string> s;
  for (const auto& kv : lin) s.insert(kv.first);
  return s;
}

std::set<std::string> AffineExpr::all_symbols() const {
  std::set<std::string> s = index_symbols();
  for (const auto& x : off.symbols()) s.insert(x);
  for (const auto& kv : lin)
    for (const auto& x : kv.second.symbols()) s.insert(x);
  return s;
}

bool AffineExpr::strictly_affine() const {
  for (const auto& kv : lin)
    if (!kv.second.is_constant()) return false;
  return off.degree() <= 1;
}

bool AffineExpr::integer_coefficients() const {
  for (const auto& kv : lin)
    if (!kv.second.is_constant() || !is_integer(kv.second.constant_value())) return false;
  for (const auto& kv : off.terms())
    if (!is_integer(kv.second)) return false;
  return true;
}

}  // namespace perfseer
