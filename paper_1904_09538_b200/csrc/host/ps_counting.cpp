// Counting engine (see ps_counting.hpp). Behaviour follows the reference's
// Alg. 1 / Alg. 2 implementation (counting.cpp:111-674) so every count,
// pattern key and footprint is identical; the cache is keyed by a 128-bit
// structural hash instead of a JSON dump per lookup.
#include "ps_counting.hpp"

#include <algorithm>
#include <atomic>
#include <mutex>
#include <sstream>
#include <unordered_map>

#include "ps_transforms.hpp"

namespace perfseer {

std::string granularity_str(Granularity g) {
  static const char* names[] = {"work_item", "sub_group", "work_group", "kernel"};
  return names[static_cast<int>(g)];
}
std::string opname_str(OpName n) {
  static const char* names[] = {"add", "mul", "madd", "div", "pow"};
  return names[static_cast<int>(n)];
}
std::string memtype_str(MemType m) { return m == MemType::global_mem ? "global" : "local"; }
std::string direction_str(Direction d) { return d == Direction::load ? "load" : "store"; }
std::string synckind_str(SyncKind k) {
  static const char* names[] = {"barrier_local", "kernel_launch", "group_launch"};
  return names[static_cast<int>(k)];
}

bool AccessPattern::uniform() const {
  auto it = lstrides.find(0);
  return it != lstrides.end() && it->second.is_zero();
}

namespace {
std::string stride_map_text(const std::map<int, Poly>& m) {
  std::string s = "{";
  bool first = true;
  for (const auto& [axis, p] : m) {
    s += (first ? "" : ";") + std::to_string(axis) + ":" + p.str();
    first = false;
  }
  return s + "}";
}
}  // namespace

std::string AccessPattern::key() const {
  return "mem:" + memtype_str(mem) + ":" + direction_str(dir) + ":" + std::to_string(dtype_bytes) +
         ":tag=" + tag + ":ls=" + stride_map_text(lstrides) + ":gs=" + stride_map_text(gstrides) +
         ":loop=" + (loop_stride ? loop_stride->str() : std::string("-"));
}

std::string AccessPattern::str() const {
  return key() + ":afr=" + afr.str() + ":" + granularity_str(gran);
}

// ---------------------------------------------------------------------------
// Assumption reasoning

namespace {

long long modulus_of(const std::vector<Assumption>& as, const std::string& sym) {
  long long m = 1;
  for (const auto& a : as)
    if (a.kind == Assumption::Kind::divisible && a.param == sym) m = std::max(m, a.value);
  return m;
}

// Integer at every point where each symbol is a multiple of its modulus:
// each term's coefficient times the moduli powers must be integral.
bool integral_poly(const Poly& p, const std::vector<Assumption>& as) {
  for (const auto& [mono, c] : p.terms()) {
    if (is_integer(c)) continue;
    Rational scaled = c;
    for (const auto& [sym, e] : mono.exps)
      for (int i = 0; i < e; ++i) scaled *= Rational(modulus_of(as, sym));
    if (!is_integer(scaled)) return false;
  }
  return true;
}

}  // namespace

bool integer_valued_under(const AffineExpr& e, const std::vector<Assumption>& as) {
  for (const auto& kv : e.lin)
    if (!integral_poly(kv.second, as)) return false;
  return integral_poly(e.off, as);
}

RegionSign region_sign(const Poly& p, const std::vector<Assumption>& as) {
  if (p.is_zero()) return RegionSign::zero;
  if (p.is_constant())
    return p.constant_value() >= 0 ? RegionSign::always_nonneg : RegionSign::always_neg;
  // Smallest admissible value per symbol: its largest lower bound rounded up
  // to its divisibility modulus. With all non-constant coefficients of one
  // sign, the polynomial is monotone on [low, inf) and its extreme is at low.
  std::map<std::string, long long> low;
  for (const auto& sym : p.symbols()) {
    std::optional<long long> lb;
    for (const auto& a : as)
      if (a.kind == Assumption::Kind::lower_bound && a.param == sym && (!lb || a.value > *lb))
        lb = a.value;
    if (!lb) return RegionSign::unknown;
    long long m = modulus_of(as, sym), v = *lb;
    if (m > 1) {
      long long q = v / m;
      if (q * m < v) ++q;
      v = q * m;
    }
    if (v < 0) return RegionSign::unknown;
    low[sym] = v;
  }
  bool has_pos = false, has_neg = false;
  for (const auto& [mono, c] : p.terms()) {
    if (mono.exps.empty()) continue;
    if (c > 0) has_pos = true;
    if (c < 0) has_neg = true;
  }
  const Rational at_low = p.eval(low);
  if (!has_neg) return at_low >= 0 ? RegionSign::always_nonneg : RegionSign::unknown;
  if (!has_pos) return at_low < 0 ? RegionSign::always_neg : RegionSign::unknown;
  return RegionSign::unknown;
}

// ---------------------------------------------------------------------------
// Projections

namespace {
std::atomic<uint64_t> g_projection_counter{0};
}

uint64_t projection_count() { return g_projection_counter.load(); }

Poly count_points(const LoopDomain& d, const std::set<std::string>& subset,
                  const std::vector<Assumption>& as) {
  for (const auto& iname : subset) {
    if (!d.has_iname(iname)) throw CountError("projection onto unknown iname '" + iname + "'");
    const Bound& b = d.bound(iname);
    for (const AffineExpr* side : {&b.lo, &b.hi}) {
      for (const auto& sym : side->index_symbols())
        if (!subset.count(sym))
          throw CountError("projection subset not closed under bound references: '" + iname +
                           "' depends on '" + sym + "'");
      if (!integer_valued_under(*side, as))
        throw CountError("bound " + side->str() + " of '" + iname + "' needs divisibility assumption");
    }
  }
  ++g_projection_counter;
  Poly n = Poly::constant(1);
  for (auto it = d.inames.rbegin(); it != d.inames.rend(); ++it)
    if (subset.count(*it)) {
      const Bound& b = d.bound(*it);
      n = sum_over_range(n, *it, b.lo.to_poly(), b.hi.to_poly());
    }
  for (const auto& sym : n.symbols())
    if (d.has_iname(sym)) throw CountError("projection left unresolved iname '" + sym + "'");
  return n;
}

// ---------------------------------------------------------------------------
// Per-kernel analysis

namespace {

struct AccessSite {
  Access access;
  std::set<std::string> context;       // within + reduction binders
  Direction dir;
  std::vector<std::string> loop_order;  // nesting order, binders innermost
};

// Decides a <= b over the assumed region or throws.
struct RegionOrder {
  const std::vector<Assumption>& as;
  bool le(const Poly& a, const Poly& b) const {
    switch (region_sign(b - a, as)) {
      case RegionSign::always_nonneg:
      case RegionSign::zero: return true;
      case RegionSign::always_neg: return false;
      default:
        throw CountError("footprint comparison " + a.str() + " <= " + b.str() +
                         " is undecidable; needs lower-bound assumption");
    }
  }
};

class Counter {
 public:
  explicit Counter(const Kernel& k) : k_(k), types_(infer_types(k)) {
    for (const auto& [iname, tag] : k.iname_tags) {
      if (tag.kind == InameTag::Kind::local) local_of_[tag.axis] = iname;
      if (tag.kind == InameTag::Kind::group) group_of_[tag.axis] = iname;
    }
  }

  KernelCounts run(bool accesses) {
    KernelCounts out;
    try {
      out.geometry = launch_geometry(k_);
    } catch (const SemanticError&) {
      out.geometry.reset();
    }
    for (const auto& s : k_.statements) {
      if (s.is_barrier) {
        std::set<std::string> seq;
        for (const auto& i : s.within)
          if (k_.is_sequential(i)) seq.insert(i);
        sync(out, SyncKind::barrier_local, points(seq));
        continue;
      }
      if (!s.lhs.is_scalar()) site(s, s.lhs, Direction::store, {});
      walk(s, s.rhs, {});
    }
    sync(out, SyncKind::kernel_launch, Poly::constant(1));
    if (out.geometry) sync(out, SyncKind::group_launch, out.geometry->total_groups());

    for (const auto& [key, n] : ops_)
      if (!n.is_zero())
        out.ops.push_back(CountedOp{OpKind{key.first, key.second, Granularity::sub_group}, n});
    std::sort(out.ops.begin(), out.ops.end(),
              [](const CountedOp& a, const CountedOp& b) { return a.kind.key() < b.kind.key(); });

    if (accesses) {
      group_accesses(out);
      for (const auto& a : k_.args) {
        if (a.space == MemSpace::private_mem) continue;
        auto it = by_array_.find(a.name);
        if (it != by_array_.end()) out.footprints[a.name] = union_footprint(it->second);
      }
    }
    return out;
  }

 private:
  Poly points(const std::set<std::string>& subset) {
    auto it = proj_.find(subset);
    if (it != proj_.end()) return it->second;
    Poly p = count_points(k_.domain, subset, k_.assumptions);
    proj_.emplace(subset, p);
    return p;
  }

  Poly points_with(const Statement& s, const std::vector<std::string>& binders) {
    std::set<std::string> ctx = s.within;
    ctx.insert(binders.begin(), binders.end());
    return points(ctx);
  }

  static void sync(KernelCounts& out, SyncKind kind, const Poly& n) {
    for (auto& e : out.sync)
      if (e.kind == kind) {
        e.count += n;
        return;
      }
    out.sync.push_back(CountedSync{kind, n});
  }

  void op(const ExprPtr& node, OpName name, const Poly& n) {
    ops_[{expr_dtype(node, k_, types_), name}] += n;
  }

  void site(const Statement& s, const Access& a, Direction dir,
            const std::vector<std::string>& binders) {
    if (k_.arg(a.array).space == MemSpace::private_mem) return;
    AccessSite x{a, s.within, dir, k_.ordered_within(s)};
    for (const auto& b : binders) {
      x.context.insert(b);
      x.loop_order.push_back(b);
    }
    sites_.push_back(x);
    by_array_[a.array].push_back(x);
  }

  // Alg. 1 with madd fusion: a multiply directly under an add/sub (right
  // operand preferred) fuses into one madd; a reduction accumulates once per
  // iteration, fusing a multiply at the body root. Work-removal (harness)
  // statements record accesses but no arithmetic.
  void walk(const Statement& s, const ExprPtr& e, std::vector<std::string> binders) {
    const bool count = !s.harness;
    switch (e->kind) {
      case Expr::Kind::number:
      case Expr::Kind::scalar_ref:
        return;
      case Expr::Kind::access:
        site(s, e->access, Direction::load, binders);
        return;
      case Expr::Kind::binary: {
        const Poly n = points_with(s, binders);
        if (e->op == BinOp::add || e->op == BinOp::sub) {
          auto is_mul = [](const ExprPtr& x) { return x->kind == Expr::Kind::binary && x->op == BinOp::mul; };
          const ExprPtr* fused = is_mul(e->rhs) ? &e->rhs : is_mul(e->lhs) ? &e->lhs : nullptr;
          if (count) op(e, fused ? OpName::madd : OpName::add, n);
          if (fused) {
            walk(s, *fused == e->rhs ? e->lhs : e->rhs, binders);
            walk(s, (*fused)->lhs, binders);
            walk(s, (*fused)->rhs, binders);
          } else {
            walk(s, e->lhs, binders);
            walk(s, e->rhs, binders);
          }
          return;
        }
        if (count) op(e, e->op == BinOp::mul ? OpName::mul : OpName::div, n);
        walk(s, e->lhs, binders);
        walk(s, e->rhs, binders);
        return;
      }
      case Expr::Kind::reduction: {
        ExprPtr body = e->body;
        binders.push_back(e->red_iname);
        while (body->kind == Expr::Kind::reduction) {  // split summation: one accumulator
          binders.push_back(body->red_iname);
          body = body->body;
        }
        const Poly n = points_with(s, binders);
        if (count) {
          if (body->kind == Expr::Kind::binary && body->op == BinOp::mul) {
            op(body, OpName::madd, n);
            walk(s, body->lhs, binders);
            walk(s, body->rhs, binders);
            return;
          }
          op(body, OpName::add, n);
        }
        walk(s, body, binders);
        return;
      }
    }
  }

  AccessPattern classify(const AccessSite& x) {
    const ArgDecl& decl = k_.arg(x.access.array);
    const size_t rank = decl.shape.size();
    // Row-major element strides of each array axis.
    std::vector<Poly> axis_stride(rank, Poly::constant(1));
    for (size_t d = rank; d-- > 1;) {
      if (!decl.shape[d].is_index_free())
        throw CountError("shape of '" + decl.name + "' references an iname");
      axis_stride[d - 1] = axis_stride[d] * decl.shape[d].off;
    }
    std::map<std::string, Poly> flat;
    for (size_t d = 0; d < rank; ++d)
      for (const auto& [sym, c] : x.access.subs[d].lin) flat[sym] += c * axis_stride[d];
    auto coeff = [&](const std::string& i) {
      auto it = flat.find(i);
      return it == flat.end() ? Poly() : it->second;
    };
    AccessPattern p;
    p.mem = decl.space == MemSpace::local ? MemType::local_mem : MemType::global_mem;
    p.dir = x.dir;
    p.dtype_bytes = dtype_bytes(decl.dtype);
    p.tag = x.access.tag;
    for (const auto& [axis, i] : local_of_) p.lstrides[axis] = coeff(i);
    for (const auto& [axis, i] : group_of_) p.gstrides[axis] = coeff(i);
    for (auto it = x.loop_order.rbegin(); it != x.loop_order.rend(); ++it)
      if (k_.is_sequential(*it)) {
        p.loop_stride = coeff(*it);
        break;
      }
    p.gran = (p.mem == MemType::local_mem || p.uniform()) ? Granularity::sub_group
                                                          : Granularity::work_item;
    return p;
  }

  void group_accesses(KernelCounts& out) {
    struct Group {
      AccessPattern pattern;
      Poly count;
      std::map<std::string, std::vector<AccessSite>> per_array;
    };
    std::map<std::string, Group> groups;
    for (const auto& x : sites_) {
      AccessPattern p = classify(x);
      auto& g = groups.emplace(p.key(), Group{p, Poly(), {}}).first->second;
      g.count += points(x.context);
      g.per_array[x.access.array].push_back(x);
    }
    for (auto& [key, g] : groups) {
      Poly fp;
      for (const auto& [array, xs] : g.per_array) fp += union_footprint(xs);
      g.pattern.afr = PolyRatio::of(g.count, fp);
      out.accesses.push_back(CountedAccess{g.pattern, g.count});
    }
  }

  Poly union_footprint(const std::vector<AccessSite>& xs);

  const Kernel& k_;
  std::map<std::string, Dtype> types_;
  std::map<int, std::string> local_of_, group_of_;
  std::map<std::set<std::string>, Poly> proj_;
  std::map<std::pair<Dtype, OpName>, Poly> ops_;
  std::vector<AccessSite> sites_;
  std::map<std::string, std::vector<AccessSite>> by_array_;
};

// Alg. 2: each site's index set is, per array axis, an arithmetic
// progression (offset, step, span); sites are aligned to a common step per
// axis and the union size follows by inclusion-exclusion over the sites'
// axis-interval boxes.
Poly Counter::union_footprint(const std::vector<AccessSite>& xs) {
  if (xs.empty()) return Poly();
  const ArgDecl& decl = k_.arg(xs.front().access.array);
  const size_t rank = decl.shape.size();
  const RegionOrder order{k_.assumptions};
  auto irreducible = [&](const std::string& why = "") {
    return CountError("step-irreducible footprint for '" + decl.name + "'" + why);
  };

  struct Prog {
    Poly offset, step = Poly::constant(1), span;
    bool single = true;
  };
  std::vector<std::vector<Prog>> prog(xs.size(), std::vector<Prog>(rank));
  for (size_t si = 0; si < xs.size(); ++si) {
    const AccessSite& x = xs[si];
    std::set<std::string> seen;
    for (size_t d = 0; d < rank; ++d) {
      const AffineExpr& sub = x.access.subs[d];
      for (const auto& kv : sub.lin) {
        if (!seen.insert(kv.first).second)
          throw CountError("non-rectangular footprint: iname '" + kv.first +
                           "' appears in several axes of '" + decl.name + "'");
      }
      struct Leg {
        Poly stride, trip;
      };
      std::vector<Leg> legs;
      Poly offset = sub.off;
      for (const auto& [sym, coeff] : sub.lin) {
        if (!x.context.count(sym))
          throw CountError("subscript iname '" + sym + "' outside statement context");
        const Bound& b = k_.domain.bound(sym);
        if (!b.lo.is_index_free() || !b.hi.is_index_free())
          throw CountError("non-rectangular footprint: bounds of '" + sym + "' depend on another iname");
        const Poly trip = (b.hi - b.lo + AffineExpr::constant(1)).off;
        Poly stride = coeff;
        const RegionSign sign = region_sign(stride, k_.assumptions);
        if (sign == RegionSign::zero) continue;
        if (sign == RegionSign::always_neg) {
          offset += stride * (trip - Poly::constant(1));  // walk it backwards
          stride = -stride;
        } else if (sign != RegionSign::always_nonneg) {
          throw CountError("stride sign of '" + sym + "' in '" + decl.name +
                           "' is undecidable; needs lower-bound assumption");
        }
        offset += coeff * b.lo.off;
        legs.push_back(Leg{stride, trip});
      }
      std::sort(legs.begin(), legs.end(), [&](const Leg& a, const Leg& b) {
        return order.le(a.stride, b.stride) && !(a.stride == b.stride);
      });
      Prog pr;
      pr.offset = offset;
      for (const auto& leg : legs) {
        const Poly extent = leg.stride * (leg.trip - Poly::constant(1));
        if (pr.single) {
          pr.step = leg.stride;
          pr.span = extent;
          pr.single = false;
          continue;
        }
        Poly ratio;
        if (!try_divide(leg.stride, pr.step, ratio) || !integral_poly(ratio, k_.assumptions))
          throw irreducible();
        if (!order.le(leg.stride, pr.span + pr.step))
          throw irreducible(": stride " + leg.stride.str() + " leaves gaps");
        pr.span = extent + pr.span;
      }
      prog[si][d] = pr;
    }
  }

  // Step-unit intervals [a, b] per site and axis.
  std::vector<std::vector<std::pair<Poly, Poly>>> box(xs.size(), std::vector<std::pair<Poly, Poly>>(rank));
  for (size_t d = 0; d < rank; ++d) {
    std::optional<Poly> step;
    for (size_t si = 0; si < xs.size(); ++si) {
      const Prog& pr = prog[si][d];
      if (pr.single) continue;
      if (!step)
        step = pr.step;
      else if (!(pr.step == *step))
        throw CountError("sites with mismatched steps in footprint of '" + decl.name + "'");
    }
    const Poly unit = step ? *step : Poly::constant(1);
    for (size_t si = 0; si < xs.size(); ++si) {
      const Prog& pr = prog[si][d];
      Poly a, len;
      if (!try_divide(pr.offset - prog[0][d].offset, unit, a) || !integral_poly(a, k_.assumptions))
        throw CountError("sites with incompatible offsets in footprint of '" + decl.name + "'");
      if (!pr.single && (!try_divide(pr.span, unit, len) || !integral_poly(len, k_.assumptions)))
        throw irreducible();
      box[si][d] = {a, a + len};
    }
  }

  const size_t n = xs.size();
  if (n > 20) throw CountError("too many access sites for exact footprint union");
  Poly total;
  for (size_t mask = 1; mask < (size_t(1) << n); ++mask) {
    const int members = __builtin_popcountll(mask);
    Poly term = Poly::constant(1);
    bool empty = false;
    for (size_t d = 0; d < rank && !empty; ++d) {
      std::optional<Poly> lo, hi;
      for (size_t si = 0; si < n; ++si) {
        if (!(mask >> si & 1)) continue;
        const auto& [a, b] = box[si][d];
        if (!lo) {
          lo = a;
          hi = b;
          continue;
        }
        if (order.le(*lo, a)) lo = a;
        if (order.le(b, *hi)) hi = b;
      }
      const Poly size = *hi - *lo + Poly::constant(1);
      if (members == 1) {
        term = term * size;
        continue;
      }
      bool is_member_extent = false;
      for (size_t si = 0; si < n && !is_member_extent; ++si)
        if ((mask >> si & 1) && box[si][d].first == *lo && box[si][d].second == *hi)
          is_member_extent = true;
      if (is_member_extent) {
        term = term * size;
        continue;
      }
      switch (region_sign(size, k_.assumptions)) {
        case RegionSign::always_neg:
        case RegionSign::zero: empty = true; break;
        case RegionSign::always_nonneg: term = term * size; break;
        default:
          throw CountError("footprint intersection size " + size.str() +
                           " is undecidable; needs lower-bound assumption");
      }
    }
    if (empty) continue;
    if (members % 2)
      total += term;
    else
      total -= term;
  }
  return total;
}

}  // namespace

std::vector<CountedOp> count_ops(const Kernel& k) { return Counter(k).run(false).ops; }
std::vector<CountedAccess> classify_accesses(const Kernel& k) { return Counter(k).run(true).accesses; }
std::vector<CountedSync> count_sync(const Kernel& k) { return Counter(k).run(false).sync; }
KernelCounts analyze(const Kernel& k) { return Counter(k).run(true); }

Poly footprint(const Kernel& k, const std::string& array) {
  KernelCounts c = Counter(k).run(true);
  auto it = c.footprints.find(array);
  if (it != c.footprints.end()) return it->second;
  if (!k.find_arg(array)) throw CountError("footprint of unknown array '" + array + "'");
  return Poly();
}

// ---------------------------------------------------------------------------
// Cache

namespace {

// Two independent FNV-1a streams over a canonical structural rendering.
struct Hash128 {
  uint64_t a = 1469598103934665603ull, b = 0x84222325cbf29ce4ull;
  void bytes(const std::string& s) {
    for (unsigned char c : s) {
      a = (a ^ c) * 1099511628211ull;
      b = (b ^ c) * 0x100000001b3ull + 0x9e37u;
    }
    a = (a ^ 0xff) * 1099511628211ull;
    b = (b ^ 0xfe) * 0x100000001b3ull;
  }
};

void hash_expr(Hash128& h, const ExprPtr& e) {
  if (!e) return h.bytes("~");
  switch (e->kind) {
    case Expr::Kind::number:
      h.bytes("#" + e->number.str() + (e->number_is_float ? "f" : "i"));
      return;
    case Expr::Kind::scalar_ref:
      h.bytes("$" + e->name);
      return;
    case Expr::Kind::access:
      h.bytes("@" + e->access.array + "/" + e->access.tag);
      for (const auto& s : e->access.subs) h.bytes(s.str() + "|" + [&] {
        std::string t;
        for (const auto& kv : s.lin) t += kv.first + ":" + kv.second.str() + ";";
        return t;
      }());
      return;
    case Expr::Kind::binary:
      h.bytes("(" + binop_str(e->op));
      hash_expr(h, e->lhs);
      hash_expr(h, e->rhs);
      return;
    case Expr::Kind::reduction:
      h.bytes("S" + e->red_iname);
      hash_expr(h, e->body);
      return;
  }
}

std::pair<uint64_t, uint64_t> structural_hash(const Kernel& k) {
  Hash128 h;
  h.bytes(k.name);
  for (const auto& i : k.domain.inames) {
    const Bound& b = k.domain.bound(i);
    h.bytes(i + "[" + b.lo.str() + "," + b.hi.str() + "]" + k.tag_of(i).str());
  }
  for (const auto& p : k.domain.parameters) h.bytes("p" + p);
  for (const auto& a : k.assumptions) h.bytes(a.str());
  for (const auto& a : k.args) {
    std::string s = a.name + ":" + dtype_str(a.dtype) + ":" + memspace_str(a.space);
    for (const auto& d : a.shape) s += "," + d.str();
    h.bytes(s);
  }
  for (const auto& s : k.statements) {
    std::string head = s.id + (s.is_barrier ? "!b" : "") + (s.harness ? "!h" : "");
    for (const auto& w : s.within) head += " w" + w;
    for (const auto& d : s.depends_on) head += " d" + d;
    h.bytes(head);
    if (s.is_barrier) continue;
    hash_expr(h, Expr::make_access(s.lhs));
    hash_expr(h, s.rhs);
  }
  h.bytes(k.single_work_item ? "swi" : "-");
  return {h.a, h.b};
}

struct PairHash {
  size_t operator()(const std::pair<uint64_t, uint64_t>& p) const { return p.first ^ (p.second * 31); }
};

std::mutex g_cache_mu;
std::unordered_map<std::pair<uint64_t, uint64_t>, std::shared_ptr<const KernelCounts>, PairHash> g_cache;

}  // namespace

std::shared_ptr<const KernelCounts> analyze_cached(const Kernel& k) {
  const auto key = structural_hash(k);
  {
    std::lock_guard<std::mutex> lock(g_cache_mu);
    auto it = g_cache.find(key);
    if (it != g_cache.end()) return it->second;
  }
  auto counts = std::make_shared<const KernelCounts>(analyze(k));
  std::lock_guard<std::mutex> lock(g_cache_mu);
  g_cache[key] = counts;
  return counts;
}

void clear_count_cache() {
  std::lock_guard<std::mutex> lock(g_cache_mu);
  g_cache.clear();
}

}  // namespace perfseer
