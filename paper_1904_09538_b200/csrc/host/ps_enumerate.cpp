// Enumeration oracle (see ps_enumerate.hpp). Semantics follow the
// reference's brute-force counter (oracle.cpp:76-443): every statement
// instance is visited, ops are tallied with the same madd-fusion rule,
// access strides are measured by finite differences of the flattened index,
// and footprints are the sets of distinct index tuples.
#include "ps_enumerate.hpp"

#include <functional>
#include <set>
#include <sstream>

namespace perfseer {

std::string NumericPattern::key() const {
  std::ostringstream os;
  os << "mem:" << mem << ":" << dir << ":" << dtype_bytes << ":tag=" << tag << ":ls={";
  const char* sep = "";
  for (const auto& [a, s] : lstrides) os << sep << a << ":" << s, sep = ";";
  os << "}:gs={";
  sep = "";
  for (const auto& [a, s] : gstrides) os << sep << a << ":" << s, sep = ";";
  os << "}:loop=";
  if (has_loop_stride)
    os << loop_stride;
  else
    os << "-";
  return os.str();
}

namespace {

using Env = std::map<std::string, long long>;

long long as_int(const Rational& v, const std::string& what) {
  if (!is_integer(v)) throw EvalError(what + " is not integral");
  return numerator(v).convert_to<long long>();
}

long long eval_int(const AffineExpr& a, const Env& env) {
  return as_int(a.eval(env), "affine expression " + a.str());
}

}  // namespace

NumericPattern evaluate_pattern(const AccessPattern& p, const std::map<std::string, long long>& b) {
  NumericPattern n;
  n.mem = memtype_str(p.mem);
  n.dir = direction_str(p.dir);
  n.dtype_bytes = p.dtype_bytes;
  n.tag = p.tag;
  n.gran = granularity_str(p.gran);
  for (const auto& [a, s] : p.lstrides) n.lstrides[a] = as_int(s.eval(b), "stride " + s.str());
  for (const auto& [a, s] : p.gstrides) n.gstrides[a] = as_int(s.eval(b), "stride " + s.str());
  if (p.loop_stride) {
    n.has_loop_stride = true;
    n.loop_stride = as_int(p.loop_stride->eval(b), "stride " + p.loop_stride->str());
  }
  return n;
}

NumericPattern probe_pattern(const Kernel& k, const Statement& s, const Access& a, Direction dir,
                             const std::vector<std::string>& binders,
                             const std::map<std::string, long long>& b) {
  std::map<int, std::string> local, group;
  for (const auto& [iname, tag] : k.iname_tags) {
    if (tag.kind == InameTag::Kind::local) local[tag.axis] = iname;
    if (tag.kind == InameTag::Kind::group) group[tag.axis] = iname;
  }
  const ArgDecl& decl = k.arg(a.array);
  NumericPattern p;
  p.mem = decl.space == MemSpace::local ? "local" : "global";
  p.dir = direction_str(dir);
  p.dtype_bytes = dtype_bytes(decl.dtype);
  p.tag = a.tag;
  std::vector<long long> row(decl.shape.size(), 1);
  for (size_t d = decl.shape.size(); d-- > 1;) row[d - 1] = row[d] * eval_int(decl.shape[d], b);
  auto flat = [&](const Env& env) {
    long long f = 0;
    for (size_t d = 0; d < a.subs.size(); ++d) f += eval_int(a.subs[d], env) * row[d];
    return f;
  };
  // d(flat)/d(iname) measured at two base points; affine => equal.
  auto slope = [&](const std::string& iname) {
    long long d[2];
    for (int base = 0; base < 2; ++base) {
      Env e = b;
      for (const auto& o : k.domain.inames) e[o] = base;
      const long long f0 = flat(e);
      e[iname] += 1;
      d[base] = flat(e) - f0;
    }
    if (d[0] != d[1]) throw EvalError("non-affine subscript on '" + a.array + "'");
    return d[0];
  };
  for (const auto& [axis, i] : local) p.lstrides[axis] = slope(i);
  for (const auto& [axis, i] : group) p.gstrides[axis] = slope(i);
  std::vector<std::string> order = k.ordered_within(s);
  order.insert(order.end(), binders.begin(), binders.end());
  for (auto it = order.rbegin(); it != order.rend(); ++it)
    if (k.is_sequential(*it)) {
      p.has_loop_stride = true;
      p.loop_stride = slope(*it);
      break;
    }
  const bool uniform = p.lstrides.count(0) && p.lstrides.at(0) == 0;
  p.gran = (p.mem == "local" || uniform) ? "sub_group" : "work_item";
  return p;
}

namespace {

class Visitor {
 public:
  Visitor(const Kernel& k, const Env& b, long long budget)
      : k_(k), b_(b), budget_(budget), types_(infer_types(k)) {
    for (const auto& [iname, tag] : k.iname_tags) {
      if (tag.kind == InameTag::Kind::local) local_[tag.axis] = iname;
      if (tag.kind == InameTag::Kind::group) group_[tag.axis] = iname;
    }
  }

  OracleCounts run() {
    for (const auto& s : k_.statements) {
      if (s.is_barrier) {
        count_barriers(s);
        continue;
      }
      register_sites(s);
      Env env = b_;
      loop_nest(k_.ordered_within(s), 0, env, [&](Env& e) {
        if (!s.lhs.is_scalar()) hit(s, s.lhs, Direction::store, e);
        walk(s, s.rhs, e);
      });
    }
    OracleCounts out;
    out.ops = ops_;
    out.barrier_local = barriers_;
    for (const auto& [key, ids] : groups_) {
      long long n = 0;
      std::set<std::pair<std::string, std::vector<long long>>> seen;
      for (size_t id : ids) {
        n += sites_[id].count;
        for (const auto& t : sites_[id].tuples) seen.insert({sites_[id].access.array, t});
      }
      out.access_counts[key] = n;
      out.access_footprints[key] = (long long)seen.size();
      out.access_gran[key] = sites_[ids.front()].pattern.gran;
    }
    for (const auto& [a, tuples] : per_array_) out.footprints[a] = (long long)tuples.size();
    if (!group_.empty() || k_.single_work_item) {
      long long g = 1;
      for (const auto& [axis, iname] : group_) {
        const Bound& bd = k_.domain.bound(iname);
        g *= eval_int(bd.hi, b_) - eval_int(bd.lo, b_) + 1;
      }
      out.group_launch = g;
      out.has_group_launch = true;
    } else if (!local_.empty()) {
      out.group_launch = 1;
      out.has_group_launch = true;
    }
    return out;
  }

 private:
  struct Site {
    std::string stmt;
    Access access;
    Direction dir;
    NumericPattern pattern;
    long long count = 0;
    std::set<std::vector<long long>> tuples;
  };

  void spend() {
    if (++visited_ > budget_) throw EvalError("brute-force enumeration exceeds the point budget");
  }

  void loop_nest(const std::vector<std::string>& order, size_t depth, Env& env,
                 const std::function<void(Env&)>& body) {
    if (depth == order.size()) {
      spend();
      body(env);
      return;
    }
    const std::string& i = order[depth];
    const Bound& bd = k_.domain.bound(i);
    const long long lo = eval_int(bd.lo, env), hi = eval_int(bd.hi, env);
    if (lo > hi + 1) throw EvalError("negative range for iname '" + i + "' at this binding");
    for (long long v = lo; v <= hi; ++v) {
      env[i] = v;
      loop_nest(order, depth + 1, env, body);
    }
    env.erase(i);
  }

  void count_barriers(const Statement& s) {
    std::vector<std::string> seq;
    for (const auto& i : k_.ordered_within(s))
      if (k_.is_sequential(i)) seq.push_back(i);
    Env env = b_;
    loop_nest(seq, 0, env, [&](Env&) { ++barriers_; });
  }

  NumericPattern probe(const Statement& s, const Access& a, Direction dir,
                       const std::vector<std::string>& binders) {
    return probe_pattern(k_, s, a, dir, binders, b_);
  }

  void add_site(const Statement& s, const Access& a, Direction dir, const std::vector<std::string>& binders) {
    if (k_.arg(a.array).space == MemSpace::private_mem) return;
    Site x;
    x.stmt = s.id;
    x.access = a;
    x.dir = dir;
    x.pattern = probe(s, a, dir, binders);
    groups_[x.pattern.key()].push_back(sites_.size());
    by_stmt_[s.id].push_back(sites_.size());
    sites_.push_back(std::move(x));
  }

  void register_sites(const Statement& s) {
    by_stmt_[s.id];
    if (!s.lhs.is_scalar()) add_site(s, s.lhs, Direction::store, {});
    std::vector<std::string> binders;
    std::function<void(const ExprPtr&)> rec = [&](const ExprPtr& e) {
      if (!e) return;
      if (e->kind == Expr::Kind::access) {
        add_site(s, e->access, Direction::load, binders);
      } else if (e->kind == Expr::Kind::binary) {
        rec(e->lhs);
        rec(e->rhs);
      } else if (e->kind == Expr::Kind::reduction) {
        binders.push_back(e->red_iname);
        rec(e->body);
        binders.pop_back();
      }
    };
    rec(s.rhs);
  }

  void hit(const Statement& s, const Access& a, Direction dir, const Env& env) {
    if (k_.arg(a.array).space == MemSpace::private_mem) return;
    for (size_t id : by_stmt_[s.id]) {
      Site& x = sites_[id];
      if (x.dir != dir || !(x.access == a)) continue;
      ++x.count;
      std::vector<long long> t;
      for (const auto& sub : a.subs) t.push_back(eval_int(sub, env));
      x.tuples.insert(t);
      per_array_[a.array].insert(t);
      return;
    }
    throw EvalError("internal: access site not registered");
  }

  void op(const ExprPtr& e, OpName n) { ++ops_[OpKind{expr_dtype(e, k_, types_), n}.key()]; }

  void walk(const Statement& s, const ExprPtr& e, Env& env) {
    if (!e) return;
    switch (e->kind) {
      case Expr::Kind::number:
      case Expr::Kind::scalar_ref:
        return;
      case Expr::Kind::access:
        hit(s, e->access, Direction::load, env);
        return;
      case Expr::Kind::binary: {
        if (e->op == BinOp::add || e->op == BinOp::sub) {
          auto is_mul = [](const ExprPtr& x) { return x->kind == Expr::Kind::binary && x->op == BinOp::mul; };
          const ExprPtr* f = is_mul(e->rhs) ? &e->rhs : is_mul(e->lhs) ? &e->lhs : nullptr;
          if (!s.harness) op(e, f ? OpName::madd : OpName::add);
          if (f) {
            walk(s, *f == e->rhs ? e->lhs : e->rhs, env);
            walk(s, (*f)->lhs, env);
            walk(s, (*f)->rhs, env);
          } else {
            walk(s, e->lhs, env);
            walk(s, e->rhs, env);
          }
          return;
        }
        if (!s.harness) op(e, e->op == BinOp::mul ? OpName::mul : OpName::div);
        walk(s, e->lhs, env);
        walk(s, e->rhs, env);
        return;
      }
      case Expr::Kind::reduction: {
        std::vector<std::string> binders{e->red_iname};
        ExprPtr body = e->body;
        while (body->kind == Expr::Kind::reduction) {
          binders.push_back(body->red_iname);
          body = body->body;
        }
        loop_nest(binders, 0, env, [&](Env& inner) {
          if (!s.harness) {
            if (body->kind == Expr::Kind::binary && body->op == BinOp::mul) {
              op(body, OpName::madd);
              walk(s, body->lhs, inner);
              walk(s, body->rhs, inner);
              return;
            }
            op(body, OpName::add);
          }
          walk(s, body, inner);
        });
        return;
      }
    }
  }

  const Kernel& k_;
  Env b_;
  long long budget_;
  long long visited_ = 0;
  std::map<std::string, Dtype> types_;
  std::map<int, std::string> local_, group_;
  std::map<std::string, long long> ops_;
  long long barriers_ = 0;
  std::vector<Site> sites_;
  std::map<std::string, std::vector<size_t>> groups_, by_stmt_;
  std::map<std::string, std::set<std::vector<long long>>> per_array_;
};

}  // namespace

OracleCounts brute_force_count(const Kernel& k, const std::map<std::string, long long>& bindings,
                               long long max_points) {
  for (const auto& a : k.assumptions) {
    auto it = bindings.find(a.param);
    if (it == bindings.end()) continue;
    const bool ok = a.kind == Assumption::Kind::divisible ? it->second % a.value == 0 : it->second >= a.value;
    if (!ok)
      throw EvalError("binding " + a.param + "=" + std::to_string(it->second) + " violates assumption " + a.str());
  }
  return Visitor(k, bindings, max_points).run();
}

}  // namespace perfseer
