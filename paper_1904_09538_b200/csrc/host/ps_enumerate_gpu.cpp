// GPU brute-force counter: the kernel IR at concrete bindings
// becomes a flat program of loop nests (one per statement, one per statement
// x reduction-binder set, one per barrier's sequential inames) and access
// sites; csrc/cuda/enum.cu visits every point on the device. Tallies fold
// into the same OracleCounts the CPU enumerator (ps_enumerate.cpp, reference
// oracle.cpp:76-443) produces, so the two are compared exactly.
#include <algorithm>
#include <map>
#include <set>
#include <string>
#include <vector>

#include "../../../include/perfseer_b200.h"
#include "../cuda/enum_program.h"
#include "ps_enumerate.hpp"

namespace perfseer {

namespace {

using Env = std::map<std::string, long long>;

long long as_ll(const Rational& v, const std::string& what) {
  if (!is_integer(v)) throw EvalError(what + " is not integral");
  return numerator(v).convert_to<long long>();
}

class ProgramBuilder {
 public:
  ProgramBuilder(const Kernel& k, const Env& b) : k_(k), b_(b), types_(infer_types(k)) {}

  void build() {
    for (const auto& s : k_.statements) {
      if (s.is_barrier) {
        std::vector<std::string> seq;
        for (const auto& i : k_.ordered_within(s))
          if (k_.is_sequential(i)) seq.push_back(i);
        barrier_nests_.push_back(nest_of(seq));
        continue;
      }
      const std::vector<std::string> order = k_.ordered_within(s);
      const int n = nest_of(order);
      if (!s.lhs.is_scalar()) add_site(s, s.lhs, Direction::store, {}, n, order);
      walk(s, s.rhs, n, order, {});
    }
  }

  OracleCounts fold(const std::vector<int64_t>& points, const std::vector<int64_t>& pop) const {
    OracleCounts o;
    for (const auto& [key, nest] : op_incs_) o.ops[key] += points[size_t(nest)];
    for (const auto& x : sites_) {
      o.access_counts[x.key] += points[size_t(x.site.nest)];
      o.access_gran[x.key] = x.gran;
    }
    for (const auto& [ga, bm] : group_bitmaps_) o.access_footprints[ga.first] += pop[size_t(bm)];
    for (const auto& [a, bm] : array_bitmaps_) o.footprints[a] = pop[size_t(bm)];
    for (int n : barrier_nests_) o.barrier_local += points[size_t(n)];
    std::map<int, std::string> group;
    bool has_local = false;
    for (const auto& [iname, tag] : k_.iname_tags) {
      if (tag.kind == InameTag::Kind::group) group[tag.axis] = iname;
      if (tag.kind == InameTag::Kind::local) has_local = true;
    }
    if (!group.empty() || k_.single_work_item) {
      long long g = 1;
      for (const auto& [axis, iname] : group) {
        const Bound& bd = k_.domain.bound(iname);
        g *= as_ll(bd.hi.eval(b_), "bound") - as_ll(bd.lo.eval(b_), "bound") + 1;
      }
      o.group_launch = g;
      o.has_group_launch = true;
    } else if (has_local) {
      o.has_group_launch = true;
    }
    return o;
  }

  ps_enum_program program() {
    flat_sites_.clear();
    for (int n = 0; n < int(nests_.size()); ++n)
      for (const auto& x : sites_)
        if (x.site.nest == n) flat_sites_.push_back(x.site);
    ps_enum_program p{};
    p.n_nests = int(nests_.size());
    p.nests = nests_.data();
    p.n_sites = int(flat_sites_.size());
    p.sites = flat_sites_.data();
    p.n_bitmaps = int(bitmap_bits_.size());
    p.bitmap_bits = bitmap_bits_.data();
    return p;
  }

 private:
  struct SiteInfo {
    ps_enum_site site;
    std::string key, gran;
  };

  // coefficients of an affine expression over the nest levels (+ constant)
  void coefs(const AffineExpr& e, const std::vector<std::string>& levels, int64_t* out) const {
    Env env = b_;
    for (const auto& l : levels) env[l] = 0;
    const long long c0 = as_ll(e.eval(env), "affine expression " + e.str());
    for (int d = 0; d <= PS_ENUM_MAXD; ++d) out[d] = 0;
    out[PS_ENUM_MAXD] = c0;
    for (size_t d = 0; d < levels.size(); ++d) {
      env[levels[d]] = 1;
      out[d] = as_ll(e.eval(env), "affine expression " + e.str()) - c0;
      env[levels[d]] = 0;
    }
  }

  int nest_of(const std::vector<std::string>& levels) {
    auto it = nest_ids_.find(levels);
    if (it != nest_ids_.end()) return it->second;
    if (levels.size() > PS_ENUM_MAXD) throw EvalError("enumeration nest deeper than PS_ENUM_MAXD");
    ps_enum_nest n{};
    n.depth = int(levels.size());
    for (size_t d = 0; d < levels.size(); ++d) {
      const Bound& bd = k_.domain.bound(levels[d]);
      const std::vector<std::string> outer(levels.begin(), levels.begin() + d);
      coefs(bd.lo, outer, n.lo[d]);
      coefs(bd.hi, outer, n.hi[d]);
      // box: extreme values of the affine bounds over the outer levels' boxes
      long long lo = n.lo[d][PS_ENUM_MAXD], hi = n.hi[d][PS_ENUM_MAXD];
      for (size_t e = 0; e < d; ++e) {
        const long long a = n.box_lo[e], z = n.box_lo[e] + n.box_ext[e] - 1;
        lo += std::min(n.lo[d][e] * a, n.lo[d][e] * z);
        hi += std::max(n.hi[d][e] * a, n.hi[d][e] * z);
      }
      n.box_lo[d] = lo;
      n.box_ext[d] = hi >= lo ? hi - lo + 1 : 0;
    }
    const int id = int(nests_.size());
    nests_.push_back(n);
    nest_ids_[levels] = id;
    return id;
  }

  int bitmap(std::map<std::pair<std::string, std::string>, int>& table,
             const std::pair<std::string, std::string>& key, long long bits) {
    auto it = table.find(key);
    if (it != table.end()) return it->second;
    const int id = int(bitmap_bits_.size());
    bitmap_bits_.push_back(bits);
    table[key] = id;
    return id;
  }

  void add_site(const Statement& s, const Access& a, Direction dir,
                const std::vector<std::string>& binders, int nest,
                const std::vector<std::string>& levels) {
    const ArgDecl& decl = k_.arg(a.array);
    if (decl.space == MemSpace::private_mem) return;
    if (a.subs.size() > PS_ENUM_MAXR) throw EvalError("enumeration: array rank above PS_ENUM_MAXR");
    const NumericPattern p = probe_pattern(k_, s, a, dir, binders, b_);
    SiteInfo x{};
    x.key = p.key();
    x.gran = p.gran;
    x.site.nest = nest;
    x.site.rank = int(a.subs.size());
    long long elems = 1;
    for (size_t q = 0; q < a.subs.size(); ++q) {
      coefs(a.subs[q], levels, x.site.sub[q]);
      x.site.dim[q] = as_ll(decl.shape[q].eval(b_), "array extent");
      elems *= x.site.dim[q];
    }
    x.site.bitmap_group = bitmap(group_bitmaps_, {x.key, a.array}, elems);
    x.site.bitmap_array = bitmap(array_bitmaps_raw_, {a.array, ""}, elems);
    array_bitmaps_[a.array] = x.site.bitmap_array;
    sites_.push_back(x);
  }

  void op(const ExprPtr& e, OpName n, int nest) {
    op_incs_.push_back({OpKind{expr_dtype(e, k_, types_), n}.key(), nest});
  }

  // the CPU enumerator's walk (ps_enumerate.cpp Visitor::walk), recording
  // per-nest op increments and access sites instead of visiting points
  void walk(const Statement& s, const ExprPtr& e, int nest, const std::vector<std::string>& levels,
            const std::vector<std::string>& binders) {
    if (!e) return;
    switch (e->kind) {
      case Expr::Kind::number:
      case Expr::Kind::scalar_ref:
        return;
      case Expr::Kind::access:
        add_site(s, e->access, Direction::load, binders, nest, levels);
        return;
      case Expr::Kind::binary: {
        if (e->op == BinOp::add || e->op == BinOp::sub) {
          auto is_mul = [](const ExprPtr& x) {
            return x->kind == Expr::Kind::binary && x->op == BinOp::mul;
          };
          const ExprPtr* f = is_mul(e->rhs) ? &e->rhs : is_mul(e->lhs) ? &e->lhs : nullptr;
          if (!s.harness) op(e, f ? OpName::madd : OpName::add, nest);
          if (f) {
            walk(s, *f == e->rhs ? e->lhs : e->rhs, nest, levels, binders);
            walk(s, (*f)->lhs, nest, levels, binders);
            walk(s, (*f)->rhs, nest, levels, binders);
          } else {
            walk(s, e->lhs, nest, levels, binders);
            walk(s, e->rhs, nest, levels, binders);
          }
          return;
        }
        if (!s.harness) op(e, e->op == BinOp::mul ? OpName::mul : OpName::div, nest);
        walk(s, e->lhs, nest, levels, binders);
        walk(s, e->rhs, nest, levels, binders);
        return;
      }
      case Expr::Kind::reduction: {
        std::vector<std::string> inner_levels = levels, inner_binders = binders;
        ExprPtr body = e;
        while (body->kind == Expr::Kind::reduction) {
          inner_levels.push_back(body->red_iname);
          inner_binders.push_back(body->red_iname);
          body = body->body;
        }
        const int inner = nest_of(inner_levels);
        if (!s.harness) {
          if (body->kind == Expr::Kind::binary && body->op == BinOp::mul) {
            op(body, OpName::madd, inner);
            walk(s, body->lhs, inner, inner_levels, inner_binders);
            walk(s, body->rhs, inner, inner_levels, inner_binders);
            return;
          }
          op(body, OpName::add, inner);
        }
        walk(s, body, inner, inner_levels, inner_binders);
        return;
      }
    }
  }

  const Kernel& k_;
  Env b_;
  std::map<std::string, Dtype> types_;
  std::vector<ps_enum_nest> nests_;
  std::map<std::vector<std::string>, int> nest_ids_;
  std::vector<SiteInfo> sites_;
  std::vector<ps_enum_site> flat_sites_;
  std::vector<int64_t> bitmap_bits_;
  std::map<std::pair<std::string, std::string>, int> group_bitmaps_, array_bitmaps_raw_;
  std::map<std::string, int> array_bitmaps_;
  std::vector<std::pair<std::string, int>> op_incs_;
  std::vector<int> barrier_nests_;
};

}  // namespace

OracleCounts brute_force_count_gpu(ps_ctx* ctx, const Kernel& k,
                                   const std::map<std::string, long long>& bindings) {
  for (const auto& a : k.assumptions) {
    auto it = bindings.find(a.param);
    if (it == bindings.end()) continue;
    const bool ok =
        a.kind == Assumption::Kind::divisible ? it->second % a.value == 0 : it->second >= a.value;
    if (!ok)
      throw EvalError("binding " + a.param + "=" + std::to_string(it->second) +
                      " violates assumption " + a.str());
  }
  ProgramBuilder b(k, bindings);
  b.build();
  const ps_enum_program p = b.program();
  std::vector<int64_t> points(size_t(p.n_nests)), pop(size_t(p.n_bitmaps));
  if (ps_enum_gpu_run(ctx, &p, points.data(), pop.data()) != 0) throw EvalError(ps_last_error());
  return b.fold(points, pop);
}

}  // namespace perfseer
