// Generator catalog and IR builders (see ps_catalog.hpp). The IR each
// builder emits — inames, tags, statement ids, dependencies, access tags —
// is what the reference generators emit (uipick.cpp:295-664), so counts,
// variant ids and kernel hashes agree; the CUDA realisations in
// csrc/cuda/ execute exactly these IRs.
#include "ps_catalog.hpp"

#include <algorithm>

#include "ps_lang.hpp"

namespace perfseer {

const std::vector<std::string>* Generator::allowable(const std::string& arg) const {
  for (const auto& [name, values] : variant_args)
    if (name == arg) return &values;
  return nullptr;
}

MatchCondition match_condition_from_str(const std::string& s) {
  if (s == "identical") return MatchCondition::identical;
  if (s == "subset") return MatchCondition::subset_of_user;
  if (s == "superset") return MatchCondition::superset_of_user;
  if (s == "intersect") return MatchCondition::intersect;
  throw SemanticError("unknown match condition '" + s + "'");
}

FilterTagSet FilterTagSet::parse(const std::vector<std::string>& tags) {
  FilterTagSet f;
  for (const auto& t : tags) {
    if (t.empty()) continue;
    const size_t colon = t.find(':');
    if (colon == std::string::npos) {
      f.generator_tags.insert(t);
      continue;
    }
    std::vector<std::string> values(1);
    for (char c : t.substr(colon + 1)) {
      if (c == ',')
        values.emplace_back();
      else
        values.back().push_back(c);
    }
    for (const auto& v : values)
      if (v.empty()) throw SemanticError("empty value in variant tag '" + t + "'");
    f.variant_tags[t.substr(0, colon)] = std::move(values);
  }
  return f;
}

bool generator_matches(const Generator& g, const FilterTagSet& tags, MatchCondition cond) {
  const auto& user = tags.generator_tags;
  auto contains = [](const std::set<std::string>& big, const std::set<std::string>& small) {
    return std::includes(big.begin(), big.end(), small.begin(), small.end());
  };
  switch (cond) {
    case MatchCondition::identical: return g.tags == user;
    case MatchCondition::subset_of_user: return contains(user, g.tags);
    case MatchCondition::superset_of_user: return contains(g.tags, user);
    case MatchCondition::intersect:
      return std::any_of(g.tags.begin(), g.tags.end(), [&](const std::string& t) { return user.count(t) > 0; });
  }
  return false;
}

std::vector<GeneratedKernel> KernelCollection::generate(const FilterTagSet& tags,
                                                        MatchCondition cond) const {
  std::vector<GeneratedKernel> out;
  for (const auto& g : gens_) {
    if (!generator_matches(g, tags, cond)) continue;
    for (const auto& kv : tags.variant_tags)
      if (!g.allowable(kv.first))
        throw SemanticError("variant tag argument '" + kv.first + "' is unknown to matched generator '" +
                            g.id + "'");
    // Restrict each argument to the user's values, keeping allowable order.
    std::vector<std::pair<std::string, std::vector<std::string>>> axes;
    for (const auto& [arg, allowed] : g.variant_args) {
      auto user = tags.variant_tags.find(arg);
      if (user == tags.variant_tags.end()) {
        axes.emplace_back(arg, allowed);
        continue;
      }
      std::vector<std::string> kept;
      for (const auto& v : allowed)
        if (std::find(user->second.begin(), user->second.end(), v) != user->second.end()) kept.push_back(v);
      if (kept.empty())
        throw SemanticError("variant tag empties allowable set of argument '" + arg + "' on generator '" +
                            g.id + "'");
      axes.emplace_back(arg, std::move(kept));
    }
    // Cartesian product, first argument slowest (odometer order).
    std::vector<size_t> digit(axes.size(), 0);
    for (bool more = true; more;) {
      ArgMap a;
      for (size_t i = 0; i < axes.size(); ++i) a[axes[i].first] = axes[i].second[digit[i]];
      out.push_back(g.create(a));
      more = false;
      for (size_t i = axes.size(); i-- > 0;) {
        if (++digit[i] < axes[i].second.size()) {
          more = true;
          break;
        }
        digit[i] = 0;
      }
    }
  }
  return out;
}

std::string variant_id(const std::string& generator, const ArgMap& args) {
  std::string id = generator;
  for (const auto& [k, v] : args) id += "__" + k + "-" + v;
  return id;
}

// ---------------------------------------------------------------------------
// Builder helpers

namespace {

long long int_arg(const ArgMap& a, const std::string& k) {
  auto it = a.find(k);
  if (it == a.end()) throw SemanticError("missing generator argument '" + k + "'");
  try {
    size_t used = 0;
    long long v = std::stoll(it->second, &used);
    if (used != it->second.size()) throw std::invalid_argument(k);
    return v;
  } catch (const std::exception&) {
    throw SemanticError("argument '" + k + "' is not an integer: " + it->second);
  }
}

const std::string& str_arg(const ArgMap& a, const std::string& k) {
  auto it = a.find(k);
  if (it == a.end()) throw SemanticError("missing generator argument '" + k + "'");
  return it->second;
}

bool bool_arg(const ArgMap& a, const std::string& k) {
  const std::string& v = str_arg(a, k);
  if (v == "True" || v == "true" || v == "1") return true;
  if (v == "False" || v == "false" || v == "0") return false;
  throw SemanticError("argument '" + k + "' is not a boolean: " + v);
}

AffineExpr C(long long v) { return AffineExpr::constant(v); }
AffineExpr I(const std::string& n) { return AffineExpr::index(n); }
AffineExpr P(const std::string& n) { return AffineExpr::param(n); }
AffineExpr times(long long c, const AffineExpr& e) { return e.scaled(Rational(c)); }

// Exact literal v on a 1/1024 grid, floating unless the dtype is int32.
ExprPtr literal(double v, Dtype t) {
  return Expr::make_number(Rational(static_cast<long long>(v * 1024), 1024), t != Dtype::int32);
}
ExprPtr ld(const std::string& a, std::vector<AffineExpr> subs, const std::string& tag = "") {
  return Expr::make_access(Access{a, tag, std::move(subs)});
}
ExprPtr var(const std::string& n) { return Expr::make_scalar(n); }
ExprPtr bin(BinOp o, ExprPtr l, ExprPtr r) { return Expr::make_binary(o, std::move(l), std::move(r)); }

class Builder {
 public:
  void loop(const std::string& n, const AffineExpr& lo, const AffineExpr& hi, InameTag t = InameTag::seq()) {
    k_.domain.inames.push_back(n);
    k_.domain.bounds[n] = Bound{lo, hi};
    if (t.is_parallel()) k_.iname_tags[n] = t;
  }
  void param(const std::string& n) { k_.domain.parameters.insert(n); }
  void assume(Assumption::Kind kind, const std::string& p, long long v) {
    k_.assumptions.push_back(Assumption{kind, p, v});
  }
  void array(const std::string& n, Dtype t, std::vector<AffineExpr> shape, MemSpace sp) {
    k_.args.push_back(ArgDecl{n, t, std::move(shape), sp});
  }
  void assign(const std::string& id, Access lhs, ExprPtr rhs, std::set<std::string> within,
              std::set<std::string> deps = {}) {
    Statement s;
    s.id = id;
    s.lhs = std::move(lhs);
    s.rhs = std::move(rhs);
    s.within = std::move(within);
    s.depends_on = std::move(deps);
    k_.statements.push_back(std::move(s));
  }
  void barrier(const std::string& id, std::set<std::string> within, std::set<std::string> deps = {}) {
    Statement s;
    s.id = id;
    s.is_barrier = true;
    s.within = std::move(within);
    s.depends_on = std::move(deps);
    k_.statements.push_back(std::move(s));
  }
  GeneratedKernel done(const std::string& gen, const ArgMap& args, std::map<std::string, long long> b) {
    validate(k_);
    GeneratedKernel g;
    g.id = variant_id(gen, args);
    k_.name = g.id;
    g.kernel = k_;
    g.bindings = std::move(b);
    g.geometry = launch_geometry(g.kernel);
    g.generator = gen;
    g.args = args;
    return g;
  }
  Kernel& kernel() { return k_; }

 private:
  Kernel k_;
};

GeneratedKernel wrap(const std::string& gen, const ArgMap& args, Kernel k,
                     std::map<std::string, long long> bindings) {
  GeneratedKernel g;
  g.id = variant_id(gen, args);
  k.name = g.id;
  g.kernel = std::move(k);
  g.bindings = std::move(bindings);
  g.geometry = launch_geometry(g.kernel);
  g.generator = gen;
  g.args = args;
  return g;
}

// 1-D array of E elements tiled by (L0, L1) work-groups with lid strides
// (s0, s1): global index s0 lx + s1 ly + s0 L0 gx + s1 L1 gy.
struct Tiling {
  long long E, L0, L1, s0, s1, G0, G1;

  explicit Tiling(const ArgMap& a)
      : E(int_arg(a, "nelements")), L0(int_arg(a, "lsize_0")), L1(int_arg(a, "lsize_1")),
        s0(int_arg(a, "lid_stride_0")), s1(int_arg(a, "lid_stride_1")) {
    if (E < 1 || L0 < 1 || L1 < 1 || s0 < 1 || s1 < 1)
      throw SemanticError("pattern layout arguments must be positive");
    if (s1 % (s0 * L0)) throw SemanticError("lid_stride_1 must be a multiple of lid_stride_0*lsize_0");
    if (E % (s1 * L1)) throw SemanticError("nelements must be a multiple of lid_stride_1*lsize_1");
    G0 = s1 / (s0 * L0);
    G1 = E / (s1 * L1);
  }
  void loops(Builder& b) const {
    b.loop("gy", C(0), C(G1 - 1), InameTag::group(1));
    b.loop("gx", C(0), C(G0 - 1), InameTag::group(0));
    b.loop("ly", C(0), C(L1 - 1), InameTag::local(1));
    b.loop("lx", C(0), C(L0 - 1), InameTag::local(0));
  }
  static std::set<std::string> par() { return {"gy", "gx", "ly", "lx"}; }
  static std::set<std::string> par_t() { return {"gy", "gx", "ly", "lx", "t"}; }
  AffineExpr global() const {
    return times(s0, I("lx")) + times(s1, I("ly")) + times(s0 * L0, I("gx")) + times(s1 * L1, I("gy"));
  }
  AffineExpr local() const { return I("lx") + times(L0, I("ly")); }
};

Dtype dtype_arg(const ArgMap& a) { return dtype_from_str(str_arg(a, "dtype")); }

void retag(Kernel& k, const std::string& array, const std::string& tag) {
  int hits = 0;
  std::function<ExprPtr(const ExprPtr&)> re = [&](const ExprPtr& e) -> ExprPtr {
    if (!e) return e;
    if (e->kind == Expr::Kind::access) {
      if (e->access.array != array) return e;
      ++hits;
      Access a = e->access;
      a.tag = tag;
      return Expr::make_access(std::move(a));
    }
    if (e->kind == Expr::Kind::binary) return Expr::make_binary(e->op, re(e->lhs), re(e->rhs));
    if (e->kind == Expr::Kind::reduction) return Expr::make_reduction(e->red_iname, re(e->body));
    return e;
  };
  for (auto& s : k.statements) {
    if (s.is_barrier) continue;
    if (s.lhs.array == array) {
      s.lhs.tag = tag;
      ++hits;
    }
    s.rhs = re(s.rhs);
  }
  if (hits != 1)
    throw SemanticError("tag_access expected exactly one access to '" + array + "', found " +
                        std::to_string(hits));
}

}  // namespace

// ---------------------------------------------------------------------------
// Microbenchmarks

GeneratedKernel make_gmem_pattern(const ArgMap& args) {
  const Tiling t(args);
  const Dtype dt = dtype_arg(args);
  const long long k = int_arg(args, "n_input_arrays");
  if (k < 1) throw SemanticError("n_input_arrays must be >= 1");
  Builder b;
  t.loops(b);
  for (long long i = 0; i < k; ++i) b.array("in" + std::to_string(i), dt, {C(t.E)}, MemSpace::global);
  b.array("result", dt, {C(t.E)}, MemSpace::global);
  ExprPtr sum = ld("in0", {t.global()});
  for (long long i = 1; i < k; ++i) sum = bin(BinOp::add, sum, ld("in" + std::to_string(i), {t.global()}));
  b.assign("store", Access{"result", "", {t.global()}}, sum, Tiling::par());
  return b.done("gmem_pattern", args, {});
}

GeneratedKernel make_flops_pattern(const std::string& op, const ArgMap& args) {
  const Tiling t(args);
  const Dtype dt = dtype_arg(args);
  const long long m = int_arg(args, "m");
  if (m < 1) throw SemanticError("flops iteration count must be >= 1");
  if (op != "add" && op != "mul" && op != "madd") throw SemanticError("unknown flops op '" + op + "'");
  Builder b;
  t.loops(b);
  b.loop("t", C(0), C(m - 1));
  b.array("result", dt, {C(t.E)}, MemSpace::global);
  for (int j = 0; j < 32; ++j) b.array("v" + std::to_string(j), dt, {}, MemSpace::private_mem);
  b.array("r", dt, {}, MemSpace::private_mem);
  auto v = [](int j) { return "v" + std::to_string(j); };
  for (int j = 0; j < 32; ++j)
    b.assign("init_" + std::to_string(j), Access{v(j), "", {}}, literal(0.5 + 0.015625 * j, dt), Tiling::par());
  // SHOC order: update i writes v[i%32] from v[(i+27)%32] and v[(i+21)%32];
  // the nearest dependency is 5 statements back.
  std::string prev = "init_31";
  for (int i = 0; i < 64 * 32; ++i) {
    const int j = i % 32;
    ExprPtr a = var(v((j + 27) % 32)), c = var(v((j + 21) % 32));
    ExprPtr rhs = op == "add" ? bin(BinOp::add, a, c)
                  : op == "mul" ? bin(BinOp::mul, a, c)
                                : bin(BinOp::add, bin(BinOp::mul, a, c), var(v(j)));
    const std::string id = "upd_" + std::to_string(i);
    b.assign(id, Access{v(j), "", {}}, rhs, Tiling::par_t(), {prev});
    prev = id;
  }
  ExprPtr sum = var("v0");
  for (int j = 1; j < 32; ++j) sum = bin(BinOp::add, sum, var(v(j)));
  b.assign("reduce", Access{"r", "", {}}, sum, Tiling::par(), {prev});
  b.assign("store", Access{"result", "", {t.global()}}, var("r"), Tiling::par(), {"reduce"});
  return b.done("flops_" + op + "_pattern", args, {});
}

GeneratedKernel make_lmem_shuffle(const ArgMap& args) {
  const Tiling t(args);
  const Dtype dt = dtype_arg(args);
  const long long m = int_arg(args, "m");
  if (m < 0) throw SemanticError("lmem iteration count must be >= 0");
  Builder b;
  t.loops(b);
  b.loop("t", C(0), C(m - 1));
  b.array("locbuf_a", dt, {C(t.L0 * t.L1)}, MemSpace::local);
  b.array("locbuf_b", dt, {C(t.L0 * t.L1)}, MemSpace::local);
  b.array("result", dt, {C(t.E)}, MemSpace::global);
  b.assign("init", Access{"locbuf_a", "", {t.local()}}, literal(1.0, dt), Tiling::par());
  b.assign("shuffle", Access{"locbuf_b", "", {t.local()}}, ld("locbuf_a", {t.local()}), Tiling::par_t(), {"init"});
  b.assign("store", Access{"result", "", {t.global()}}, ld("locbuf_b", {t.local()}), Tiling::par(), {"shuffle"});
  return b.done("lmem_shuffle", args, {});
}

GeneratedKernel make_barrier_knl(const ArgMap& args) {
  const Tiling t(args);
  const long long m = int_arg(args, "m");
  if (m < 0) throw SemanticError("barrier count must be >= 0");
  Builder b;
  t.loops(b);
  b.loop("t", C(0), C(m - 1));
  b.array("result", Dtype::float32, {C(t.E)}, MemSpace::global);
  b.barrier("bar", Tiling::par_t());
  b.assign("store", Access{"result", "", {t.global()}}, literal(1.0, Dtype::float32), Tiling::par(), {"bar"});
  return b.done("barrier_knl", args, {});
}

GeneratedKernel make_empty_knl(const ArgMap& args) {
  const long long groups = int_arg(args, "num_groups");
  if (groups < 1) throw SemanticError("num_groups must be >= 1");
  Builder b;
  b.loop("g0", C(0), C(groups - 1), InameTag::group(0));
  b.loop("l0", C(0), C(255), InameTag::local(0));
  return b.done("empty_knl", args, {});
}

GeneratedKernel make_overlap_knl(const ArgMap& args) {
  const Tiling t(args);
  const Dtype dt = dtype_arg(args);
  const long long m = int_arg(args, "m");
  if (m < 0) throw SemanticError("overlap ratio m must be >= 0");
  Builder b;
  t.loops(b);
  b.loop("t", C(0), C(m - 1));
  b.array("in0", dt, {C(t.E)}, MemSpace::global);
  b.array("result", dt, {C(t.E)}, MemSpace::global);
  b.array("locbuf_a", dt, {C(t.L0 * t.L1)}, MemSpace::local);
  b.array("locbuf_b", dt, {C(t.L0 * t.L1)}, MemSpace::local);
  b.array("tmp", dt, {}, MemSpace::private_mem);
  b.assign("load", Access{"tmp", "", {}}, ld("in0", {t.global()}), Tiling::par());
  b.assign("shuffle", Access{"locbuf_b", "", {t.local()}}, ld("locbuf_a", {t.local()}), Tiling::par_t(), {"load"});
  b.assign("store", Access{"result", "", {t.global()}}, var("tmp"), Tiling::par(), {"shuffle"});
  return b.done("overlap_knl", args, {});
}

// ---------------------------------------------------------------------------
// Applications: square matmul and five-point FD

GeneratedKernel make_matmul_sq(const ArgMap& args) {
  const Dtype dt = dtype_arg(args);
  const bool pf = bool_arg(args, "prefetch");
  const long long n = int_arg(args, "n"), l0 = int_arg(args, "lsize_0"), l1 = int_arg(args, "lsize_1");
  if (!bool_arg(args, "groups_fit"))
    throw SemanticError("matmul_sq requires groups_fit:True (conditionals are not generated)");
  if (l0 != l1) throw SemanticError("matmul_sq uses square tiles (lsize_0 == lsize_1)");
  const long long T = l0;
  if (n % T != 0 || n < T) throw SemanticError("matmul_sq requires n to be a multiple of the tile size");
  const std::string d = dtype_str(dt);

  if (!pf) {
    Kernel k = make_kernel("{[i,j,k]: 0<=i,j,k<n}", {"c[i,j] = sum(k, a[i,k]*b[k,j])"},
                           {{"a", dt, {"n", "n"}}, {"b", dt, {"n", "n"}}, {"c", dt, {"n", "n"}}});
    retag(k, "a", "mm-noPF-a");
    retag(k, "b", "mm-noPF-b");
    k = assume_lower_bound(assume_divisible(k, "n", T), "n", T);
    k = split_iname(split_iname(k, "i", T), "j", T);
    k = tag_inames(k, {{"i_out", InameTag::group(1)}, {"i_in", InameTag::local(1)},
                       {"j_out", InameTag::group(0)}, {"j_in", InameTag::local(0)}});
    return wrap("matmul_sq", args, std::move(k), {{"n", n}});
  }

  Builder b;
  b.param("n");
  const AffineExpr last_tile = P("n").scaled(Rational(1, T)) - C(1);
  b.loop("i_out", C(0), last_tile, InameTag::group(1));
  b.loop("i_in", C(0), C(T - 1), InameTag::local(1));
  b.loop("j_out", C(0), last_tile, InameTag::group(0));
  b.loop("j_in", C(0), C(T - 1), InameTag::local(0));
  b.loop("k_out", C(0), last_tile);
  b.loop("k_in", C(0), C(T - 1));
  b.assume(Assumption::Kind::divisible, "n", T);
  b.assume(Assumption::Kind::lower_bound, "n", T);
  for (const char* a : {"a", "b", "c"}) b.array(a, dt, {P("n"), P("n")}, MemSpace::global);
  b.array("a_fetch", dt, {C(T), C(T)}, MemSpace::local);
  b.array("b_fetch", dt, {C(T), C(T)}, MemSpace::local);
  b.array("acc", dt, {}, MemSpace::private_mem);
  const std::set<std::string> par{"i_out", "i_in", "j_out", "j_in"};
  std::set<std::string> tile = par, inner = par;
  tile.insert("k_out");
  inner.insert({"k_out", "k_in"});
  const AffineExpr row = times(T, I("i_out")) + I("i_in"), col = times(T, I("j_out")) + I("j_in");
  b.assign("acc_init", Access{"acc", "", {}}, literal(0.0, dt), par);
  b.barrier("bar_pre", tile, {"acc_init"});
  b.assign("fetch_a", Access{"a_fetch", "", {I("i_in"), I("j_in")}},
           ld("a", {row, times(T, I("k_out")) + I("j_in")}, "mm-PF-a"), tile, {"bar_pre"});
  b.assign("fetch_b", Access{"b_fetch", "", {I("i_in"), I("j_in")}},
           ld("b", {times(T, I("k_out")) + I("i_in"), col}, "mm-PF-b"), tile, {"bar_pre"});
  b.barrier("bar_post", tile, {"fetch_a", "fetch_b"});
  b.assign("update", Access{"acc", "", {}},
           bin(BinOp::add, var("acc"),
               bin(BinOp::mul, ld("a_fetch", {I("i_in"), I("k_in")}), ld("b_fetch", {I("k_in"), I("j_in")}))),
           inner, {"bar_post"});
  b.assign("store", Access{"c", "", {row, col}}, var("acc"), par, {"update"});
  (void)d;
  return b.done("matmul_sq", args, {{"n", n}});
}

GeneratedKernel make_matmul_sq_rm(const ArgMap& args) {
  const std::string keep = str_arg(args, "keep");
  const bool pf = bool_arg(args, "prefetch");
  ArgMap base_args = args;
  base_args.erase("keep");
  GeneratedKernel base = make_matmul_sq(base_args);
  const std::string v = pf ? "PF" : "noPF";
  if (keep != "a" && keep != "b") throw SemanticError("matmul_sq_rm keep must be 'a' or 'b'");
  Kernel k = remove_work(base.kernel, {"c"}, {"mm-" + v + "-" + (keep == "a" ? "b" : "a")});
  return wrap("matmul_sq_rm", args, std::move(k), base.bindings);
}

GeneratedKernel make_fd_stencil(const ArgMap& args) {
  const Dtype dt = dtype_arg(args);
  const std::string tile = str_arg(args, "tile");
  const long long n = int_arg(args, "n");
  long long T;
  if (tile == "16x16")
    T = 16;
  else if (tile == "18x18")
    T = 18;
  else
    throw SemanticError("fd tile must be 16x16 or 18x18");
  const long long In = T - 2;  // interior points per tile side
  if (n % In != 0 || n < In)
    throw SemanticError("finite_diff requires n to be a multiple of " + std::to_string(In));
  Builder b;
  b.param("n");
  const AffineExpr last = P("n").scaled(Rational(1, In)) - C(1);
  b.loop("i_out", C(0), last, InameTag::group(1));
  b.loop("j_out", C(0), last, InameTag::group(0));
  b.loop("l1", C(0), C(T - 1), InameTag::local(1));
  b.loop("l0", C(0), C(T - 1), InameTag::local(0));
  b.loop("c1", C(0), C(In - 1));
  b.loop("c0", C(0), C(In - 1));
  b.assume(Assumption::Kind::divisible, "n", In);
  b.assume(Assumption::Kind::lower_bound, "n", In);
  const AffineExpr w = P("n") + C(2);
  b.array("u", dt, {w, w}, MemSpace::global);
  b.array("res", dt, {P("n"), P("n")}, MemSpace::global);
  b.array("u_fetch", dt, {C(T), C(T)}, MemSpace::local);
  b.assign("fetch", Access{"u_fetch", "", {I("l1"), I("l0")}},
           ld("u", {times(In, I("i_out")) + I("l1"), times(In, I("j_out")) + I("l0")}, "fd-" + tile + "-u"),
           {"i_out", "j_out", "l1", "l0"});
  b.barrier("bar", {"i_out", "j_out"}, {"fetch"});
  auto uf = [](long long dr, long long dc) { return ld("u_fetch", {I("c1") + C(dr), I("c0") + C(dc)}); };
  ExprPtr rhs = bin(BinOp::add, uf(0, 1), uf(1, 0));
  rhs = bin(BinOp::sub, rhs, bin(BinOp::mul, literal(4.0, dt), uf(1, 1)));
  rhs = bin(BinOp::add, rhs, uf(1, 2));
  rhs = bin(BinOp::add, rhs, uf(2, 1));
  b.assign("compute",
           Access{"res", "fd-" + tile + "-res", {times(In, I("i_out")) + I("c1"), times(In, I("j_out")) + I("c0")}},
           rhs, {"i_out", "j_out", "c1", "c0"}, {"bar"});
  return b.done("finite_diff", args, {{"n", n}});
}

GeneratedKernel make_fd_stencil_rm(const ArgMap& args) {
  const std::string keep = str_arg(args, "keep");
  ArgMap base_args = args;
  base_args.erase("keep");
  GeneratedKernel base = make_fd_stencil(base_args);
  if (keep != "u" && keep != "res") throw SemanticError("finite_diff_rm keep must be 'u' or 'res'");
  Kernel k = remove_work(base.kernel, {keep == "u" ? "res" : "u"});
  return wrap("finite_diff_rm", args, std::move(k), base.bindings);
}

// ---------------------------------------------------------------------------
// DG differentiation: res[m,k,i] = sum_j dm[m,i,j] u[k,j]
// with i split by 16 (g.1/l.1) and k split by 16 (g.0/l.0); nmatrices fixed
// (fix_parameters), nelements and nunit_nodes symbolic (so predictions can
// sweep them). Tags follow the paper's Fig. 5 names with '/' dropped.

namespace {

struct DgShape {
  std::string variant;
  long long nel, np, nmat;
  explicit DgShape(const ArgMap& a)
      : variant(str_arg(a, "variant")), nel(int_arg(a, "nelements")), np(int_arg(a, "nunit_nodes")),
        nmat(int_arg(a, "nmatrices")) {
    if (variant != "noPF" && variant != "uPF" && variant != "dmPF" && variant != "dmPFtrans")
      throw SemanticError("dg_diff variant must be noPF, uPF, dmPF or dmPFtrans");
    if (nel < 16 || nel % 16) throw SemanticError("dg_diff requires nelements to be a multiple of 16");
    if (np < 16 || np % 16) throw SemanticError("dg_diff requires nunit_nodes to be a multiple of 16 (pad)");
    if (nmat < 1 || nmat > 4) throw SemanticError("dg_diff supports 1..4 matrices");
  }
};

}  // namespace

GeneratedKernel make_dg_diff(const ArgMap& args) {
  const DgShape s(args);
  if (str_arg(args, "dtype") != "float32") throw SemanticError("dg_diff is float32");
  const Dtype dt = Dtype::float32;
  const bool trans = s.variant == "dmPFtrans";
  const bool upf = s.variant == "uPF";
  Builder b;
  b.param("nelements");
  b.param("nunit_nodes");
  const AffineExpr kt = P("nelements").scaled(Rational(1, 16)) - C(1);
  const AffineExpr it = P("nunit_nodes").scaled(Rational(1, 16)) - C(1);
  // Loop order follows each variant's schedule (prioritize_loops): noPF and
  // dmPF keep m outermost; uPF sweeps j_out, j_in with m innermost.
  if (!upf) b.loop("m", C(0), C(s.nmat - 1));
  b.loop("k_out", C(0), kt, InameTag::group(0));
  b.loop("k_in", C(0), C(15), InameTag::local(0));
  b.loop("i_out", C(0), it, InameTag::group(1));
  b.loop("i_in", C(0), C(15), InameTag::local(1));
  if (s.variant == "noPF") {
    b.loop("j", C(0), P("nunit_nodes") - C(1));
  } else {
    b.loop("j_out", C(0), it);
    b.loop("j_in", C(0), C(15));
  }
  if (upf) b.loop("m", C(0), C(s.nmat - 1));
  for (const char* p : {"nelements", "nunit_nodes"}) {
    b.assume(Assumption::Kind::divisible, p, 16);
    b.assume(Assumption::Kind::lower_bound, p, 16);
  }
  const AffineExpr NP = P("nunit_nodes"), NE = P("nelements");
  b.array("diff_mat", dt, {C(s.nmat), NP, NP}, MemSpace::global);
  if (trans) {
    b.array("u", dt, {NP, NE}, MemSpace::global);
    b.array("res", dt, {C(s.nmat), NP, NE}, MemSpace::global);
  } else {
    b.array("u", dt, {NE, NP}, MemSpace::global);
    b.array("res", dt, {C(s.nmat), NE, NP}, MemSpace::global);
  }
  const AffineExpr k = times(16, I("k_out")) + I("k_in"), i = times(16, I("i_out")) + I("i_in");
  const std::set<std::string> par{"k_out", "k_in", "i_out", "i_in"};
  auto with = [&](std::initializer_list<const char*> extra) {
    std::set<std::string> w = par;
    for (const char* e : extra) w.insert(e);
    return w;
  };
  auto res_access = [&](const std::string& tag) {
    return trans ? Access{"res", tag, {I("m"), i, k}} : Access{"res", tag, {I("m"), k, i}};
  };

  if (s.variant == "noPF") {
    b.assign("compute", res_access("dg-noPF-res"),
             Expr::make_reduction("j", bin(BinOp::mul, ld("diff_mat", {I("m"), i, I("j")}, "dg-uPFnoPF-dm"),
                                           ld("u", {k, I("j")}, "dg-noPF-u"))),
             with({"m"}));
  } else if (upf) {
    const AffineExpr j = times(16, I("j_out")) + I("j_in");
    b.array("u_fetch", dt, {C(16), C(16)}, MemSpace::local);
    b.array("acc", dt, {C(s.nmat)}, MemSpace::private_mem);
    b.assign("acc_init", Access{"acc", "", {I("m")}}, literal(0.0, dt), with({"m"}));
    b.barrier("bar_pre", with({"j_out"}), {"acc_init"});
    b.assign("fetch", Access{"u_fetch", "", {I("i_in"), I("k_in")}},
             ld("u", {times(16, I("k_out")) + I("i_in"), times(16, I("j_out")) + I("k_in")}, "dg-uPF-u"),
             with({"j_out"}), {"bar_pre"});
    b.barrier("bar_post", with({"j_out"}), {"fetch"});
    // u_fetch[k_in, j_in] is invariant in the innermost m loop: it is read
    // once per (j_out, j_in) into a private value and reused for the nmat
    // accumulators (as any compiler hoists it, and as the sm_100a kernel does),
    // so local loads count Np per work-item, not nmat * Np.
    b.array("u_val", dt, {}, MemSpace::private_mem);
    b.assign("u_read", Access{"u_val", "", {}}, ld("u_fetch", {I("k_in"), I("j_in")}),
             with({"j_out", "j_in"}), {"bar_post"});
    b.assign("update", Access{"acc", "", {I("m")}},
             bin(BinOp::add, ld("acc", {I("m")}),
                 bin(BinOp::mul, ld("diff_mat", {I("m"), i, j}, "dg-uPFnoPF-dm"), var("u_val"))),
             with({"j_out", "j_in", "m"}), {"u_read"});
    b.assign("store", res_access("dg-uPF-res"), ld("acc", {I("m")}), with({"m"}), {"update"});
  } else {
    const AffineExpr j = times(16, I("j_out")) + I("j_in");
    const std::string v = trans ? "dmPFtrans" : "dmPF";
    b.array("dm_fetch", dt, {C(16), C(16)}, MemSpace::local);
    b.array("acc", dt, {}, MemSpace::private_mem);
    b.assign("acc_init", Access{"acc", "", {}}, literal(0.0, dt), with({"m"}));
    b.barrier("bar_pre", with({"m", "j_out"}), {"acc_init"});
    b.assign("fetch", Access{"dm_fetch", "", {I("i_in"), I("k_in")}},
             ld("diff_mat", {I("m"), i, times(16, I("j_out")) + I("k_in")}, "dg-dmPF-dm"),
             with({"m", "j_out"}), {"bar_pre"});
    b.barrier("bar_post", with({"m", "j_out"}), {"fetch"});
    b.assign("update", Access{"acc", "", {}},
             bin(BinOp::add, var("acc"),
                 bin(BinOp::mul, ld("dm_fetch", {I("i_in"), I("j_in")}),
                     ld("u", trans ? std::vector<AffineExpr>{j, k} : std::vector<AffineExpr>{k, j},
                        "dg-" + v + "-u"))),
             with({"m", "j_out", "j_in"}), {"bar_post"});
    b.assign("store", res_access("dg-" + v + "-res"), var("acc"), with({"m"}), {"update"});
  }
  return b.done("dg_diff", args, {{"nelements", s.nel}, {"nunit_nodes", s.np}});
}

GeneratedKernel make_dg_diff_rm(const ArgMap& args) {
  const std::string keep = str_arg(args, "keep");
  ArgMap base_args = args;
  base_args.erase("keep");
  GeneratedKernel base = make_dg_diff(base_args);
  std::set<std::string> drop;
  if (keep == "u")
    drop = {"diff_mat", "res"};
  else if (keep == "dm")
    drop = {"u", "res"};
  else if (keep == "res")
    drop = {"u", "diff_mat"};
  else
    throw SemanticError("dg_diff_rm keep must be u, dm or res");
  Kernel k = remove_work(base.kernel, drop);
  return wrap("dg_diff_rm", args, std::move(k), base.bindings);
}

// ---------------------------------------------------------------------------
// Catalogs

namespace {

Generator gen(const std::string& id, std::vector<std::pair<std::string, std::vector<std::string>>> vargs,
              std::function<GeneratedKernel(const ArgMap&)> create, std::set<std::string> tags = {}) {
  Generator g;
  g.id = id;
  g.tags = tags.empty() ? std::set<std::string>{id} : std::move(tags);
  g.variant_args = std::move(vargs);
  g.create = std::move(create);
  return g;
}

using VArgs = std::vector<std::pair<std::string, std::vector<std::string>>>;

VArgs pattern_args(const std::vector<std::string>& sizes, std::vector<std::pair<std::string, std::vector<std::string>>> front,
                   bool with_dtype = true, const std::string& lsize = "16",
                   const std::string& s1 = "2048") {
  VArgs v;
  if (with_dtype) v.push_back({"dtype", {"float32"}});
  for (auto& f : front) v.push_back(std::move(f));
  v.push_back({"nelements", sizes});
  v.push_back({"lsize_0", {lsize}});
  v.push_back({"lsize_1", {lsize}});
  v.push_back({"lid_stride_0", {"1"}});
  v.push_back({"lid_stride_1", {s1}});
  return v;
}

}  // namespace

std::vector<Generator> builtin_generators() {
  std::vector<Generator> out;
  const std::vector<std::string> sizes{"524288", "786432", "1048576", "1310720"};
  const std::vector<std::string> iters{"1024", "1152", "1280", "1408"};
  {
    VArgs v{{"dtype", {"float32"}}, {"nelements", sizes}, {"lsize_0", {"16"}}, {"lsize_1", {"16"}},
            {"lid_stride_0", {"1"}}, {"lid_stride_1", {"2048"}}, {"n_input_arrays", {"1", "2"}}};
    out.push_back(gen("gmem_pattern", v, make_gmem_pattern));
  }
  for (const std::string op : {"add", "mul", "madd"})
    out.push_back(gen("flops_" + op + "_pattern", pattern_args(sizes, {{"m", iters}}),
                      [op](const ArgMap& a) { return make_flops_pattern(op, a); }));
  out.push_back(gen("lmem_shuffle", pattern_args(sizes, {{"m", iters}}), make_lmem_shuffle));
  {
    VArgs v{{"m", {"256", "512", "768", "1024"}}, {"nelements", {"524288"}}, {"lsize_0", {"16"}},
            {"lsize_1", {"16"}}, {"lid_stride_0", {"1"}}, {"lid_stride_1", {"2048"}}};
    out.push_back(gen("barrier_knl", v, make_barrier_knl));
  }
  out.push_back(gen("empty_knl", {{"num_groups", {"16", "32", "64", "128", "256", "512"}}}, make_empty_knl));
  {
    std::vector<std::string> ms;
    for (int m = 0; m <= 16; ++m) ms.push_back(std::to_string(m));
    out.push_back(gen("overlap_knl", pattern_args({"524288", "1048576"}, {{"m", ms}}), make_overlap_knl));
  }
  const std::vector<std::string> mm_n{"2048", "2560", "3072", "3584"};
  out.push_back(gen("matmul_sq",
                    {{"dtype", {"float32", "float64"}}, {"prefetch", {"True", "False"}}, {"lsize_0", {"16"}},
                     {"lsize_1", {"16"}}, {"groups_fit", {"True"}}, {"n", mm_n}},
                    make_matmul_sq));
  out.push_back(gen("matmul_sq_rm",
                    {{"dtype", {"float32"}}, {"prefetch", {"True", "False"}}, {"keep", {"a", "b"}},
                     {"lsize_0", {"16"}}, {"lsize_1", {"16"}}, {"groups_fit", {"True"}}, {"n", mm_n}},
                    make_matmul_sq_rm));
  const std::vector<std::string> fd_n{"2240", "2464", "2688", "2912"};
  out.push_back(gen("finite_diff", {{"dtype", {"float32"}}, {"tile", {"16x16", "18x18"}}, {"n", fd_n}},
                    make_fd_stencil));
  out.push_back(gen("finite_diff_rm",
                    {{"dtype", {"float32"}}, {"tile", {"16x16", "18x18"}}, {"keep", {"u", "res"}}, {"n", fd_n}},
                    make_fd_stencil_rm));
  return out;
}

std::vector<Generator> b200_generators() {
  std::vector<Generator> out;
  // HBM streaming: >= 1 GiB per array (L2 is 126 MB).
  const std::vector<std::string> hbm{"268435456", "402653184", "536870912", "671088640"};
  {
    VArgs v{{"dtype", {"float32"}}, {"nelements", hbm}, {"lsize_0", {"16"}}, {"lsize_1", {"16"}},
            {"lid_stride_0", {"1"}}, {"lid_stride_1", {"2048"}}, {"n_input_arrays", {"1", "2"}}};
    out.push_back(gen("gmem_pattern", v, make_gmem_pattern, {"gmem_pattern", "gmem_pattern_16"}));
    // 18x18 work-groups, gid(0) stride 18.
    VArgs v18{{"dtype", {"float32"}}, {"nelements", {"268406784", "402610176", "536813568", "671016960"}},
              {"lsize_0", {"18"}}, {"lsize_1", {"18"}}, {"lid_stride_0", {"1"}}, {"lid_stride_1", {"2304"}},
              {"n_input_arrays", {"1"}}};
    out.push_back(gen("gmem_pattern_18", v18, make_gmem_pattern, {"gmem_pattern", "gmem_pattern_18"}));
  }
  const std::vector<std::string> flop_sizes{"1048576", "2097152"};
  const std::vector<std::string> flop_iters{"64", "128"};
  for (const std::string op : {"add", "mul", "madd"})
    out.push_back(gen("flops_" + op + "_pattern", pattern_args(flop_sizes, {{"m", flop_iters}}),
                      [op](const ArgMap& a) { return make_flops_pattern(op, a); }));
  out.push_back(gen("lmem_shuffle", pattern_args({"1048576", "2097152"}, {{"m", {"512", "1024"}}}),
                    make_lmem_shuffle));
  out.push_back(gen("barrier_knl",
                    {{"m", {"256", "512", "768", "1024"}}, {"nelements", {"2097152"}}, {"lsize_0", {"16"}},
                     {"lsize_1", {"16"}}, {"lid_stride_0", {"1"}}, {"lid_stride_1", {"2048"}}},
                    make_barrier_knl));
  out.push_back(gen("empty_knl", {{"num_groups", {"16", "64", "256", "1024", "4096", "16384"}}}, make_empty_knl));
  {
    std::vector<std::string> ms;
    for (int m = 0; m <= 16; m += 2) ms.push_back(std::to_string(m));
    out.push_back(gen("overlap_knl", pattern_args({"134217728", "268435456"}, {{"m", ms}}), make_overlap_knl));
  }
  // BASELINE.json config 1: matmul n = 512..8192.
  const std::vector<std::string> mm_n{"512", "1024", "2048", "3072", "4096", "6144", "8192"};
  out.push_back(gen("matmul_sq",
                    {{"dtype", {"float32"}}, {"prefetch", {"True", "False"}}, {"lsize_0", {"16"}},
                     {"lsize_1", {"16"}}, {"groups_fit", {"True"}}, {"n", mm_n}},
                    make_matmul_sq));
  out.push_back(gen("matmul_sq_rm",
                    {{"dtype", {"float32"}}, {"prefetch", {"True", "False"}}, {"keep", {"a", "b"}},
                     {"lsize_0", {"16"}}, {"lsize_1", {"16"}}, {"groups_fit", {"True"}},
                     {"n", {"1024", "2048", "4096", "8192"}}},
                    make_matmul_sq_rm));
  // BASELINE.json config 0: grids 1024^2..8192^2 (multiples of lcm(14, 16)).
  // The application sweep adds 1680, 2800, 3360, 5600 and 6272 between the
  // four calibration sizes: the held-out VALIDATION sizes of model selection.
  const std::vector<std::string> fd_n{"1120", "2240", "4480", "8176"};
  const std::vector<std::string> fd_app_n{"1120", "1680", "2240", "2800", "3360",
                                          "4480", "5600", "6272", "8176"};
  out.push_back(gen("finite_diff", {{"dtype", {"float32"}}, {"tile", {"16x16", "18x18"}}, {"n", fd_app_n}},
                    make_fd_stencil));
  out.push_back(gen("finite_diff_rm",
                    {{"dtype", {"float32"}}, {"tile", {"16x16", "18x18"}}, {"keep", {"u", "res"}}, {"n", fd_n}},
                    make_fd_stencil_rm));
  // BASELINE.json config 2: DG, 3-D orders 1-7, 10^4..10^6 elements. Nodes
  // per element (k+1)(k+2)(k+3)/6 = 4, 10, 20, 35, 56, 84, 120 padded to the
  // 16-wide work-group: 16 (orders 1 and 2), 32, 48, 64, 96, 128;
  // Np = 64 is also the paper's own setting.
  const std::vector<std::string> dg_np{"16", "32", "48", "64", "96", "128"};
  out.push_back(gen("dg_diff",
                    {{"dtype", {"float32"}}, {"variant", {"noPF", "uPF", "dmPF", "dmPFtrans"}},
                     {"nmatrices", {"3"}}, {"nunit_nodes", dg_np},
                     {"nelements", {"10000", "100000", "1000000"}}},
                    make_dg_diff));
  out.push_back(gen("dg_diff_rm",
                    {{"dtype", {"float32"}}, {"variant", {"noPF", "uPF", "dmPF", "dmPFtrans"}},
                     {"keep", {"u", "dm", "res"}}, {"nmatrices", {"3"}}, {"nunit_nodes", dg_np},
                     {"nelements", {"100000", "1000000"}}},
                    make_dg_diff_rm));
  return out;
}

GeneratedKernel kernel_from_variant_id(const std::string& id) {
  std::vector<std::string> parts;
  for (size_t pos = 0;;) {
    const size_t next = id.find("__", pos);
    parts.push_back(id.substr(pos, next == std::string::npos ? std::string::npos : next - pos));
    if (next == std::string::npos) break;
    pos = next + 2;
  }
  ArgMap args;
  for (size_t i = 1; i < parts.size(); ++i) {
    const size_t dash = parts[i].find('-');
    if (dash == std::string::npos) throw SemanticError("malformed variant argument '" + parts[i] + "'");
    args[parts[i].substr(0, dash)] = parts[i].substr(dash + 1);
  }
  const std::string& g = parts[0];
  if (g == "gmem_pattern") return make_gmem_pattern(args);
  if (g == "flops_add_pattern") return make_flops_pattern("add", args);
  if (g == "flops_mul_pattern") return make_flops_pattern("mul", args);
  if (g == "flops_madd_pattern") return make_flops_pattern("madd", args);
  if (g == "lmem_shuffle") return make_lmem_shuffle(args);
  if (g == "barrier_knl") return make_barrier_knl(args);
  if (g == "empty_knl") return make_empty_knl(args);
  if (g == "overlap_knl") return make_overlap_knl(args);
  if (g == "matmul_sq") return make_matmul_sq(args);
  if (g == "matmul_sq_rm") return make_matmul_sq_rm(args);
  if (g == "finite_diff") return make_fd_stencil(args);
  if (g == "finite_diff_rm") return make_fd_stencil_rm(args);
  if (g == "dg_diff") return make_dg_diff(args);
  if (g == "dg_diff_rm") return make_dg_diff_rm(args);
  throw SemanticError("unknown generator '" + g + "' in variant id '" + id + "'");
}

}  // namespace perfseer
