// Feature grammar, matching and evaluation (reference behaviour
// features.cpp:41-493; grammar SPEC.md:323-331).
#include "ps_features.hpp"

#include <atomic>
#include <sstream>

#include "ps_executor.hpp"
#include "ps_lang.hpp"

namespace perfseer {

std::string constraint_rel_str(ConstraintRel r) {
  return r == ConstraintRel::lt ? "<" : r == ConstraintRel::gt ? ">" : "";
}

namespace {

std::string constraint_list(const std::vector<StrideConstraint>& cs) {
  std::string s = "{";
  for (size_t i = 0; i < cs.size(); ++i)
    s += (i ? ";" : "") + std::to_string(cs[i].axis) + ":" + constraint_rel_str(cs[i].rel) +
         cs[i].rhs.str();
  return s + "}";
}

bool starts(const std::string& s, const char* prefix) { return s.rfind(prefix, 0) == 0; }

ConstraintRel strip_rel(std::string& s) {
  if (!s.empty() && (s[0] == '<' || s[0] == '>')) {
    ConstraintRel r = s[0] == '<' ? ConstraintRel::lt : ConstraintRel::gt;
    s.erase(0, 1);
    return r;
  }
  return ConstraintRel::eq;
}

std::vector<StrideConstraint> constraint_set(const std::string& body, const std::string& id) {
  std::vector<std::string> parts;
  std::string cur;
  for (char c : body) {
    if (c == ';') {
      parts.push_back(cur);
      cur.clear();
    } else {
      cur.push_back(c);
    }
  }
  if (!cur.empty()) parts.push_back(cur);
  std::vector<StrideConstraint> out;
  std::set<int> axes;
  for (const auto& part : parts) {
    size_t colon = part.find(':');
    if (colon == std::string::npos) throw EvalError("malformed stride constraint '" + part + "' in " + id);
    int axis = 0;
    try {
      axis = std::stoi(part.substr(0, colon));
    } catch (...) {
      throw EvalError("malformed stride axis in '" + part + "' in " + id);
    }
    if (!axes.insert(axis).second)
      throw EvalError("duplicate stride axis " + std::to_string(axis) + " in " + id);
    std::string rest = part.substr(colon + 1);
    ConstraintRel rel = strip_rel(rest);
    if (rest.empty()) throw EvalError("empty stride constraint value in " + id);
    out.push_back(StrideConstraint{axis, rel, parse_affine_params(rest)});
  }
  if (out.empty()) throw EvalError("empty constraint set in " + id);
  return out;
}

FeatureSpec parse_mem_access(const std::string& id, std::string s) {
  FeatureSpec f;
  f.cls = FeatureSpec::Class::mem_access;
  int last_rank = 0;
  auto order = [&](int rank, const char* field) {
    if (rank <= last_rank)
      throw EvalError(std::string("feature field '") + field + "' out of order in " + id);
    last_rank = rank;
  };
  while (!s.empty()) {
    if (s[0] != '_') throw EvalError("malformed feature id: " + id);
    s.erase(0, 1);
    if (starts(s, "tag:")) {
      order(1, "tag");
      f.tag = s.substr(4);
      if (f.tag.empty()) throw EvalError("empty access tag in " + id);
      if (f.tag.find_first_of("_{") != std::string::npos)
        throw EvalError("access tag may not contain '_' or '{': " + id);
      s.clear();
    } else if (starts(s, "global") || starts(s, "local")) {
      order(2, "mem type");
      const bool g = s[0] == 'g';
      f.mem = g ? MemType::global_mem : MemType::local_mem;
      s.erase(0, g ? 6 : 5);
    } else if (starts(s, "float32") || starts(s, "float64") || starts(s, "int32")) {
      order(3, "data type");
      const size_t len = starts(s, "int32") ? 5 : 7;
      f.mem_dtype = dtype_from_str(s.substr(0, len));
      s.erase(0, len);
    } else if (starts(s, "load") || starts(s, "store")) {
      order(4, "direction");
      const bool ld = s[0] == 'l';
      f.dir = ld ? Direction::load : Direction::store;
      s.erase(0, ld ? 4 : 5);
    } else if (starts(s, "lstrides:{") || starts(s, "gstrides:{")) {
      const bool local = s[0] == 'l';
      order(local ? 5 : 6, local ? "lstrides" : "gstrides");
      size_t close = s.find('}');
      if (close == std::string::npos) throw EvalError("unclosed constraint braces in " + id);
      auto cs = constraint_set(s.substr(10, close - 10), id);
      (local ? f.lstride_cons : f.gstride_cons) = std::move(cs);
      s.erase(0, close + 1);
    } else if (starts(s, "afr:")) {
      order(7, "afr");
      std::string body = s.substr(4);
      if (body.find('_') != std::string::npos)
        throw EvalError("feature field after afr is out of order in " + id);
      if (body.empty()) throw EvalError("empty afr constraint in " + id);
      AfrConstraint c;
      c.rel = strip_rel(body);
      c.rhs = parse_affine_params(body);
      f.afr_con = c;
      s.clear();
    } else {
      throw EvalError("unknown or out-of-order feature field near '_" + s + "' in " + id);
    }
  }
  if (!f.tag.empty() && (f.mem || f.mem_dtype || f.dir || !f.lstride_cons.empty() ||
                         !f.gstride_cons.empty() || f.afr_con))
    throw EvalError("tag-based feature carries no other constraints: " + id);
  return f;
}

}  // namespace

std::string FeatureSpec::id() const {
  switch (cls) {
    case Class::op: return "f_op_" + dtype_str(dtype) + "_" + opname_str(op);
    case Class::sync: return "f_sync_" + synckind_str(sync);
    case Class::thread_groups: return "f_thread_groups";
    case Class::wall_time: return "f_exec_wall_time_" + executor_id;
    case Class::mem_access: {
      std::string s = "f_mem_access";
      if (!tag.empty()) return s + "_tag:" + tag;
      if (mem) s += "_" + memtype_str(*mem);
      if (mem_dtype) s += "_" + dtype_str(*mem_dtype);
      if (dir) s += "_" + direction_str(*dir);
      if (!lstride_cons.empty()) s += "_lstrides:" + constraint_list(lstride_cons);
      if (!gstride_cons.empty()) s += "_gstrides:" + constraint_list(gstride_cons);
      if (afr_con) s += "_afr:" + constraint_rel_str(afr_con->rel) + afr_con->rhs.str();
      return s;
    }
  }
  return "f_?";
}

FeatureSpec parse_feature(const std::string& id) {
  if (!starts(id, "f_")) throw EvalError("feature id must start with 'f_': " + id);
  const std::string rest = id.substr(2);
  FeatureSpec f;
  if (starts(rest, "op_")) {
    f.cls = FeatureSpec::Class::op;
    const std::string body = rest.substr(3);
    const size_t us = body.find('_');
    if (us == std::string::npos) throw EvalError("op feature needs dtype and op: " + id);
    f.dtype = dtype_from_str(body.substr(0, us));
    static const std::map<std::string, OpName> ops = {{"add", OpName::add}, {"mul", OpName::mul},
                                                      {"madd", OpName::madd}, {"div", OpName::div},
                                                      {"pow", OpName::pow_}};
    auto it = ops.find(body.substr(us + 1));
    if (it == ops.end()) throw EvalError("unknown op '" + body.substr(us + 1) + "' in " + id);
    f.op = it->second;
    return f;
  }
  if (starts(rest, "sync_")) {
    f.cls = FeatureSpec::Class::sync;
    const std::string kind = rest.substr(5);
    if (kind == "barrier_local") f.sync = SyncKind::barrier_local;
    else if (kind == "kernel_launch") f.sync = SyncKind::kernel_launch;
    else if (kind == "group_launch") f.sync = SyncKind::group_launch;
    else throw EvalError("unknown sync kind '" + kind + "' in " + id);
    return f;
  }
  if (rest == "thread_groups") {
    f.cls = FeatureSpec::Class::thread_groups;
    return f;
  }
  if (starts(rest, "exec_wall_time_")) {
    f.cls = FeatureSpec::Class::wall_time;
    f.executor_id = rest.substr(15);
    if (f.executor_id.empty()) throw EvalError("wall-time feature needs an executor id: " + id);
    return f;
  }
  if (starts(rest, "mem_access")) return parse_mem_access(id, rest.substr(10));
  throw EvalError("unknown feature class in '" + id + "'");
}

namespace {

bool holds(ConstraintRel rel, const Rational& lhs, const Rational& rhs) {
  return rel == ConstraintRel::eq ? lhs == rhs : rel == ConstraintRel::lt ? lhs < rhs : lhs > rhs;
}

Rational stride_value(const std::map<int, Poly>& m, int axis,
                      const std::map<std::string, long long>& b) {
  auto it = m.find(axis);
  return it == m.end() ? Rational(0) : it->second.eval(b);  // absent axis: no dependence
}

}  // namespace

bool pattern_matches(const FeatureSpec& spec, const AccessPattern& p,
                     const std::map<std::string, long long>& b) {
  if (spec.cls != FeatureSpec::Class::mem_access)
    throw EvalError("pattern_matches on non-memory feature " + spec.id());
  if (!spec.tag.empty()) return p.tag == spec.tag;
  if (spec.mem && *spec.mem != p.mem) return false;
  if (spec.mem_dtype && dtype_bytes(*spec.mem_dtype) != p.dtype_bytes) return false;
  if (spec.dir && *spec.dir != p.dir) return false;
  for (const auto& c : spec.lstride_cons)
    if (!holds(c.rel, stride_value(p.lstrides, c.axis, b), c.rhs.eval(b))) return false;
  for (const auto& c : spec.gstride_cons)
    if (!holds(c.rel, stride_value(p.gstrides, c.axis, b), c.rhs.eval(b))) return false;
  if (spec.afr_con && !holds(spec.afr_con->rel, p.afr.eval(b), spec.afr_con->rhs.eval(b)))
    return false;
  return true;
}

void check_bindings(const Kernel& k, const std::map<std::string, long long>& b) {
  for (const auto& a : k.assumptions) {
    auto it = b.find(a.param);
    if (it == b.end()) continue;
    const bool ok = a.kind == Assumption::Kind::divisible ? it->second % a.value == 0
                                                          : it->second >= a.value;
    if (!ok)
      throw EvalError("binding " + a.param + "=" + std::to_string(it->second) +
                      " violates assumption " + a.str());
  }
  for (const auto& p : k.domain.parameters)
    if (!b.count(p)) throw EvalError("missing binding for parameter '" + p + "'");
}

namespace {

// Sub-group entries count once per 32 (configurable) work-items; the
// division must be exact and the work-group a whole number of sub-groups.
std::atomic<bool> g_round_up_subgroups{false};

Rational per_granularity(const Rational& raw, Granularity g, const KernelCounts& c, int sgs,
                         const std::string& what) {
  long long div = 1;
  if (g == Granularity::sub_group) {
    div = sgs;
    const long long wg = c.geometry ? c.geometry->flat_work_group_size() : 0;
    if (wg && wg % sgs != 0) {
      // Reference semantics: an error (features.cpp:318-326).
      // Opt-in extension: a work-group of wg work-items issues
      // ceil(wg / sgs) sub-groups, so every sub-group entry converts at
      // ceil(wg/sgs)/wg per work-item execution. The factor does not depend on
      // the sizes (tabulable); the value need not be an integer.
      if (!g_round_up_subgroups.load())
        throw EvalError("work-group size " + std::to_string(wg) +
                        " is not a multiple of the sub-group size " + std::to_string(sgs));
      return raw * Rational((wg + sgs - 1) / sgs) / Rational(wg);
    }
  } else if (g == Granularity::work_group) {
    if (!c.geometry) throw EvalError("work-group granularity needs launch geometry");
    div = c.geometry->flat_work_group_size();
  }
  Rational v = raw / Rational(div);
  if (!is_integer(v))
    throw EvalError(what + ": count " + raw.str() + " is not divisible by the granularity divisor " +
                    std::to_string(div));
  return v;
}

// The symbolic counterpart of per_granularity for sub-group entries.
Rational sub_group_factor(const KernelCounts& c, int sgs) {
  const long long wg = c.geometry ? c.geometry->flat_work_group_size() : 0;
  if (wg && wg % sgs != 0 && g_round_up_subgroups.load())
    return Rational((wg + sgs - 1) / sgs) / Rational(wg);
  return Rational(1, sgs);
}

}  // namespace

double evaluate_feature_counts(const FeatureSpec& spec, const KernelCounts& c,
                               const std::map<std::string, long long>& b, int sgs,
                               std::optional<Poly>* symbolic) {
  Poly sym;
  Rational val(0);
  switch (spec.cls) {
    case FeatureSpec::Class::op:
      for (const auto& e : c.ops) {
        if (e.kind.dtype != spec.dtype || e.kind.op != spec.op) continue;
        val += per_granularity(e.count.eval(b), e.kind.gran, c, sgs, spec.id());
        sym += e.count * sub_group_factor(c, sgs);
      }
      break;
    case FeatureSpec::Class::mem_access:
      for (const auto& e : c.accesses) {
        if (!pattern_matches(spec, e.pattern, b)) continue;
        val += per_granularity(e.count.eval(b), e.pattern.gran, c, sgs, spec.id());
        sym += e.pattern.gran == Granularity::sub_group
                   ? e.count * sub_group_factor(c, sgs)
                   : e.count;
      }
      break;
    case FeatureSpec::Class::sync:
      for (const auto& e : c.sync) {
        if (e.kind != spec.sync) continue;
        val += e.count.eval(b);
        sym += e.count;
      }
      break;
    case FeatureSpec::Class::thread_groups: {
      if (!c.geometry)
        throw EvalError("thread_groups needs launch geometry (tag inames or mark the kernel "
                        "single-work-item)");
      sym = c.geometry->total_groups();
      val = sym.eval(b);
      break;
    }
    case FeatureSpec::Class::wall_time:
      throw EvalError("wall-time feature " + spec.id() + " is not a count feature");
  }
  if (symbolic) *symbolic = sym;
  return to_double(val);
}

FeatureValue evaluate_feature(const FeatureSpec& spec, const Kernel& k,
                              const std::map<std::string, long long>& b, Executor* executor,
                              int trials, int sgs, bool use_cache) {
  FeatureValue out;
  if (spec.cls == FeatureSpec::Class::wall_time) {
    if (!executor) throw EvalError("wall-time feature " + spec.id() + " requires an executor");
    check_bindings(k, b);
    out.numeric = measure_kernel(*executor, k, b, trials).mean_seconds;
    return out;
  }
  check_bindings(k, b);
  std::shared_ptr<const KernelCounts> counts =
      use_cache ? analyze_cached(k) : std::make_shared<const KernelCounts>(analyze(k));
  out.numeric = evaluate_feature_counts(spec, *counts, b, sgs, &out.symbolic);
  return out;
}

std::string FeatureTable::to_csv() const {
  std::ostringstream os;
  os << "kernel";
  for (const auto& c : columns) os << "," << c;
  os << "\n";
  os.precision(17);
  for (size_t r = 0; r < row_ids.size(); ++r) {
    os << row_ids[r];
    for (double v : values[r]) os << "," << v;
    os << "\n";
  }
  return os.str();
}

FeatureTable FeatureTable::from_csv(const std::string& text) {
  FeatureTable t;
  std::istringstream is(text);
  std::string line;
  bool header = true;
  while (std::getline(is, line)) {
    if (line.empty() || line[0] == '#') continue;
    std::vector<std::string> cells(1);
    for (char c : line) {
      if (c == ',')
        cells.emplace_back();
      else if (c != '\r')
        cells.back().push_back(c);
    }
    if (header) {
      if (cells[0] != "kernel") throw EvalError("feature CSV must start with a 'kernel' column");
      t.columns.assign(cells.begin() + 1, cells.end());
      header = false;
      continue;
    }
    std::vector<double> row;
    for (size_t i = 1; i < cells.size(); ++i) row.push_back(std::stod(cells[i]));
    if (row.size() != t.columns.size())
      throw EvalError("feature CSV row width mismatch at kernel " + cells[0]);
    t.row_ids.push_back(cells[0]);
    t.values.push_back(std::move(row));
  }
  return t;
}

const std::vector<double>& FeatureTable::row(const std::string& id) const {
  for (size_t i = 0; i < row_ids.size(); ++i)
    if (row_ids[i] == id) return values[i];
  throw EvalError("no feature row for kernel '" + id + "'");
}

FeatureTable gather_feature_values(const std::vector<FeatureSpec>& features,
                                   const std::vector<KernelInstance>& kernels, Executor* executor,
                                   int trials, int sgs) {
  FeatureTable t;
  for (const auto& f : features) t.columns.push_back(f.id());
  for (const auto& inst : kernels) {
    std::vector<double> row;
    row.reserve(features.size());
    for (const auto& f : features) {
      try {
        row.push_back(evaluate_feature(f, inst.kernel, inst.bindings, executor, trials, sgs).numeric);
      } catch (const Error& e) {
        throw EvalError("kernel '" + inst.id + "', feature " + f.id() + ": " + e.what());
      }
    }
    t.row_ids.push_back(inst.id);
    t.values.push_back(std::move(row));
  }
  return t;
}

}  // namespace perfseer

namespace perfseer {
void set_partial_subgroup_round_up(bool on) { g_round_up_subgroups.store(on); }
bool partial_subgroup_round_up() { return g_round_up_subgroups.load(); }
}  // namespace perfseer
