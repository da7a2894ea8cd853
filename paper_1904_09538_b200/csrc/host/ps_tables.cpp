// K18 host side: compile calibrated models x kernel variants into exact
// count tables for batched prediction (ps_eval_batched).
//
// For each variant the model's count features are symbolic polynomials in
// the variant's size parameters (counting engine + evaluate_feature's
// granularity rule, features.cpp:342-415). They are checked against the
// numeric feature values at several admissible sizes (so parameter-dependent
// pattern matching or divisibility would be caught, not silently frozen),
// then stored as integer-coefficient polynomials over a common denominator
// in the point coordinates. The GPU evaluates them exactly in 128-bit
// integers, converts to double, and runs the model bytecode.
#include "ps_tables.hpp"

#include <cmath>

#include "json.hpp"
#include "ps_catalog.hpp"
#include "ps_model.hpp"

namespace perfseer {

namespace {

// Sample bindings around `base` that keep every divisibility and lower-bound
// assumption: base * {1, 2, 3} rounded to the largest modulus.
std::vector<std::map<std::string, long long>> sample_bindings(const Kernel& k,
                                                              const std::map<std::string, long long>& base) {
  std::vector<std::map<std::string, long long>> out{base};
  for (long long mult : {2LL, 3LL, 5LL}) {
    std::map<std::string, long long> b = base;
    for (auto& [name, v] : b) {
      long long mod = k.divisibility_of(name).value_or(1);
      v = ((v * mult + mod - 1) / mod) * mod;
    }
    out.push_back(b);
  }
  return out;
}

}  // namespace

VariantTables build_variant_tables(const std::string& spec_json) {
  auto spec = nlohmann::json::parse(spec_json);
  VariantTables t;
  std::map<std::string, int> model_index;
  for (const auto& v : spec.at("variants")) {
    const std::string id = v.at("id").get<std::string>();
    const std::string text = v.at("model").get<std::string>();
    GeneratedKernel g = kernel_from_variant_id(id);
    Model m = parse_model_file(text);
    auto counts = analyze_cached(g.kernel);

    // One compiled model per (text, parameter values): the same model text
    // calibrated on different machines (or runs) stays distinct.
    std::vector<double> p = v.at("params").get<std::vector<double>>();
    if (p.size() != m.params.size())
      throw EvalError("variant '" + id + "': " + std::to_string(p.size()) + " params for a model with " +
                      std::to_string(m.params.size()));
    std::string key = text;
    key.push_back('\0');
    for (double x : p) key.append(reinterpret_cast<const char*>(&x), sizeof x);
    int mi;
    auto it = model_index.find(key);
    if (it == model_index.end()) {
      mi = int(t.models.size());
      model_index[key] = mi;
      t.models.push_back(compile_model_program(m, false));
      t.params.push_back(p);
      t.model_nf.push_back(int(m.features.size()));
    } else {
      mi = it->second;
    }
    const int group = v.value("group", 0);
    if (group < 0 || group >= 8)
      throw EvalError("variant '" + id + "': group " + std::to_string(group) + " outside 0..7");
    std::map<std::string, int> coords;
    for (const auto& [name, c] : v.at("coords").items()) coords[name] = c.get<int>();
    for (const auto& p : g.kernel.domain.parameters)
      if (!coords.count(p)) throw EvalError("variant '" + id + "': parameter '" + p + "' has no point coordinate");

    t.var_group.push_back(group);
    t.var_model.push_back(mi);
    t.var_id.push_back(id);
    t.var_feat_base.push_back(int(t.feat_begin.size()));
    for (size_t f = 0; f < m.features.size(); ++f) {
      std::optional<Poly> sym;
      evaluate_feature_counts(m.features[f], *counts, g.bindings, 32, &sym);
      // The symbolic value must reproduce the numeric one at every sample.
      for (const auto& b : sample_bindings(g.kernel, g.bindings)) {
        const double num = evaluate_feature_counts(m.features[f], *counts, b, 32);
        const double symv = to_double(sym->eval(b));
        if (num != symv)
          throw EvalError("variant '" + id + "', feature " + m.feature_ids[f] +
                          ": symbolic count disagrees with evaluation at a sample size "
                          "(parameter-dependent match); not tabulable");
      }
      BigInt den(1);
      for (const auto& [mono, c] : sym->terms()) den = lcm(den, denominator(c));
      t.feat_begin.push_back(int(t.term_coef.size()));
      t.feat_den.push_back(den.convert_to<long long>());
      for (const auto& [mono, c] : sym->terms()) {
        t.term_coef.push_back(numerator(c * Rational(den)).convert_to<long long>());
        std::array<int8_t, 4> e{0, 0, 0, 0};
        for (const auto& [sname, x] : mono.exps) {
          const int ci = coords.at(sname);
          if (ci < 0 || ci > 3) throw EvalError("point coordinates are 0..3");
          e[size_t(ci)] = int8_t(e[size_t(ci)] + x);
        }
        t.term_exp.push_back(e);
      }
      t.feat_end.push_back(int(t.term_coef.size()));
    }
  }
  for (int g : t.var_group) t.ngroups = std::max(t.ngroups, g + 1);
  if (t.var_model.size() > 256)
    throw EvalError("at most 256 variants per table set (the argmin is one byte per group)");
  for (const auto& pr : t.models)
    if (pr.n_slots > 64) throw EvalError("model program needs " + std::to_string(pr.n_slots) +
                                         " registers (device evaluator: 64)");
  return t;
}

// Rational::convert_to<double> of acc/den: reduce to lowest terms, then one
// double division (ps_exact.hpp), so table values equal evaluate_feature's.
double rational_to_double(__int128 acc, long long den) {
  if (den == 1) return double(acc);
  __int128 a = acc < 0 ? -acc : acc, b = den;
  while (b) {
    __int128 r = a % b;
    a = b;
    b = r;
  }
  if (a > 1) {
    acc /= a;
    den /= (long long)a;
  }
  return double(acc) / double(den);
}

std::vector<double> eval_point_cpu(const VariantTables& t, size_t v, const int64_t* point) {
  const size_t nf = size_t(t.model_nf[size_t(t.var_model[v])]);
  std::vector<double> f(nf);
  for (size_t j = 0; j < nf; ++j) {
    const size_t slot = size_t(t.var_feat_base[v]) + j;
    __int128 acc = 0;
    for (int k = t.feat_begin[slot]; k < t.feat_end[slot]; ++k) {
      __int128 term = t.term_coef[size_t(k)];
      for (int c = 0; c < 4; ++c)
        for (int e = 0; e < t.term_exp[size_t(k)][size_t(c)]; ++e) term *= point[c];
      acc += term;
    }
    f[j] = rational_to_double(acc, t.feat_den[slot]);
  }
  return f;
}

}  // namespace perfseer
