// Host-side C ABI over the C++ port (declared in include/perfseer_b200.h,
// "host pipeline" section): catalog expansion, count-feature tables, the
// reference-exact CPU fit, prediction, and model bytecode export. Strings in,
// caller-owned buffers out; errors via ps_last_error().
#include <cstring>
#include <sstream>

#include "../../../include/perfseer_b200.h"
#include "../cuda/runtime_internal.h"
#include "json.hpp"
#include "ps_catalog.hpp"
#include "ps_executor.hpp"
#include "ps_model.hpp"

using namespace perfseer;

namespace {

std::vector<std::string> split_lines(const char* text) {
  std::vector<std::string> out;
  if (!text) return out;
  std::istringstream is(text);
  std::string line;
  while (std::getline(is, line)) {
    while (!line.empty() && (line.back() == '\r' || line.back() == ' ')) line.pop_back();
    if (!line.empty()) out.push_back(line);
  }
  return out;
}

int copy_out(const std::string& s, char* out, size_t cap, size_t* needed) {
  if (needed) *needed = s.size() + 1;
  if (!out || cap < s.size() + 1)
    return ps::set_error(PS_ERR_ARG, "output buffer too small (%zu bytes needed)", s.size() + 1);
  std::memcpy(out, s.c_str(), s.size() + 1);
  return PS_OK;
}

template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const std::exception& e) {
    return ps::set_error(PS_ERR_ARG, "%s", e.what());
  }
}

Model model_from_text(const char* text) {
  if (!text) throw EvalError("null model text");
  return parse_model_file(text);
}

FitOptions fit_options(const ps_fit_opts* o) {
  FitOptions f;
  if (!o) return f;
  f.lambda0 = o->lambda0;
  f.lambda_decrease = o->lambda_decrease;
  f.lambda_increase = o->lambda_increase;
  f.step_tol = o->step_tol;
  f.grad_tol = o->grad_tol;
  f.max_iterations = o->max_iterations;
  f.nonnegative = o->nonnegative != 0;
  return f;
}

}  // namespace

extern "C" {

int ps_catalog(const char* catalog, const char* tags, const char* match, char* out, size_t cap,
               size_t* needed) {
  return guarded([&] {
    const std::string which = catalog ? catalog : "b200";
    std::vector<Generator> gens;
    if (which == "reference")
      gens = builtin_generators();
    else if (which == "b200")
      gens = b200_generators();
    else
      throw SemanticError("unknown catalog '" + which + "' (reference | b200)");
    KernelCollection coll(std::move(gens));
    auto kernels = coll.generate(FilterTagSet::parse(split_lines(tags)),
                                 match_condition_from_str(match && *match ? match : "superset"));
    std::string s;
    for (const auto& g : kernels) s += g.id + "\t" + bindings_str(g.bindings) + "\n";
    return copy_out(s, out, cap, needed);
  });
}

int ps_model_info(const char* model_text, char* out, size_t cap, size_t* needed) {
  return guarded([&] {
    Model m = model_from_text(model_text);
    nlohmann::json j;
    j["output"] = m.output_id;
    j["expression"] = m.expr_src;
    j["params"] = m.params;
    j["features"] = m.feature_ids;
    std::vector<int> cost;
    for (bool c : cost_parameter_mask(m)) cost.push_back(c ? 1 : 0);
    j["cost_params"] = cost;
    return copy_out(j.dump(), out, cap, needed);
  });
}

int ps_feature_table(const char* model_text, const char* variant_ids, int sub_group_size,
                     double* out, int64_t cap_values) {
  return guarded([&] {
    Model m = model_from_text(model_text);
    const auto ids = split_lines(variant_ids);
    const int64_t need = int64_t(ids.size()) * int64_t(m.features.size());
    if (cap_values < need) throw EvalError("feature table buffer too small");
    std::vector<KernelInstance> inst;
    inst.reserve(ids.size());
    for (const auto& id : ids) {
      GeneratedKernel g = kernel_from_variant_id(id);
      inst.push_back(KernelInstance{g.id, g.kernel, g.bindings});
    }
    FeatureTable t = gather_feature_values(m.features, inst, nullptr, 60, sub_group_size);
    for (size_t r = 0; r < t.values.size(); ++r)
      for (size_t c = 0; c < t.values[r].size(); ++c) out[r * m.features.size() + c] = t.values[r][c];
    return PS_OK;
  });
}

int ps_fit_cpu(const char* model_text, const double* features, const double* t, int nr, int scale,
               const ps_fit_opts* opts, double* params_out, ps_fit_stats* stats) {
  return guarded([&] {
    Model m = model_from_text(model_text);
    const size_t nf = m.features.size();
    CalibrationProblem p;
    for (int r = 0; r < nr; ++r)
      p.rows.push_back(CalibrationRow{std::vector<double>(features + size_t(r) * nf, features + size_t(r + 1) * nf), t[r]});
    CalibratedModel cm = fit_model(m, scale ? scale_features_by_output(p) : p, fit_options(opts));
    const auto pv = cm.param_vector();
    std::copy(pv.begin(), pv.end(), params_out);
    if (stats) {
      stats->residual_norm = cm.residual_norm;
      stats->iterations = cm.iterations;
      stats->converged = cm.converged ? 1 : 0;
      stats->status = 0;
    }
    return PS_OK;
  });
}

int ps_initial_point(const char* model_text, const double* features, const double* t, int nr, int scale,
                     double* params_out) {
  return guarded([&] {
    Model m = model_from_text(model_text);
    const size_t nf = m.features.size();
    CalibrationProblem p;
    for (int r = 0; r < nr; ++r)
      p.rows.push_back(CalibrationRow{std::vector<double>(features + size_t(r) * nf, features + size_t(r + 1) * nf), t[r]});
    const auto p0 = initial_point(m, scale ? scale_features_by_output(p) : p);
    std::copy(p0.begin(), p0.end(), params_out);
    return PS_OK;
  });
}

int ps_predict_cpu(const char* model_text, const double* params, const char* variant_ids,
                   int sub_group_size, double* out, int64_t cap) {
  return guarded([&] {
    Model m = model_from_text(model_text);
    const auto ids = split_lines(variant_ids);
    if (cap < int64_t(ids.size())) throw EvalError("prediction buffer too small");
    CalibratedModel cm;
    cm.model = m;
    for (size_t i = 0; i < m.params.size(); ++i) cm.param_values[m.params[i]] = params[i];
    for (size_t i = 0; i < ids.size(); ++i) {
      GeneratedKernel g = kernel_from_variant_id(ids[i]);
      out[i] = predict(cm, g.kernel, g.bindings, sub_group_size);
    }
    return PS_OK;
  });
}

int ps_model_bytecode(const char* model_text, int which, int32_t* ops, int cap_ops, double* consts,
                      int cap_consts, int* n_ops, int* n_consts, int* max_stack) {
  return guarded([&] {
    Model m = model_from_text(model_text);
    if (which < -1 || which >= int(m.params.size())) throw EvalError("bytecode index out of range");
    Bytecode bc = compile_bytecode(which < 0 ? m.expr : differentiate(m, size_t(which)));
    if (n_ops) *n_ops = int(bc.ops.size());
    if (n_consts) *n_consts = int(bc.consts.size());
    if (max_stack) *max_stack = bc.max_stack;
    if (int(bc.ops.size()) > cap_ops || int(bc.consts.size()) > cap_consts)
      throw EvalError("bytecode buffer too small");
    std::copy(bc.ops.begin(), bc.ops.end(), ops);
    std::copy(bc.consts.begin(), bc.consts.end(), consts);
    return PS_OK;
  });
}

int ps_geo_mean_rel_error(const double* pred, const double* meas, int n, double* out) {
  return guarded([&] {
    *out = geo_mean_rel_error(std::vector<double>(pred, pred + n), std::vector<double>(meas, meas + n));
    return PS_OK;
  });
}

}  // extern "C"
