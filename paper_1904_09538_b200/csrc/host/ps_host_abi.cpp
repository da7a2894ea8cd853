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
#include "ps_enumerate.hpp"
#include "ps_executor.hpp"
#include "ps_json.hpp"
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

int ps_kernel_json(const char* variant_id, char* out, size_t cap, size_t* needed) {
  return guarded([&] {
    if (!variant_id) throw EvalError("ps_kernel_json: null variant id");
    GeneratedKernel g = kernel_from_variant_id(variant_id);
    nlohmann::json j;
    j["id"] = g.id;
    j["kernel"] = kernel_to_json(g.kernel);
    j["bindings"] = g.bindings;
    return copy_out(j.dump(), out, cap, needed);
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
      stats->trials = 0;
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
    // scale: 0 reference start on raw rows, 1 reference start on output-scaled
    // rows (what fit_model uses), 2 relative-residual QR start (B200 fit).
    const auto p0 = scale == 2 ? initial_point_relative(m, p)
                               : initial_point(m, scale ? scale_features_by_output(p) : p);
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

int ps_model_program(const char* model_text, int with_jacobian, char* out, size_t cap, size_t* needed) {
  return guarded([&] {
    Model m = model_from_text(model_text);
    Program pr = compile_model_program(m, with_jacobian != 0);
    nlohmann::json j;
    j["insns"] = pr.insns;
    j["consts"] = pr.consts;
    j["outputs"] = pr.outputs;
    j["n_slots"] = pr.n_slots;
    j["n_nodes"] = pr.n_nodes;
    return copy_out(j.dump(), out, cap, needed);
  });
}

int ps_fit_lm_jobs(ps_ctx* ctx, int njobs, const ps_lm_job* jobs, double* kernel_seconds) {
  return guarded([&] {
    if (!ctx || !jobs || njobs < 1) throw EvalError("ps_fit_lm_jobs: bad argument");
    // one value program and one value+Jacobian program per distinct model text
    std::map<std::string, std::pair<Program, Program>> progs;
    std::map<std::string, int> nfeat;
    std::vector<ps::LmJobHost> hj(static_cast<size_t>(njobs));
    for (int j = 0; j < njobs; ++j) {
      const ps_lm_job& in = jobs[j];
      if (!in.model_text || !in.features || !in.t || !in.params_inout || !in.stats)
        throw EvalError("ps_fit_lm_jobs: job " + std::to_string(j) + " has a null pointer");
      auto it = progs.find(in.model_text);
      if (it == progs.end()) {
        Model m = model_from_text(in.model_text);
        nfeat[in.model_text] = int(m.features.size());
        it = progs.emplace(in.model_text, std::make_pair(compile_model_program(m, false),
                                                         compile_model_program(m, true))).first;
      }
      if (nfeat[in.model_text] != in.nf)
        throw EvalError("ps_fit_lm_jobs: job " + std::to_string(j) + ": model has " +
                        std::to_string(nfeat[in.model_text]) + " features, job gives " + std::to_string(in.nf));
      if (in.nr < 1 || in.nbatch < 1)
        throw EvalError("ps_fit_lm_jobs: job " + std::to_string(j) + ": nr and nbatch must be >= 1");
      auto view = [](const Program& pr) {
        return ps::LmProgramHost{pr.insns.data(), pr.consts.data(), pr.outputs.data(), int(pr.insns.size() / 2),
                                 int(pr.consts.size()), int(pr.outputs.size()), pr.n_slots};
      };
      ps::LmJobHost& h = hj[size_t(j)];
      h.value = view(it->second.first);
      h.full = view(it->second.second);
      h.np = int(it->second.second.outputs.size()) - 1;
      h.nf = in.nf;
      h.nr = in.nr;
      h.nbatch = in.nbatch;
      h.mode = in.mode;
      h.shared_rows = in.shared_rows;
      h.features = in.features;
      h.t = in.t;
      h.opts = in.opts;
      h.params = in.params_inout;
      h.stats = in.stats;
    }
    const int rc = ps::fit_lm_jobs_gpu(reinterpret_cast<ps::Ctx*>(ctx), njobs, hj.data(), kernel_seconds);
    if (rc) throw EvalError(ps_last_error());
    return PS_OK;
  });
}

int ps_set_option(const char* key, const char* value) {
  return guarded([&] {
    const std::string k = key ? key : "", v = value ? value : "";
    if (k == "partial_subgroups") {
      if (v != "strict" && v != "round_up") throw EvalError("partial_subgroups: strict | round_up");
      set_partial_subgroup_round_up(v == "round_up");
      clear_count_cache();
      return PS_OK;
    }
    if (k == "launch_geometry") {
      if (v != "realised" && v != "literal") throw EvalError("launch_geometry: realised | literal");
      ps::set_literal_geometry(v == "literal");
      return PS_OK;
    }
    if (k == "k18_jit") {
      if (v != "on" && v != "off") throw EvalError("k18_jit: on | off");
      ps::set_k18_jit(v == "on");
      return PS_OK;
    }
    if (k == "measure_queue_ahead") {
      if (v != "on" && v != "off") throw EvalError("measure_queue_ahead: on | off");
      ps::set_queue_ahead(v == "on");
      return PS_OK;
    }
    throw EvalError("unknown option '" + k + "'");
  });
}

int ps_geo_mean_rel_error(const double* pred, const double* meas, int n, double* out) {
  return guarded([&] {
    *out = geo_mean_rel_error(std::vector<double>(pred, pred + n), std::vector<double>(meas, meas + n));
    return PS_OK;
  });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// K18 tables

#include <mutex>
#include <thread>

#include "ps_tables.hpp"

struct ps_tables {
  perfseer::VariantTables t;
  // flattened model programs for the device
  std::vector<int32_t> model_insn_begin, model_out, model_regs, model_const_begin, model_param_begin;
  std::vector<uint32_t> insns;
  std::vector<double> consts, params;
  std::vector<int8_t> term_exp;
  // K18 kernels specialised to these tables (eval_jit.cu), per device; one
  // table set may be evaluated from several contexts (GPUs) on several threads
  mutable std::map<int, void*> jit;
  mutable std::mutex jit_mu;
  ps::FlatTables flat() const {
    ps::FlatTables f{};
    f.nvar = int(t.var_model.size());
    f.ngroups = t.ngroups;
    f.nmodels = int(t.models.size());
    f.var_group = t.var_group.data();
    f.var_model = t.var_model.data();
    f.var_feat_base = t.var_feat_base.data();
    f.feat_begin = t.feat_begin.data();
    f.feat_end = t.feat_end.data();
    f.feat_den = t.feat_den.data();
    f.term_coef = t.term_coef.data();
    f.term_exp = term_exp.data();
    f.nslots = int(t.feat_begin.size());
    f.nterms = int(t.term_coef.size());
    f.model_nf = t.model_nf.data();
    f.model_insn_begin = model_insn_begin.data();
    f.insns = insns.data();
    f.model_out = model_out.data();
    f.model_regs = model_regs.data();
    f.model_const_begin = model_const_begin.data();
    f.consts = consts.data();
    f.model_param_begin = model_param_begin.data();
    f.params = params.data();
    return f;
  }
};

extern "C" {

int ps_tables_build(const char* spec_json, ps_tables** out) {
  return guarded([&] {
    if (!spec_json || !out) throw EvalError("ps_tables_build: null argument");
    auto* h = new ps_tables();
    try {
      h->t = build_variant_tables(spec_json);
    } catch (...) {
      delete h;
      throw;
    }
    h->model_insn_begin.push_back(0);
    h->model_const_begin.push_back(0);
    h->model_param_begin.push_back(0);
    for (size_t m = 0; m < h->t.models.size(); ++m) {
      const auto& pr = h->t.models[m];
      h->insns.insert(h->insns.end(), pr.insns.begin(), pr.insns.end());
      h->consts.insert(h->consts.end(), pr.consts.begin(), pr.consts.end());
      h->params.insert(h->params.end(), h->t.params[m].begin(), h->t.params[m].end());
      h->model_insn_begin.push_back(int32_t(h->insns.size() / 2));
      h->model_out.push_back(pr.outputs.at(0));
      h->model_regs.push_back(pr.n_slots);
      h->model_const_begin.push_back(int32_t(h->consts.size()));
      h->model_param_begin.push_back(int32_t(h->params.size()));
    }
    for (const auto& e : h->t.term_exp) h->term_exp.insert(h->term_exp.end(), e.begin(), e.end());
    *out = h;
    return PS_OK;
  });
}

int ps_tables_info(const ps_tables* t, int* nvar, int* ngroups, int64_t* nterms) {
  if (!t) return ps::set_error(PS_ERR_ARG, "null tables");
  if (nvar) *nvar = int(t->t.var_model.size());
  if (ngroups) *ngroups = t->t.ngroups;
  if (nterms) *nterms = int64_t(t->t.term_coef.size());
  return PS_OK;
}

int ps_tables_free(ps_tables* t) {
  delete t;
  return PS_OK;
}

// The tables' specialised K18 kernel on ctx's device (compiled and loaded on
// first use), or null when the interpreter is selected.
static int jit_kernel_for(ps_ctx* ctx, const ps_tables* tables, void** kernel, double* seconds) {
  *kernel = nullptr;
  if (seconds) *seconds = 0.0;
  if (!ps::k18_jit_enabled()) return PS_OK;
  auto* c = reinterpret_cast<ps::Ctx*>(ctx);
  std::lock_guard<std::mutex> lock(tables->jit_mu);
  auto it = tables->jit.find(c->device);
  if (it != tables->jit.end()) {
    *kernel = it->second;
    return PS_OK;
  }
  const int rc = ps::k18_jit_kernel(c, tables->flat(), kernel, seconds);
  if (rc == PS_OK) tables->jit[c->device] = *kernel;  // null: too large, the interpreter
  return rc;
}

int ps_eval_prepare(ps_ctx* ctx, const ps_tables* tables, double* jit_seconds) {
  if (!ctx || !tables) return ps::set_error(PS_ERR_ARG, "ps_eval_prepare: null argument");
  void* k = nullptr;
  return jit_kernel_for(ctx, tables, &k, jit_seconds);
}

int ps_eval_jit_source(const ps_tables* tables, char* out, size_t cap, size_t* needed) {
  return guarded([&] {
    if (!tables) throw EvalError("ps_eval_jit_source: null tables");
    return copy_out(ps::k18_jit_source(tables->flat()), out, cap, needed);
  });
}

int ps_eval_jit_compile(const ps_tables* tables, size_t* cubin_bytes) {
  if (!tables) return ps::set_error(PS_ERR_ARG, "ps_eval_jit_compile: null tables");
  std::vector<char> cubin;
  const int rc = ps::k18_jit_compile(ps::k18_jit_source(tables->flat()), &cubin);
  if (rc == PS_OK && cubin_bytes) *cubin_bytes = cubin.size();
  return rc;
}

int ps_eval_batched(ps_ctx* ctx, const ps_tables* tables, const int64_t* points, int64_t npts,
                    double* pred, uint8_t* argmin, double* kernel_seconds) {
  if (!ctx || !tables || !points || !pred || !argmin) return ps::set_error(PS_ERR_ARG, "ps_eval_batched: null argument");
  void* jit = nullptr;
  if (int rc = jit_kernel_for(ctx, tables, &jit, nullptr)) return rc;
  return ps::eval_tables_gpu(reinterpret_cast<ps::Ctx*>(ctx), tables->flat(), points, npts, pred, argmin,
                             kernel_seconds, jit);
}

// The same evaluation on host threads (exact int128 features, double model).
int ps_eval_cpu(const ps_tables* tables, const int64_t* points, int64_t npts, double* pred,
                uint8_t* argmin, int threads) {
  return guarded([&] {
    if (!tables || !points || !pred || !argmin) throw EvalError("ps_eval_cpu: null argument");
    const auto& t = tables->t;
    const size_t nvar = t.var_model.size();
    const int ng = t.ngroups;
    auto work = [&](int64_t lo, int64_t hi) {
      for (int64_t pt = lo; pt < hi; ++pt) {
        std::vector<int> besti(size_t(ng), -1);
        std::vector<double> best(size_t(ng), 0.0);
        for (size_t v = 0; v < nvar; ++v) {
          const auto f = eval_point_cpu(t, v, points + pt * 4);
          const int m = t.var_model[v];
          double y;
          run_program(t.models[size_t(m)], t.params[size_t(m)].data(), f.data(), &y);
          pred[pt * int64_t(nvar) + int64_t(v)] = y;
          const int g = t.var_group[v];
          if (besti[size_t(g)] < 0 || y < best[size_t(g)]) {
            best[size_t(g)] = y;
            besti[size_t(g)] = int(v);
          }
        }
        for (int g = 0; g < ng; ++g) argmin[pt * ng + g] = uint8_t(besti[size_t(g)]);
      }
    };
    const int n = std::max(1, threads);
    std::vector<std::thread> pool;
    for (int i = 0; i < n; ++i)
      pool.emplace_back(work, npts * i / n, npts * (i + 1) / n);
    for (auto& th : pool) th.join();
    return PS_OK;
  });
}

}  // extern "C"

// SPEC acceptance 1 at any size: symbolic counts (analyze), the CPU
// enumerator (brute_force_count, oracle.cpp:429-443) or the GPU enumerator,
// as one JSON record of the variant at its own bindings.
int ps_enumerate(ps_ctx* ctx, const char* variant_id, int mode, char* out, size_t cap,
                 size_t* needed) {
  return guarded([&] {
    const GeneratedKernel g = kernel_from_variant_id(variant_id ? variant_id : "");
    nlohmann::json j;
    auto ll = [&](const Poly& p) {
      const Rational v = p.eval(g.bindings);
      if (!is_integer(v)) throw EvalError("non-integral count");
      return numerator(v).convert_to<long long>();
    };
    if (mode == 0) {
      const KernelCounts c = analyze(g.kernel);
      std::map<std::string, long long> ops, acc, fp;
      for (const auto& e : c.ops)
        if (long long v = ll(e.count)) ops[e.kind.key()] += v;
      for (const auto& e : c.accesses)
        if (long long v = ll(e.count)) acc[evaluate_pattern(e.pattern, g.bindings).key()] += v;
      for (const auto& [a, p] : c.footprints) fp[a] = ll(p);
      long long bar = 0;
      for (const auto& e : c.sync)
        if (e.kind == SyncKind::barrier_local) bar = ll(e.count);
      j["ops"] = ops;
      j["access_counts"] = acc;
      j["footprints"] = fp;
      j["barrier_local"] = bar;
    } else {
      if (mode == 2 && !ctx) throw EvalError("ps_enumerate: GPU mode needs a context");
      const OracleCounts o = mode == 2 ? brute_force_count_gpu(ctx, g.kernel, g.bindings)
                                       : brute_force_count(g.kernel, g.bindings, 2'000'000'000LL);
      std::map<std::string, long long> ops, acc;
      for (const auto& [k, v] : o.ops)
        if (v) ops[k] = v;
      for (const auto& [k, v] : o.access_counts)
        if (v) acc[k] = v;
      j["ops"] = ops;
      j["access_counts"] = acc;
      j["access_footprints"] = o.access_footprints;
      j["footprints"] = o.footprints;
      j["barrier_local"] = o.barrier_local;
      j["group_launch"] = o.group_launch;
    }
    return copy_out(j.dump(), out, cap, needed);
  });
}
