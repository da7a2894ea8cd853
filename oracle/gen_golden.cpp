// TEST INFRASTRUCTURE ONLY. Golden-fixture generator linked against the
// UNMODIFIED reference library (oracle/_ref/libperfseer_ref.a, built from
// /root/reference/proj/src by oracle/Makefile). Emits JSON on stdout:
//   kernels : outputs of small generated kernels under the reference's own IR
//             interpreter run_reference (tests/support.hpp:50-162) with its
//             seed_value inputs (support.hpp:35-44) — pins oracle/suite_ref.c;
//   counts  : full symbolic KernelCounts of every catalog kernel
//             (counting.cpp:217-252, 697-715) and their values at the bindings;
//   features: feature values (features.cpp:342-415) for the model feature ids;
//   fits    : fit_model results (model.cpp:485-606) on canned problems.
// Regenerate with `make -C oracle golden` (writes tests/golden/reference.json).
#include <cmath>
#include <iostream>
#include <random>

#include "json.hpp"
#include "perfseer/counting.hpp"
#include "perfseer/executor.hpp"
#include "perfseer/features.hpp"
#include "perfseer/lang.hpp"
#include "perfseer/model.hpp"
#include "perfseer/transforms.hpp"
#include "perfseer/uipick.hpp"
#include "support.hpp"

using namespace perfseer;
using nlohmann::json;

static std::string rat_str(const Rational& r) { return r.str(); }

static json counts_json(const KernelCounts& c, const std::map<std::string, long long>& b) {
  json j;
  json ops = json::array();
  for (const auto& e : c.ops)
    ops.push_back({{"key", e.kind.key()}, {"gran", granularity_str(e.kind.gran)},
                   {"count", e.count.str()}, {"value", rat_str(e.count.eval(b))}});
  j["ops"] = ops;
  json acc = json::array();
  for (const auto& e : c.accesses)
    acc.push_back({{"pattern", e.pattern.str()}, {"count", e.count.str()},
                   {"value", rat_str(e.count.eval(b))},
                   {"afr_value", rat_str(e.pattern.afr.eval(b))}});
  j["accesses"] = acc;
  json sync = json::array();
  for (const auto& e : c.sync)
    sync.push_back({{"kind", synckind_str(e.kind)}, {"count", e.count.str()},
                    {"value", rat_str(e.count.eval(b))}});
  j["sync"] = sync;
  json fp = json::object();
  for (const auto& [a, p] : c.footprints) fp[a] = {{"poly", p.str()}, {"value", rat_str(p.eval(b))}};
  j["footprints"] = fp;
  if (c.geometry) {
    j["work_group_size"] = c.geometry->work_group_size;
    json ng = json::array();
    for (const auto& g : c.geometry->num_groups) ng.push_back(g.str());
    j["num_groups"] = ng;
  }
  return j;
}

static const std::vector<std::string> kFeatureIds = {
    "f_op_float32_add",
    "f_op_float32_mul",
    "f_op_float32_madd",
    "f_op_float64_madd",
    "f_mem_access_local_float32",
    "f_mem_access_global_float32_load",
    "f_mem_access_global_float32_store",
    "f_mem_access_global_float32_lstrides:{0:1;1:>1}_gstrides:{0:16;1:>16}_afr:1",
    "f_mem_access_global_float32_load_lstrides:{0:1;1:>15}_gstrides:{0:0}_afr:>1",
    "f_mem_access_global_float32_load_lstrides:{0:1;1:>15}_gstrides:{0:16}_afr:>1",
    "f_mem_access_tag:mm-PF-a",
    "f_mem_access_tag:mm-PF-b",
    "f_mem_access_tag:mm-noPF-a",
    "f_mem_access_tag:mm-noPF-b",
    "f_mem_access_tag:fd-16x16-u",
    "f_mem_access_tag:fd-16x16-res",
    "f_mem_access_tag:fd-18x18-u",
    "f_mem_access_tag:fd-18x18-res",
    "f_sync_barrier_local",
    "f_sync_kernel_launch",
    "f_sync_group_launch",
    "f_thread_groups",
};

static json run_kernel_json(const std::string& id, const Kernel& k,
                            const std::map<std::string, long long>& b,
                            const std::string& output) {
  auto out = testing::run_reference(k, b);
  json j;
  j["id"] = id;
  j["bindings"] = b;
  j["output"] = output;
  j["values"] = out.at(output);
  return j;
}

int main() {
  json root;
  root["generator"] = "oracle/gen_golden.cpp against /root/reference/proj (unmodified)";

  // ---- 1. kernel outputs under the reference interpreter ------------------
  json kernels = json::array();
  auto pat = [](std::map<std::string, std::string> a) {
    a.emplace("dtype", "float32");
    a.emplace("lsize_0", "16");
    a.emplace("lsize_1", "16");
    a.emplace("lid_stride_0", "1");
    a.emplace("lid_stride_1", "64");
    a.emplace("nelements", "2048");
    return a;
  };
  for (const std::string k : {"1", "2"}) {
    GeneratedKernel g = make_gmem_pattern(pat({{"n_input_arrays", k}}));
    kernels.push_back(run_kernel_json(g.id, g.kernel, g.bindings, "result"));
  }
  {
    // Non-unit strides: lid_stride_0 = 2 leaves gaps (only the index set is written).
    GeneratedKernel g = make_gmem_pattern(pat({{"n_input_arrays", "2"}, {"lid_stride_0", "2"},
                                               {"lid_stride_1", "128"}, {"nelements", "4096"}}));
    kernels.push_back(run_kernel_json(g.id, g.kernel, g.bindings, "result"));
  }
  for (const std::string n : {"32", "48"}) {
    for (const std::string pf : {"False"}) {
      GeneratedKernel g = make_matmul_sq({{"dtype", "float32"}, {"prefetch", pf},
                                          {"lsize_0", "16"}, {"lsize_1", "16"},
                                          {"groups_fit", "True"}, {"n", n}});
      kernels.push_back(run_kernel_json(g.id, g.kernel, g.bindings, "c"));
    }
    // The PF kernel stages tiles (not functional under run_reference); its
    // output equals the untiled matmul source on the same inputs.
    Kernel src = make_kernel("{[i,j,k]: 0<=i,j,k<n}", {"c[i,j] = sum(k, a[i,k]*b[k,j])"},
                             {{"a", Dtype::float32, {"n", "n"}},
                              {"b", Dtype::float32, {"n", "n"}},
                              {"c", Dtype::float32, {"n", "n"}}});
    GeneratedKernel pf = make_matmul_sq({{"dtype", "float32"}, {"prefetch", "True"},
                                         {"lsize_0", "16"}, {"lsize_1", "16"},
                                         {"groups_fit", "True"}, {"n", n}});
    kernels.push_back(run_kernel_json(pf.id, src, pf.bindings, "c"));
    for (const std::string pfv : {"True", "False"})
      for (const std::string keep : {"a", "b"}) {
        GeneratedKernel g = make_matmul_sq_rm({{"dtype", "float32"}, {"prefetch", pfv},
                                               {"keep", keep}, {"lsize_0", "16"},
                                               {"lsize_1", "16"}, {"groups_fit", "True"},
                                               {"n", n}});
        kernels.push_back(run_kernel_json(g.id, g.kernel, g.bindings, "tgt_read_dest"));
      }
  }
  for (const auto& [tile, n] : std::vector<std::pair<std::string, std::string>>{
           {"16x16", "28"}, {"16x16", "42"}, {"18x18", "32"}, {"18x18", "48"}}) {
    Kernel fd_src = make_kernel(
        "{[i,j]: 0<=i,j<n}",
        {"res[i,j] = u[i,j+1] + u[i+1,j] - 4*u[i+1,j+1] + u[i+1,j+2] + u[i+2,j+1]"},
        {{"u", Dtype::float32, {"n + 2", "n + 2"}}, {"res", Dtype::float32, {"n", "n"}}});
    GeneratedKernel g = make_fd_stencil({{"dtype", "float32"}, {"tile", tile}, {"n", n}});
    kernels.push_back(run_kernel_json(g.id, fd_src, g.bindings, "res"));
    GeneratedKernel ru = make_fd_stencil_rm({{"dtype", "float32"}, {"tile", tile}, {"keep", "u"},
                                             {"n", n}});
    kernels.push_back(run_kernel_json(ru.id, ru.kernel, ru.bindings, "tgt_read_dest"));
    GeneratedKernel rr = make_fd_stencil_rm({{"dtype", "float32"}, {"tile", tile},
                                             {"keep", "res"}, {"n", n}});
    kernels.push_back(run_kernel_json(rr.id, rr.kernel, rr.bindings, "res"));
  }
  // DG differentiation (the B200 catalog's dg_diff, ps_catalog.cpp
  // make_dg_diff; the reference has no DG generator): every variant computes
  // res[m,k,i] = sum_j diff_mat[m,i,j] u[k,j] (dmPFtrans: u and res with the
  // element index last). The staged variants are not functional under
  // run_reference, so all four are pinned to the untiled source kernel, as
  // the matmul PF case above; seed-pattern inputs keep every sum exact.
  for (const auto& [nel, np] : std::vector<std::pair<std::string, std::string>>{
           {"32", "16"}, {"48", "32"}}) {
    const std::map<std::string, long long> b{{"nel", std::stoll(nel)}, {"np", std::stoll(np)}};
    for (const std::string v : {"noPF", "uPF", "dmPF", "dmPFtrans"}) {
      const bool trans = v == "dmPFtrans";
      Kernel src = make_kernel(
          "{[m,k,i,j]: 0<=m<3 and 0<=k<nel and 0<=i,j<np}",
          {trans ? "res[m,i,k] = sum(j, diff_mat[m,i,j]*u[j,k])"
                 : "res[m,k,i] = sum(j, diff_mat[m,i,j]*u[k,j])"},
          {{"diff_mat", Dtype::float32, {"3", "np", "np"}},
           {"u", Dtype::float32, trans ? std::vector<std::string>{"np", "nel"}
                                       : std::vector<std::string>{"nel", "np"}},
           {"res", Dtype::float32, trans ? std::vector<std::string>{"3", "np", "nel"}
                                         : std::vector<std::string>{"3", "nel", "np"}}});
      const std::string id = "dg_diff__dtype-float32__nelements-" + nel +
                             "__nmatrices-3__nunit_nodes-" + np + "__variant-" + v;
      kernels.push_back(run_kernel_json(id, src, b, "res"));
    }
  }
  root["kernels"] = kernels;

  // ---- 2./3. counts and features over the whole built-in catalog ----------
  KernelCollection coll(builtin_generators());
  std::vector<GeneratedKernel> all = coll.generate(FilterTagSet::parse({}));
  std::vector<FeatureSpec> specs;
  for (const auto& id : kFeatureIds) specs.push_back(parse_feature(id));
  json counts = json::object(), feats = json::object();
  for (const auto& g : all) {
    KernelCounts c = analyze(g.kernel);
    counts[g.id] = counts_json(c, g.bindings);
    json fv = json::object();
    for (size_t i = 0; i < specs.size(); ++i) {
      try {
        fv[kFeatureIds[i]] = evaluate_feature(specs[i], g.kernel, g.bindings).numeric;
      } catch (const Error& e) {
        fv[kFeatureIds[i]] = std::string("error: ") + e.what();
      }
    }
    feats[g.id] = fv;
  }
  root["catalog_ids"] = [&] {
    json ids = json::array();
    for (const auto& g : all) ids.push_back(g.id);
    return ids;
  }();
  root["counts"] = counts;
  root["features"] = feats;

  // ---- 4. fits on canned problems -----------------------------------------
  json fits = json::array();
  auto fit_case = [&](const std::string& name, const Model& m, const CalibrationProblem& p,
                      bool scale) {
    json j;
    j["name"] = name;
    j["output"] = m.output_id;
    j["expression"] = m.expr_src;
    json rows = json::array();
    for (const auto& r : p.rows) rows.push_back({{"features", r.features}, {"output", r.output}});
    j["rows"] = rows;
    j["scaled"] = scale;
    try {
      CalibratedModel cm = fit_model(m, scale ? scale_features_by_output(p) : p);
      std::vector<double> pv = cm.param_vector();
      j["params"] = pv;
      j["residual_norm"] = cm.residual_norm;
      j["iterations"] = cm.iterations;
      j["converged"] = cm.converged;
      j["warnings"] = cm.warnings;
    } catch (const Error& e) {
      j["error"] = e.what();
    }
    fits.push_back(j);
  };
  {
    Model m = parse_model("f_exec_wall_time_d",
                          "p_a * f_op_float32_madd + p_b * f_thread_groups + p_c * "
                          "f_sync_kernel_launch");
    std::mt19937_64 rng(17);
    std::uniform_real_distribution<double> dist(1.0, 100.0);
    std::normal_distribution<double> noise(0.0, 0.02);
    CalibrationProblem prob;
    for (int r = 0; r < 20; ++r) {
      double f0 = dist(rng) * 1e6, f1 = dist(rng) * 10, f2 = 1.0;
      double t = (3.25e-9 * f0 + 1.5e-6 * f1 + 2e-4 * f2) * (1.0 + noise(rng));
      prob.rows.push_back(CalibrationRow{{f0, f1, f2}, t});
    }
    fit_case("linear3_noisy_scaled", m, prob, true);
    fit_case("linear3_noisy_unscaled", m, prob, false);
  }
  {
    Model m = parse_model(
        "f_exec_wall_time_synthetic_dev",
        "p_launch * f_sync_kernel_launch + "
        "(p_g * f_mem_access_global_float32) * "
        "sstep(p_g * f_mem_access_global_float32 - p_o * f_mem_access_local_float32; p_edge) + "
        "(p_o * f_mem_access_local_float32) * "
        "sstep(p_o * f_mem_access_local_float32 - p_g * f_mem_access_global_float32; p_edge)");
    for (int seed : {5, 6, 7}) {
      std::mt19937_64 rng(seed);
      std::uniform_real_distribution<double> dist(0.5, 2.0);
      CalibrationProblem prob;
      for (int r = 0; r < 24; ++r) {
        double fg = dist(rng) * 10, fl = dist(rng) * 10;
        double cg = 3e-3 * fg, co = 1e-3 * fl;
        prob.rows.push_back(CalibrationRow{{1.0, fg, fl}, 1e-4 + std::max(cg, co)});
      }
      fit_case("overlap_seed" + std::to_string(seed), m, prob, seed != 7);
    }
  }
  {
    Model m = parse_model("f_exec_wall_time_d", "p_a * f_thread_groups + p_b");
    CalibrationProblem prob;
    for (int i = 1; i <= 4; ++i)
      prob.rows.push_back(CalibrationRow{{static_cast<double>(i)}, 10.0 - 2.0 * i});
    fit_case("negative_param", m, prob, false);
    CalibrationProblem one;
    one.rows.push_back(CalibrationRow{{1.0}, 2.0});
    fit_case("rank_deficient", m, one, false);
  }
  root["fits"] = fits;

  std::cout << root.dump(1) << "\n";
  return 0;
}
