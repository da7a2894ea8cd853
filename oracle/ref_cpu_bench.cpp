// TEST/BASELINE INFRASTRUCTURE ONLY. CPU timing of the UNMODIFIED reference
// library (oracle/_ref/libperfseer_ref.a, built from /root/reference/proj/src
// by oracle/Makefile) on the host cores — the `cpu_baseline` of kind
// "reference" for the modelling half of the path:
//   analyze               counting.cpp:217-252 (uncached), kernels/s
//   gather_feature_values features.cpp:417-493 (count cache + JSON hash), rows/s
//   fit_model             model.cpp:485-606 on the matmul calibration rows, fits/s
//   predict               model.cpp:615-623 at seeded C5 matmul points (n in
//                         16Z within [512, 8192], PF/noPF), evals/s on 1 thread
//                         and on T std::threads (the count cache is shared)
// usage: ref_cpu_bench [seconds_per_section=2] [threads=hardware]
//        ref_cpu_bench --fits problems.json [threads=hardware]
//   the second form runs fit_model on caller-given problems (bench.py: every
//   model of the round on its measured calibration rows, output-scaled as in
//   model.cpp:421-435) once on one thread and once spread over T threads,
//   and prints the fitted parameters (to pin K17's reference mode against the
//   reference library itself) with both timings.
// prints one JSON object.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <random>
#include <thread>
#include <vector>

#include <fstream>
#include <sstream>

#include "json.hpp"
#include "perfseer/counting.hpp"
#include "perfseer/features.hpp"
#include "perfseer/model.hpp"
#include "perfseer/uipick.hpp"

using namespace perfseer;
using Clock = std::chrono::steady_clock;

namespace {

double secs(Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); }

const char* kOut = "f_exec_wall_time_cuda_b200_0";
const char* kExpr =
    "p_launch * f_sync_kernel_launch + p_group * f_thread_groups + p_madd * f_op_float32_madd"
    " + p_l * f_mem_access_local_float32 + p_pfa * f_mem_access_tag:mm-PF-a"
    " + p_pfb * f_mem_access_tag:mm-PF-b + p_nopfa * f_mem_access_tag:mm-noPF-a"
    " + p_nopfb * f_mem_access_tag:mm-noPF-b";

}  // namespace

static int run_fits(const char* path, int threads) {
  std::ifstream in(path);
  std::stringstream ss;
  ss << in.rdbuf();
  const auto doc = nlohmann::json::parse(ss.str());
  std::vector<Model> models;
  std::vector<CalibrationProblem> probs;
  for (const auto& p : doc.at("problems")) {
    models.push_back(parse_model_file(p.at("model").get<std::string>()));
    CalibrationProblem cp;
    const auto f = p.at("features").get<std::vector<std::vector<double>>>();
    const auto t = p.at("t").get<std::vector<double>>();
    for (size_t k = 0; k < t.size(); ++k) cp.rows.push_back(CalibrationRow{f[k], t[k]});
    probs.push_back(p.value("scale", true) ? scale_features_by_output(cp) : cp);
  }
  const size_t n = probs.size();
  std::vector<std::vector<double>> params(n);
  std::vector<std::string> errors(n);
  auto fit_one = [&](size_t i) {
    try {
      params[i] = fit_model(models[i], probs[i]).param_vector();
    } catch (const std::exception& e) {
      errors[i] = e.what();
    }
  };
  auto t0 = Clock::now();
  for (size_t i = 0; i < n; ++i) fit_one(i);
  const double one = secs(t0);
  t0 = Clock::now();
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&, t] {
      for (size_t i = size_t(t); i < n; i += size_t(threads)) fit_one(i);
    });
  for (auto& th : pool) th.join();
  const double many = secs(t0);
  nlohmann::json out;
  out["kind"] = "reference";
  out["library"] = "oracle/_ref/libperfseer_ref.a (unmodified /root/reference/proj/src)";
  out["fits"] = n;
  out["seconds_1thread"] = one;
  out["threads"] = threads;
  out["seconds_threads"] = many;
  nlohmann::json ps = nlohmann::json::array();
  for (size_t i = 0; i < n; ++i) {
    if (!errors[i].empty()) {
      ps.push_back(errors[i]);
      continue;
    }
    nlohmann::json v = nlohmann::json::array();
    for (double x : params[i]) {  // exact bits as hex so nothing is lost in printing
      uint64_t b;
      std::memcpy(&b, &x, sizeof b);
      char buf[24];
      std::snprintf(buf, sizeof buf, "%016llx", (unsigned long long)b);
      v.push_back(buf);
    }
    ps.push_back(v);
  }
  out["params_hex"] = ps;
  std::printf("%s\n", out.dump().c_str());
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 2 && std::string(argv[1]) == "--fits")
    return run_fits(argv[2], argc > 3 ? std::atoi(argv[3]) : std::max(1u, std::thread::hardware_concurrency()));
  const double budget = argc > 1 ? std::atof(argv[1]) : 2.0;
  const int threads = argc > 2 ? std::atoi(argv[2]) : std::max(1u, std::thread::hardware_concurrency());

  const auto all = KernelCollection(builtin_generators()).generate(FilterTagSet::parse({}));
  const auto mm = KernelCollection(builtin_generators())
                      .generate(FilterTagSet::parse({"matmul_sq", "dtype:float32"}));
  const Model model = parse_model(kOut, kExpr);

  // analyze, uncached
  size_t analyzed = 0;
  auto t0 = Clock::now();
  while (secs(t0) < budget)
    for (const auto& g : all) {
      volatile size_t n = analyze(g.kernel).accesses.size();
      (void)n;
      ++analyzed;
    }
  const double analyze_rate = analyzed / secs(t0);

  // gather_feature_values (through the reference's cached, hashed path)
  std::vector<KernelInstance> inst;
  for (const auto& g : mm) inst.push_back(KernelInstance{g.id, g.kernel, g.bindings});
  size_t rows = 0;
  t0 = Clock::now();
  FeatureTable table;
  while (secs(t0) < budget) {
    table = gather_feature_values(model.features, inst);
    rows += inst.size();
  }
  const double gather_rate = rows / secs(t0);

  // fit_model: synthetic times from fixed costs with 1% deterministic jitter
  const std::vector<double> truth{5e-6, 6e-11, 1.4e-12, 2.4e-12, 3.5e-13, 3.2e-13, 3.7e-12, 1.5e-13};
  CalibrationProblem prob;
  std::mt19937_64 rng(7);
  std::normal_distribution<double> nd(0.0, 0.01);
  for (const auto& r : table.values) {
    CalibrationRow row;
    row.features = r;
    row.output = eval_model(model, truth, r) * std::exp(nd(rng));
    prob.rows.push_back(row);
  }
  const CalibrationProblem scaled = scale_features_by_output(prob);
  size_t fits = 0;
  t0 = Clock::now();
  CalibratedModel cm;
  while (secs(t0) < budget) {
    cm = fit_model(model, scaled);
    ++fits;
  }
  const double fit_rate = fits / secs(t0);

  // predict at seeded C5 points
  std::vector<std::pair<const GeneratedKernel*, long long>> pts;
  std::mt19937_64 prng(7);
  for (int i = 0; i < 100000; ++i)
    pts.push_back({&mm[i % mm.size()], 16 * (512 / 16 + static_cast<long long>(prng() % (8192 / 16 - 512 / 16 + 1)))});
  auto run = [&](size_t lo, size_t step, double until, size_t* done, double* sink) {
    const auto start = Clock::now();
    size_t k = 0;
    double acc = 0;
    for (size_t i = lo; secs(start) < until; i += step) {
      const auto& [g, n] = pts[i % pts.size()];
      acc += predict(cm, g->kernel, {{"n", n}});
      ++k;
    }
    *done = k;
    *sink = acc;
  };
  size_t one = 0;
  double sink = 0;
  t0 = Clock::now();
  run(0, 1, budget, &one, &sink);
  const double predict_rate_1 = one / secs(t0);
  std::vector<size_t> done(threads);
  std::vector<double> sinks(threads);
  std::vector<std::thread> pool;
  t0 = Clock::now();
  for (int t = 0; t < threads; ++t) pool.emplace_back(run, t, threads, budget, &done[t], &sinks[t]);
  for (auto& th : pool) th.join();
  size_t total = 0;
  for (size_t d : done) total += d;
  const double predict_rate_n = total / secs(t0);

  std::printf(
      "{\"kind\": \"reference\", \"library\": \"oracle/_ref/libperfseer_ref.a (unmodified "
      "/root/reference/proj/src)\", \"threads\": %d, \"catalog_kernels\": %zu, "
      "\"analyze_kernels_per_s\": %.1f, \"gather_rows_per_s\": %.1f, \"fit_rows\": %zu, "
      "\"fit_params\": %zu, \"fits_per_s\": %.2f, \"predict_evals_per_s_1thread\": %.1f, "
      "\"predict_evals_per_s\": %.1f, \"predict_sample\": \"matmul PF/noPF at seeded n in 16Z within "
      "[512, 8192], %.1f s per section\"}\n",
      threads, all.size(), analyze_rate, gather_rate, prob.rows.size(), model.params.size(), fit_rate,
      predict_rate_1, predict_rate_n, budget);
  return sink == 12345.678 ? 1 : 0;
}
