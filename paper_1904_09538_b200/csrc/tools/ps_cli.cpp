// `perfseer` command line over the B200 port: the reference's six-stage
// pipeline (SPEC.md "MODULE cli"; subcommand surface of the reference
// tools/perfseer.cpp:475-583) with the B200 executor as a measurement device.
//
//   count      symbolic counts of one kernel (+ values at --bind)
//   generate   expand catalog kernels from filter tags into a directory
//   measure    time a kernel directory on --device (synthetic spec JSON, or
//              cuda:<N>[,<N>...] for the sm_100a executor behind ps_measure,
//              one host thread and context per GPU, LPT-sharded)
//   features   evaluate a model's input features over a kernel directory
//   calibrate  fit a model to a feature table + measurement CSV
//   predict    predicted seconds for one kernel or a directory
//   report     per-variant series, geomean errors, rankings, overlap class
//
// Stage files keep the reference formats (kernel JSON perfseer-kernel/1,
// measurement/feature/prediction CSV, calibrated-model JSON, manifests), so a
// pipeline may mix stages run by either tool. Errors exit 1 with
// "error: <message>"; a measure run with failing kernels writes the rest,
// lists the failures in the CSV header and exits 2.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <optional>
#include <thread>
#include <memory>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "../../../include/perfseer_b200.h"
#include "json.hpp"
#include "ps_catalog.hpp"
#include "ps_counting.hpp"
#include "ps_errors.hpp"
#include "ps_executor.hpp"
#include "ps_features.hpp"
#include "ps_json.hpp"
#include "ps_lang.hpp"
#include "ps_manifest.hpp"
#include "ps_model.hpp"

namespace fs = std::filesystem;
using nlohmann::json;
using namespace perfseer;

namespace {

// ---------------------------------------------------------------------------
// argument handling: "--name value" options (repeatable) and bare flags

struct Spec {
  std::set<std::string> valued, flags, required;
};

struct Args {
  std::map<std::string, std::vector<std::string>> values;
  std::set<std::string> flags;

  bool has(const std::string& k) const { return values.count(k) || flags.count(k); }
  std::string one(const std::string& k, const std::string& dflt = "") const {
    auto it = values.find(k);
    return it == values.end() ? dflt : it->second.back();
  }
  std::vector<std::string> all(const std::string& k) const {
    auto it = values.find(k);
    return it == values.end() ? std::vector<std::string>{} : it->second;
  }
};

Args parse_args(const std::vector<std::string>& argv, const Spec& spec) {
  Args a;
  for (size_t i = 0; i < argv.size(); ++i) {
    std::string key = argv[i], val;
    if (key.rfind("--", 0) != 0) throw Error("unexpected argument '" + key + "'");
    const size_t eq = key.find('=');
    const bool inline_val = eq != std::string::npos;
    if (inline_val) {
      val = key.substr(eq + 1);
      key = key.substr(0, eq);
    }
    key = key.substr(2);
    if (spec.flags.count(key) && !inline_val) {
      a.flags.insert(key);
    } else if (spec.valued.count(key)) {
      if (!inline_val) {
        if (i + 1 >= argv.size()) throw Error("--" + key + " needs a value");
        val = argv[++i];
      }
      a.values[key].push_back(val);
    } else {
      throw Error("unknown option --" + key);
    }
  }
  for (const auto& r : spec.required)
    if (!a.has(r)) throw Error("--" + r + " is required");
  return a;
}

struct Globals {
  long long seed = 0;
  bool seed_given = false;
  int sub_group_size = 32;
};

// ---------------------------------------------------------------------------
// files

std::string slurp(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw Error("cannot open " + path);
  std::stringstream ss;
  ss << f.rdbuf();
  return ss.str();
}

void spit(const std::string& path, const std::string& text) {
  const fs::path p(path);
  if (!p.parent_path().empty()) fs::create_directories(p.parent_path());
  std::ofstream f(path, std::ios::binary);
  if (!f) throw Error("cannot write " + path);
  f << text;
}

std::string hash_of(const std::string& path) { return file_hash_hex(slurp(path)); }

std::string g17(double v) {
  char b[40];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}

std::map<std::string, long long> bindings_of(const std::vector<std::string>& items) {
  std::map<std::string, long long> env;
  for (const auto& it : items) {
    const size_t eq = it.find('=');
    if (eq == std::string::npos) throw Error("binding must be name=value: " + it);
    env[it.substr(0, eq)] = std::stoll(it.substr(eq + 1));
  }
  return env;
}

// A kernel file is either kernel JSON or the text front end (lang.cpp).
Kernel read_kernel(const std::string& path) {
  const std::string text = slurp(path);
  if (fs::path(path).extension() == ".json") return kernel_from_json(json::parse(text));
  return parse_kernel_text(text, fs::path(path).stem().string());
}

// A `generate` output directory: manifest.json lists id, file, bindings.
struct KernelDir {
  json manifest;
  std::vector<KernelInstance> kernels;
};

KernelDir read_kernel_dir(const std::string& dir) {
  const fs::path mf = fs::path(dir) / "manifest.json";
  if (!fs::exists(mf)) throw Error("no manifest.json in " + dir);
  KernelDir d;
  d.manifest = json::parse(slurp(mf.string()));
  for (const auto& e : d.manifest.at("kernels")) {
    KernelInstance ki;
    ki.id = e.at("id").get<std::string>();
    ki.kernel = kernel_from_json(json::parse(slurp((fs::path(dir) / e.at("file").get<std::string>()).string())));
    for (auto it = e.at("bindings").begin(); it != e.at("bindings").end(); ++it)
      ki.bindings[it.key()] = it.value().get<long long>();
    d.kernels.push_back(std::move(ki));
  }
  return d;
}

// ---------------------------------------------------------------------------
// count

json exact_value(const Poly& p, const std::map<std::string, long long>& env, bool& ok) {
  if (!ok) return nullptr;
  try {
    const Rational v = p.eval(env);
    return json{{"num", numerator(v).str()}, {"den", denominator(v).str()}};
  } catch (const Error&) {
    ok = false;  // an unbound symbol: the remaining values are not evaluated
    return nullptr;
  }
}

json count_map_json(const KernelCounts& c, const std::map<std::string, long long>& env, int sgs) {
  bool ok = true;
  json out;
  json ops = json::array();
  for (const auto& e : c.ops)
    ops.push_back({{"dtype", dtype_str(e.kind.dtype)},
                   {"op", opname_str(e.kind.op)},
                   {"granularity", granularity_str(e.kind.gran)},
                   {"count", e.count.str()},
                   {"value", exact_value(e.count, env, ok)}});
  out["ops"] = ops;
  json acc = json::array();
  for (const auto& e : c.accesses)
    acc.push_back({{"pattern", e.pattern.key()},
                   {"granularity", granularity_str(e.pattern.gran)},
                   {"afr", e.pattern.afr.str()},
                   {"count", e.count.str()},
                   {"value", exact_value(e.count, env, ok)}});
  out["accesses"] = acc;
  json sync = json::object();
  for (const auto& e : c.sync)
    sync[synckind_str(e.kind)] = {{"count", e.count.str()}, {"value", exact_value(e.count, env, ok)}};
  out["sync"] = sync;
  json fp = json::object();
  for (const auto& [arr, p] : c.footprints) fp[arr] = {{"count", p.str()}, {"value", exact_value(p, env, ok)}};
  out["footprints"] = fp;
  if (c.geometry) {
    json groups = json::array();
    for (const auto& p : c.geometry->num_groups)
      groups.push_back({{"count", p.str()}, {"value", exact_value(p, env, ok)}});
    out["geometry"] = {{"work_group_size", c.geometry->work_group_size},
                       {"num_groups", groups},
                       {"sub_group_size", sgs}};
  }
  return out;
}

int run_count(const Args& a, const Globals& g) {
  const std::string path = a.one("kernel");
  const Kernel k = read_kernel(path);
  json j = count_map_json(analyze(k), bindings_of(a.all("bind")), g.sub_group_size);
  j["kernel"] = k.name;
  j["manifest"] = make_manifest("count", {{"kernel", hash_of(path)}}, g.seed).to_json();
  const std::string text = j.dump(2) + "\n";
  if (a.has("out"))
    spit(a.one("out"), text);
  else
    std::cout << text;
  return 0;
}

// ---------------------------------------------------------------------------
// generate

std::vector<std::string> tag_lines(const std::string& text) {
  std::vector<std::string> out;
  std::istringstream in(text);
  for (std::string line; std::getline(in, line);) {
    line.erase(line.find_last_not_of(" \r") + 1);
    if (!line.empty() && line.front() != '#') out.push_back(line);
  }
  return out;
}

int run_generate(const Args& a, const Globals& g) {
  std::vector<std::string> tags = a.all("tag");
  std::map<std::string, std::string> hashes;
  if (a.has("tags")) {
    const std::string text = slurp(a.one("tags"));
    hashes["tags"] = file_hash_hex(text);
    for (auto& t : tag_lines(text)) tags.push_back(std::move(t));
  }
  const std::string which = a.one("catalog", "reference");
  if (which != "reference" && which != "b200") throw Error("--catalog must be reference or b200");
  const std::string match = a.one("match", "superset");
  const KernelCollection coll(which == "b200" ? b200_generators() : builtin_generators());
  const auto kernels = coll.generate(FilterTagSet::parse(tags), match_condition_from_str(match));
  if (kernels.empty()) std::cerr << "warning: no generators matched the tag set\n";

  const fs::path dir(a.one("out"));
  json list = json::array();
  for (const auto& gk : kernels) {
    const std::string file = gk.id + ".json";
    spit((dir / file).string(), kernel_to_json(gk.kernel).dump(2) + "\n");
    json args = json::object(), binds = json::object();
    for (const auto& [k, v] : gk.args) args[k] = v;
    for (const auto& [k, v] : gk.bindings) binds[k] = v;
    list.push_back({{"id", gk.id}, {"file", file}, {"generator", gk.generator}, {"args", args},
                    {"bindings", binds}, {"work_group_size", gk.geometry.work_group_size}});
  }
  json m;
  m["manifest"] = make_manifest("generate", hashes, g.seed).to_json();
  m["tags"] = tags;
  m["match"] = match;
  m["kernels"] = list;
  spit((dir / "manifest.json").string(), m.dump(2) + "\n");
  std::cout << "generated " << kernels.size() << " kernels into " << dir.string() << "\n";
  return 0;
}

// ---------------------------------------------------------------------------
// measure: a synthetic device spec (the reference's CPU test double) or the
// B200 executor ("cuda:<N>")

// Estimated seconds of one trial of a catalog kernel (for sharding only).
double estimate_seconds(const std::string& id) {
  ps_kernel_desc d;
  ps_io_info io;
  if (ps_desc_from_id(id.c_str(), &d) != PS_OK || ps_kernel_io(&d, &io) != PS_OK) return 1e-5;
  return io.bytes_global / 6.0e12 + io.flops / 30e12 + io.bytes_shared / 30e12 + 4e-6;
}

// `--device cuda:0,1,...`: one CudaExecutor (one ps_ctx) per GPU, each driven
// by its own host thread (ABI threading contract: one context per GPU, not
// reentrant); kernels are LPT-balanced over the GPUs on their estimated time,
// and the records are merged back into directory order.
std::vector<int> cuda_devices(const std::string& dev) {
  std::vector<int> out;
  std::stringstream ss(dev.substr(5));
  for (std::string tok; std::getline(ss, tok, ',');) out.push_back(std::stoi(tok));
  if (out.empty()) throw Error("--device cuda:<N>[,<N>...] lists no device");
  return out;
}

int run_measure(const Args& a, const Globals& g) {
  const std::string dev = a.one("device");
  const int trials = std::stoi(a.one("trials", "60"));
  std::map<std::string, std::string> hashes;
  const KernelDir kd = read_kernel_dir(a.one("kernels"));
  const size_t nk = kd.kernels.size();
  std::vector<std::optional<MeasurementRecord>> recs(nk);
  std::vector<std::string> errs(nk);
  std::string dev_id;
  if (dev.rfind("cuda:", 0) == 0) {
    const int warmup = std::stoi(a.one("warmup", "5"));
    const std::vector<int> gpus = cuda_devices(dev);
    hashes["device"] = file_hash_hex(dev);
    // LPT: longest first onto the least-loaded GPU
    std::vector<size_t> order(nk);
    for (size_t i = 0; i < nk; ++i) order[i] = i;
    std::vector<double> est(nk);
    for (size_t i = 0; i < nk; ++i) est[i] = estimate_seconds(kd.kernels[i].id);
    std::stable_sort(order.begin(), order.end(), [&](size_t x, size_t y) { return est[x] > est[y]; });
    std::vector<std::vector<size_t>> shard(gpus.size());
    std::vector<double> load(gpus.size(), 0.0);
    for (size_t i : order) {
      const size_t r = std::min_element(load.begin(), load.end()) - load.begin();
      shard[r].push_back(i);
      load[r] += est[i];
    }
    std::vector<std::string> ids(gpus.size());
    std::vector<std::string> init_err(gpus.size());
    std::vector<std::thread> pool;
    for (size_t r = 0; r < gpus.size(); ++r)
      pool.emplace_back([&, r] {
        try {
          CudaExecutor ex(gpus[r], warmup);
          ids[r] = ex.id();
          for (size_t i : shard[r]) {
            const auto& ki = kd.kernels[i];
            try {
              MeasurementRecord rec = measure_kernel(ex, ki.kernel, ki.bindings, trials);
              rec.kernel_id = ki.id;
              recs[i] = std::move(rec);
            } catch (const std::exception& e) {
              errs[i] = ki.id + ": " + e.what();
            }
          }
        } catch (const std::exception& e) {
          init_err[r] = e.what();
          for (size_t i : shard[r]) errs[i] = kd.kernels[i].id + ": " + e.what();
        }
      });
    for (auto& t : pool) t.join();
    for (size_t r = 0; r < gpus.size(); ++r) dev_id += (r ? "+" : "") + (ids[r].empty() ? "cuda_b200_?" : ids[r]);
  } else {
    SyntheticDeviceSpec spec = SyntheticDeviceSpec::from_json_string(slurp(dev));
    if (g.seed_given) spec.seed = static_cast<uint64_t>(g.seed);
    SyntheticDevice ex(spec);
    hashes["device"] = hash_of(dev);
    dev_id = ex.id();
    for (size_t i = 0; i < nk; ++i) {
      const auto& ki = kd.kernels[i];
      try {
        MeasurementRecord rec = measure_kernel(ex, ki.kernel, ki.bindings, trials);
        rec.kernel_id = ki.id;
        recs[i] = std::move(rec);
      } catch (const Error& e) {
        errs[i] = ki.id + ": " + e.what();
      }
    }
  }
  std::vector<MeasurementRecord> ok;
  std::vector<std::string> failures;
  for (size_t i = 0; i < nk; ++i) {
    if (recs[i]) ok.push_back(std::move(*recs[i]));
    if (!errs[i].empty()) failures.push_back(errs[i]);
  }
  std::string head = make_manifest("measure", hashes, g.seed_given ? g.seed : 0).comment_line() + "\n";
  head += "# device: " + dev_id + ", trials: " + std::to_string(trials) + "\n";
  for (const auto& f : failures) head += "# failed: " + f + "\n";
  spit(a.one("out"), head + measurements_to_csv(ok));
  for (const auto& f : failures) std::cerr << "failed: " << f << "\n";
  return failures.empty() ? 0 : 2;
}

// ---------------------------------------------------------------------------
// features / calibrate / predict

int run_features(const Args& a, const Globals& g) {
  const std::string mpath = a.one("model");
  const Model model = parse_model_file(slurp(mpath));
  const KernelDir kd = read_kernel_dir(a.one("kernels"));
  const FeatureTable t = gather_feature_values(model.features, kd.kernels, nullptr, 60, g.sub_group_size);
  spit(a.one("out"), make_manifest("features", {{"model", hash_of(mpath)}}, g.seed).comment_line() + "\n" +
                         t.to_csv());
  return 0;
}

// Joins measurement rows to feature rows by kernel id, in measurement order;
// a measured kernel without a feature row is skipped.
CalibrationProblem join_rows(const Model& m, const FeatureTable& t,
                             const std::vector<MeasurementRecord>& meas) {
  std::vector<size_t> col;
  for (const auto& fid : m.feature_ids) {
    const auto it = std::find(t.columns.begin(), t.columns.end(), fid);
    if (it == t.columns.end()) throw Error("feature table lacks column " + fid);
    col.push_back(static_cast<size_t>(it - t.columns.begin()));
  }
  std::map<std::string, size_t> row_of;
  for (size_t i = t.row_ids.size(); i-- > 0;) row_of[t.row_ids[i]] = i;  // first occurrence wins
  CalibrationProblem p;
  for (const auto& r : meas) {
    const auto it = row_of.find(r.kernel_id);
    if (it == row_of.end()) continue;
    CalibrationRow row;
    for (size_t c : col) row.features.push_back(t.values[it->second][c]);
    row.output = r.mean_seconds;
    p.rows.push_back(std::move(row));
  }
  if (p.rows.empty()) throw Error("no measurement rows matched the feature table");
  return p;
}

int run_calibrate(const Args& a, const Globals& g) {
  const std::string mpath = a.one("model"), fpath = a.one("features"), tpath = a.one("measurements");
  const Model model = parse_model_file(slurp(mpath));
  const CalibrationProblem raw =
      join_rows(model, FeatureTable::from_csv(slurp(fpath)), measurements_from_csv(slurp(tpath)));
  const bool scaled = !a.has("no-scale");
  FitOptions opt;
  opt.nonnegative = a.has("nonnegative");
  CalibratedModel cm = fit_model(model, scaled ? scale_features_by_output(raw) : raw, opt);
  if (scaled) {  // residual of the fitted model on the unscaled rows
    const auto pv = cm.param_vector();
    double ss = 0.0;
    for (const auto& r : raw.rows) {
      const double d = r.output - eval_model(model, pv, r.features);
      ss += d * d;
    }
    cm.residual_norm_unscaled = std::sqrt(ss);
  }
  cm.measurement_hash = hash_of(tpath);
  json j = json::parse(cm.to_json_string());
  j["manifest"] = make_manifest("calibrate",
                                {{"model", hash_of(mpath)}, {"features", hash_of(fpath)},
                                 {"measurements", cm.measurement_hash}},
                                g.seed)
                      .to_json();
  spit(a.one("out"), j.dump(2) + "\n");
  for (const auto& w : cm.warnings) std::cerr << "warning: " << w << "\n";
  std::cout << "residual_norm " << g17(cm.residual_norm) << ", iterations " << cm.iterations
            << (cm.converged ? ", converged" : ", not converged") << "\n";
  return 0;
}

int run_predict(const Args& a, const Globals& g) {
  const std::string mpath = a.one("model");
  const CalibratedModel cm = CalibratedModel::from_json_string(slurp(mpath));
  if (a.has("kernel")) {
    const double t = predict(cm, read_kernel(a.one("kernel")), bindings_of(a.all("bind")), g.sub_group_size);
    std::cout << g17(t) << "\n";
    return 0;
  }
  if (!a.has("kernels")) throw Error("predict needs --kernel or --kernels");
  const KernelDir kd = read_kernel_dir(a.one("kernels"));
  std::ostringstream os;
  os.precision(17);
  os << make_manifest("predict", {{"model", hash_of(mpath)}}, g.seed).comment_line() << "\n"
     << "kernel,bindings,predicted_seconds\n";
  for (const auto& ki : kd.kernels)
    os << ki.id << "," << bindings_str(ki.bindings) << ","
       << predict(cm, ki.kernel, ki.bindings, g.sub_group_size) << "\n";
  spit(a.one("out", "predictions.csv"), os.str());
  return 0;
}

// ---------------------------------------------------------------------------
// report

std::map<std::string, double> read_predictions(const std::string& text) {
  std::map<std::string, double> out;
  std::istringstream in(text);
  bool header_seen = false;
  for (std::string line; std::getline(in, line);) {
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (line.empty() || line.front() == '#') continue;
    if (!header_seen) {
      header_seen = true;
      continue;
    }
    // kernel,bindings,predicted_seconds (bindings never contain ',')
    std::vector<std::string> cells;
    std::istringstream ls(line);
    for (std::string c; std::getline(ls, c, ',');) cells.push_back(c);
    if (cells.size() < 3) throw Error("malformed prediction CSV line: " + line);
    out[cells[0]] = std::stod(cells[2]);
  }
  return out;
}

int run_report(const Args& a, const Globals& g) {
  const std::string mp = a.one("measured"), pp = a.one("predicted");
  const auto meas = measurements_from_csv(slurp(mp));
  const auto pred = read_predictions(slurp(pp));
  const json gen = json::parse(slurp(a.one("manifest")));

  // variant = generator + non-size args; size = the ladder args
  static const std::set<std::string> kSizeArgs{"n", "nelements", "m", "num_groups"};
  std::map<std::string, std::pair<std::string, std::string>> vs_of;
  for (const auto& e : gen.at("kernels")) {
    std::string variant = e.value("generator", "?"), size;
    for (auto it = e.at("args").begin(); it != e.at("args").end(); ++it) {
      const std::string v = it.value().get<std::string>();
      if (kSizeArgs.count(it.key()))
        size += (size.empty() ? "" : ";") + it.key() + "=" + v;
      else
        variant += "_" + it.key() + "-" + v;
    }
    vs_of[e.at("id").get<std::string>()] = {variant, size.empty() ? "-" : size};
  }
  struct Point {
    std::string variant, size;
    double measured, predicted;
  };
  std::vector<Point> pts;
  for (const auto& r : meas) {
    const auto p = pred.find(r.kernel_id);
    if (p == pred.end()) throw Error("prediction missing for kernel " + r.kernel_id);
    const auto v = vs_of.find(r.kernel_id);
    pts.push_back(v == vs_of.end() ? Point{r.kernel_id, bindings_str(r.bindings), r.mean_seconds, p->second}
                                   : Point{v->second.first, v->second.second, r.mean_seconds, p->second});
  }
  const std::string stamp =
      make_manifest("report", {{"measured", hash_of(mp)}, {"predicted", hash_of(pp)}}, g.seed).comment_line() +
      "\n";
  const fs::path out(a.one("out"));

  std::ostringstream series;
  series.precision(17);
  series << stamp << "variant,size,measured_seconds,predicted_seconds\n";
  for (const auto& p : pts) series << p.variant << "," << p.size << "," << p.measured << "," << p.predicted << "\n";
  spit((out / "series.csv").string(), series.str());

  std::map<std::string, std::pair<std::vector<double>, std::vector<double>>> per_variant;
  std::vector<double> ap, am;
  for (const auto& p : pts) {
    per_variant[p.variant].first.push_back(p.predicted);
    per_variant[p.variant].second.push_back(p.measured);
    ap.push_back(p.predicted);
    am.push_back(p.measured);
  }
  std::ostringstream summary;
  summary.precision(17);
  summary << stamp << "variant,geo_mean_rel_error\n";
  for (const auto& [v, pm] : per_variant) summary << v << "," << geo_mean_rel_error(pm.first, pm.second) << "\n";
  summary << "overall," << geo_mean_rel_error(ap, am) << "\n";
  if (a.has("full-time")) {
    const CombineKind k = classify_overlap(std::stod(a.one("full-time")), std::stod(a.one("removed-time", "0")),
                                           std::stod(a.one("onchip-est", "0")));
    summary << "overlap_diagnosis," << (k == CombineKind::linear ? "linear" : "max_overlap") << "\n";
  }
  spit((out / "summary.csv").string(), summary.str());

  // winner per size: strict '<', first minimum in measurement order
  std::map<std::string, std::vector<const Point*>> by_size;
  for (const auto& p : pts) by_size[p.size].push_back(&p);
  std::ostringstream rank;
  rank << stamp << "size,measured_winner,predicted_winner,correct\n";
  for (const auto& [size, group] : by_size) {
    if (group.size() < 2) continue;
    const Point *mw = group.front(), *pw = group.front();
    for (const Point* p : group) {
      if (p->measured < mw->measured) mw = p;
      if (p->predicted < pw->predicted) pw = p;
    }
    rank << size << "," << mw->variant << "," << pw->variant << "," << (mw->variant == pw->variant ? "yes" : "no")
         << "\n";
  }
  spit((out / "ranking.csv").string(), rank.str());
  return 0;
}

// ---------------------------------------------------------------------------

struct Command {
  const char* name;
  const char* help;
  Spec spec;
  std::function<int(const Args&, const Globals&)> run;
};

const std::vector<Command>& commands() {
  static const std::vector<Command> cmds = {
      {"count", "symbolic operation/access/sync counts", {{"kernel", "bind", "out"}, {}, {"kernel"}}, run_count},
      {"generate",
       "expand measurement kernels from filter tags",
       {{"tag", "tags", "match", "out", "catalog"}, {}, {"out"}},
       run_generate},
      {"measure",
       "run kernels on an executor (synthetic spec JSON or cuda:<N>[,<N>...])",
       {{"device", "kernels", "trials", "warmup", "out"}, {}, {"device", "kernels", "out"}},
       run_measure},
      {"features",
       "evaluate model input features",
       {{"model", "kernels", "out"}, {}, {"model", "kernels", "out"}},
       run_features},
      {"calibrate",
       "fit model parameters",
       {{"model", "features", "measurements", "out"},
        {"no-scale", "nonnegative"},
        {"model", "features", "measurements", "out"}},
       run_calibrate},
      {"predict", "predict execution time", {{"model", "kernel", "bind", "kernels", "out"}, {}, {"model"}}, run_predict},
      {"report",
       "measured-vs-predicted tables and rankings",
       {{"measured", "predicted", "manifest", "out", "full-time", "removed-time", "onchip-est"},
        {},
        {"measured", "predicted", "manifest", "out"}},
       run_report},
  };
  return cmds;
}

void usage(std::ostream& os) {
  os << "usage: perfseer [--seed N] [--sub-group-size N] <command> [options]\n"
     << "       perfseer --version\ncommands:\n";
  for (const auto& c : commands()) os << "  " << c.name << std::string(12 - std::string(c.name).size(), ' ') << c.help << "\n";
}

}  // namespace

int main(int argc, char** argv) {
  Globals g;
  int i = 1;
  try {
    for (; i < argc; ++i) {  // global options precede the subcommand
      const std::string s = argv[i];
      if (s == "--version") {
        std::cout << "perfseer " << kToolVersion << "\n";
        return 0;
      }
      if (s == "--help" || s == "-h") {
        usage(std::cout);
        return 0;
      }
      if (s.rfind("--", 0) != 0) break;
      if (i + 1 >= argc) throw Error(s + " needs a value");
      if (s == "--seed") {
        g.seed = std::stoll(argv[++i]);
        g.seed_given = true;
      } else if (s == "--sub-group-size") {
        g.sub_group_size = std::stoi(argv[++i]);
      } else {
        throw Error("unknown option " + s);
      }
    }
    if (i >= argc) {
      usage(std::cerr);
      return 1;
    }
    const std::string name = argv[i];
    const auto& cmds = commands();
    const auto c = std::find_if(cmds.begin(), cmds.end(), [&](const Command& x) { return name == x.name; });
    if (c == cmds.end()) throw Error("unknown command '" + name + "'");
    // global options may also follow the subcommand
    std::vector<std::string> rest;
    for (int j = i + 1; j < argc; ++j) {
      const std::string s = argv[j];
      if ((s == "--seed" || s == "--sub-group-size") && j + 1 < argc) {
        if (s == "--seed") {
          g.seed = std::stoll(argv[++j]);
          g.seed_given = true;
        } else {
          g.sub_group_size = std::stoi(argv[++j]);
        }
        continue;
      }
      rest.push_back(s);
    }
    return c->run(parse_args(rest, c->spec), g);
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
