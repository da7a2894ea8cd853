// TEST INFRASTRUCTURE ONLY. Counts and feature values of arbitrary kernels
// given as perfseer-kernel/1 JSON — the B200 catalog the bench actually
// fits (DG variants and their ten dg-* work-removed tags, the gmem 18x18
// pattern, the B200 size ladders), which the reference's own generators
// cannot produce. Built twice: against the UNMODIFIED reference library
// (oracle/Makefile -> oracle/_ref/ref_catalog, which writes
// tests/golden/catalog_reference.jsonl) and against the port
// (tests/refapi.mk -> tests/_build/port_ref_catalog); tests/test_catalog_pin.py
// requires the two outputs to be identical line for line.
//
// stdin (JSON lines): first {"features": [feature ids], "sub_group_size": N},
// then one {"id", "kernel", "bindings"} per kernel (host.kernel_json).
// stdout (JSON lines): per kernel {"id", "hash": kernel_hash (kernel_json.cpp:254),
// "counts": analyze (counting.cpp:697-715) at the bindings, "features":
// [evaluate_feature (features.cpp:342-415) numeric value, or "error: <what>"]}.
#include <iostream>
#include <string>

#include "json.hpp"
#include "perfseer/counting.hpp"
#include "perfseer/features.hpp"
#include "perfseer/kernel_json.hpp"

using namespace perfseer;
using nlohmann::json;

static json counts_json(const KernelCounts& c, const std::map<std::string, long long>& b) {
  json j;
  json ops = json::array();
  for (const auto& e : c.ops)
    ops.push_back({e.kind.key(), granularity_str(e.kind.gran), e.count.str(), e.count.eval(b).str()});
  j["ops"] = ops;
  json acc = json::array();
  for (const auto& e : c.accesses)
    acc.push_back({e.pattern.str(), e.count.str(), e.count.eval(b).str(), e.pattern.afr.eval(b).str()});
  j["accesses"] = acc;
  json sync = json::array();
  for (const auto& e : c.sync) sync.push_back({synckind_str(e.kind), e.count.str(), e.count.eval(b).str()});
  j["sync"] = sync;
  json fp = json::object();
  for (const auto& [a, p] : c.footprints) fp[a] = {p.str(), p.eval(b).str()};
  j["footprints"] = fp;
  if (c.geometry) {
    j["work_group_size"] = c.geometry->work_group_size;
    json ng = json::array();
    for (const auto& g : c.geometry->num_groups) ng.push_back(g.str());
    j["num_groups"] = ng;
  }
  return j;
}

int main() {
  std::string line;
  if (!std::getline(std::cin, line)) return 1;
  const json head = json::parse(line);
  std::vector<FeatureSpec> specs;
  for (const auto& f : head.at("features")) specs.push_back(parse_feature(f.get<std::string>()));
  const int sgs = head.value("sub_group_size", 32);
  while (std::getline(std::cin, line)) {
    if (line.empty()) continue;
    const json in = json::parse(line);
    const Kernel k = kernel_from_json(in.at("kernel"));
    const auto b = in.at("bindings").get<std::map<std::string, long long>>();
    json out;
    out["id"] = in.at("id");
    char hash[32];
    std::snprintf(hash, sizeof hash, "%016llx", (unsigned long long)kernel_hash(k));
    out["hash"] = hash;
    out["counts"] = counts_json(analyze(k), b);
    json vals = json::array();
    for (const auto& s : specs) {
      try {
        vals.push_back(evaluate_feature(s, k, b, nullptr, 60, sgs).numeric);
      } catch (const std::exception& e) {
        vals.push_back(std::string("error: ") + e.what());
      }
    }
    out["features"] = vals;
    std::cout << out.dump() << "\n";
  }
  return 0;
}
