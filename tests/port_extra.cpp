// Symbolic counts of this repo's own generators (incl. the DG builders, which
// have no reference) against the enumeration oracle of the port, at small
// admissible sizes. Built and run by tests/test_port_extra.py.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include "doctest.h"

#include <cstdlib>

#include "perfseer/counting.hpp"
#include "perfseer/manifest.hpp"
#include "perfseer/oracle.hpp"
#include "perfseer/uipick.hpp"

using namespace perfseer;

namespace {

long long to_ll(const Poly& p, const std::map<std::string, long long>& b) {
  Rational v = p.eval(b);
  REQUIRE(is_integer(v));
  return numerator(v).convert_to<long long>();
}

void check(const GeneratedKernel& g) {
  const KernelCounts c = analyze(g.kernel);
  const OracleCounts o = brute_force_count(g.kernel, g.bindings, 50'000'000);
  std::map<std::string, long long> ops;
  for (const auto& e : c.ops)
    if (long long v = to_ll(e.count, g.bindings)) ops[e.kind.key()] += v;
  CHECK(ops == o.ops);
  std::map<std::string, long long> acc;
  for (const auto& e : c.accesses) {
    const long long v = to_ll(e.count, g.bindings);
    if (v) acc[evaluate_pattern(e.pattern, g.bindings).key()] += v;
  }
  std::map<std::string, long long> oacc;
  for (const auto& [k, v] : o.access_counts)
    if (v) oacc[k] = v;
  CHECK(acc == oacc);
  for (const auto& [a, p] : c.footprints) CHECK(to_ll(p, g.bindings) == o.footprints.at(a));
  long long bar = 0;
  for (const auto& e : c.sync)
    if (e.kind == SyncKind::barrier_local) bar = to_ll(e.count, g.bindings);
  CHECK(bar == o.barrier_local);
  if (!(ops == o.ops) || !(acc == oacc)) std::fprintf(stderr, "  mismatch in %s\n", g.id.c_str());
}

}  // namespace


TEST_CASE("DG variants and their work-removed kernels: symbolic == enumeration") {
  for (const std::string v : {"noPF", "uPF", "dmPF", "dmPFtrans"}) {
    ArgMap a{{"dtype", "float32"}, {"variant", v}, {"nmatrices", "3"}, {"nunit_nodes", "32"},
             {"nelements", "48"}};
    check(make_dg_diff(a));
    for (const std::string keep : {"u", "dm", "res"}) {
      ArgMap r = a;
      r["keep"] = keep;
      check(make_dg_diff_rm(r));
    }
  }
}

TEST_CASE("pattern microbenchmarks at small sizes: symbolic == enumeration") {
  ArgMap p{{"dtype", "float32"}, {"lsize_0", "16"}, {"lsize_1", "16"}, {"lid_stride_0", "1"},
           {"lid_stride_1", "64"}, {"nelements", "2048"}};
  for (const std::string k : {"1", "2"}) {
    ArgMap a = p;
    a["n_input_arrays"] = k;
    check(make_gmem_pattern(a));
  }
  ArgMap q = p;
  q["m"] = "2";
  check(make_flops_pattern("madd", q));
  check(make_lmem_shuffle(q));
  check(make_overlap_knl(q));
  ArgMap b = q;
  b.erase("dtype");
  check(make_barrier_knl(b));
  ArgMap g18{{"dtype", "float32"}, {"lsize_0", "18"}, {"lsize_1", "18"}, {"lid_stride_0", "1"},
             {"lid_stride_1", "72"}, {"nelements", "2592"}, {"n_input_arrays", "1"}};
  check(make_gmem_pattern(g18));
}

TEST_CASE("applications at small sizes: symbolic == enumeration") {
  for (const std::string pf : {"True", "False"}) {
    ArgMap a{{"dtype", "float32"}, {"prefetch", pf}, {"lsize_0", "16"}, {"lsize_1", "16"},
             {"groups_fit", "True"}, {"n", "48"}};
    check(make_matmul_sq(a));
    for (const std::string keep : {"a", "b"}) {
      ArgMap r = a;
      r["keep"] = keep;
      check(make_matmul_sq_rm(r));
    }
  }
  for (const auto& [tile, n] : std::vector<std::pair<std::string, std::string>>{{"16x16", "28"},
                                                                              {"18x18", "32"}}) {
    ArgMap a{{"dtype", "float32"}, {"tile", tile}, {"n", n}};
    check(make_fd_stencil(a));
    for (const std::string keep : {"u", "res"}) {
      ArgMap r = a;
      r["keep"] = keep;
      check(make_fd_stencil_rm(r));
    }
  }
}

TEST_CASE("every B200 catalog variant id round-trips through kernel_from_variant_id") {
  KernelCollection coll(b200_generators());
  for (const auto& g : coll.generate(FilterTagSet::parse({}))) {
    GeneratedKernel again = kernel_from_variant_id(g.id);
    CHECK(again.kernel == g.kernel);
    CHECK(again.bindings == g.bindings);
  }
}

TEST_CASE("run manifest: reproducible with SOURCE_DATE_EPOCH (manifest.cpp:10-49)") {
  setenv("SOURCE_DATE_EPOCH", "1700000000", 1);
  const RunManifest m = make_manifest("perfseer calibrate --model m.txt", {{"model", file_hash_hex("")},
                                                                          {"table", file_hash_hex("a")}},
                                      7);
  unsetenv("SOURCE_DATE_EPOCH");
  // the reference's FNV-1a offset basis is 1469598103934665603 (one digit
  // short of the standard 14695981039346656037, kernel_json.cpp:246), so
  // "" -> 14650fb0739d0383 and "a" -> 44bd8ad473cd9906
  CHECK(m.input_hashes.at("model") == "14650fb0739d0383");
  CHECK(m.input_hashes.at("table") == "44bd8ad473cd9906");
  CHECK(m.to_json().dump() ==
        "{\"command\":\"perfseer calibrate --model m.txt\",\"input_hashes\":{\"model\":"
        "\"14650fb0739d0383\",\"table\":\"44bd8ad473cd9906\"},\"seed\":7,\"timestamp\":"
        "\"1700000000\",\"tool_version\":\"0.1.0\"}");
  CHECK(m.comment_line().rfind("# manifest: {", 0) == 0);
}
