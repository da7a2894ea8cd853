// Exact count tables for batched prediction (K18), see ps_tables.cpp.
#pragma once

#include <array>
#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "ps_model.hpp"

namespace perfseer {

struct VariantTables {
  // per variant
  std::vector<int32_t> var_group, var_model, var_feat_base;
  std::vector<std::string> var_id;
  // per feature slot: terms [feat_begin, feat_end) over a common denominator
  std::vector<int32_t> feat_begin, feat_end;
  std::vector<int64_t> feat_den;
  // per term: integer coefficient and exponents of point coordinates 0..3
  std::vector<int64_t> term_coef;
  std::vector<std::array<int8_t, 4>> term_exp;
  // per model: the value program (CSE'd straight-line, compile_program)
  std::vector<Program> models;
  std::vector<std::vector<double>> params;
  std::vector<int32_t> model_nf;
  int ngroups = 0;
};

/// spec: {"variants": [{"id": variant id (any admissible size), "model": model
/// text, "params": [fitted values], "group": application index, "coords":
/// {"<size parameter>": point coordinate 0..3}}]}
VariantTables build_variant_tables(const std::string& spec_json);

/// CPU evaluation of one variant's features at a point (int128, exact).
std::vector<double> eval_point_cpu(const VariantTables& t, size_t v, const int64_t* point);

}  // namespace perfseer
