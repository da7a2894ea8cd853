// K17/K18 placeholders (batched LM fit, batched prediction).
#include "runtime_internal.h"

extern "C" int ps_fit_lm_batched(ps_ctx*, const ps_bytecode*, const ps_bytecode*, int, int,
                                 const double*, const double*, int, int, const ps_fit_opts*,
                                 double*, ps_fit_stats*) {
  return ps::set_error(PS_ERR_ARG, "ps_fit_lm_batched: not built in this revision");
}
extern "C" int ps_eval_batched(ps_ctx*, const ps_variant_tables*, const int64_t*, int64_t, double*,
                               uint8_t*) {
  return ps::set_error(PS_ERR_ARG, "ps_eval_batched: not built in this revision");
}
