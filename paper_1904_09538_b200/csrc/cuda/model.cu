// K18 placeholder (batched prediction) until eval.cu lands.
#include "runtime_internal.h"

extern "C" int ps_eval_batched(ps_ctx*, const ps_variant_tables*, const int64_t*, int64_t, double*,
                               uint8_t*) {
  return ps::set_error(PS_ERR_ARG, "ps_eval_batched: not built in this revision");
}
