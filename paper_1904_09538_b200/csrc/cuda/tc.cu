// K16: tcgen05 dense-contraction matmul variant (placeholder until the
// tcgen05/TMEM kernel lands; fails loudly instead of falling back).
#include "runtime_internal.h"

namespace ps {
int tc_launch(Ctx*, const ps_kernel_desc*) {
  return set_error(PS_ERR_ARG, "matmul_sq_tc: tcgen05 variant not built in this revision");
}
}  // namespace ps
