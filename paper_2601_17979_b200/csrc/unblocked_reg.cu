// unblocked_reg.cu -- kernel (2), register-resident fast path (placeholder:
// the planner reports it unavailable until the specialised kernel lands).
#include "launch.h"

namespace bsvd {

Plan plan_unblocked_reg(int dtype, int bm, int bn, int need_v) {
    (void)dtype; (void)bm; (void)bn; (void)need_v;
    Plan p{};
    p.kernel = 0;
    return p;
}

int launch_unblocked_reg_d32(SolveArgs<double> a, const Plan& p, cudaStream_t st) {
    (void)a; (void)p; (void)st;
    return BSVD_ERR_UNSUPPORTED;
}

}  // namespace bsvd
