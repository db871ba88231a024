// k_sep2d.cu -- K2: 2D separable stepper (placeholder until the DMMA path lands).
#include "pr_internal.cuh"

namespace pr {
pr_status run_sep2d(const Sep2dArgs &a, cudaStream_t s)
{
    (void)a; (void)s;
    set_error("2D separable stepper not built yet");
    return PR_EINVAL;
}
}  // namespace pr

extern "C" pr_status pr_op_create_sep2d(int n, double dt, pr_op *out)
{
    (void)n; (void)dt;
    if (out) *out = nullptr;
    pr::set_error("2D separable operator not built yet");
    return PR_EINVAL;
}
