// tcgen05 / TMEM / TMA attention kernels for sm_100a (forward and backward).
#include "common.cuh"

namespace spattn {
bool tc_fwd_supported(const FwdArgs&) { return false; }
void launch_attn_fwd_tc(const FwdArgs&, const ProblemSet&, cudaStream_t) {}
bool tc_bwd_supported(const BwdArgs&) { return false; }
void launch_attn_bwd_tc(const BwdArgs&, const ProblemSet&, cudaStream_t) {}
}  // namespace spattn
