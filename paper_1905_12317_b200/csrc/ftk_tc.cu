// Tensor-core engine (tcgen05) -- under construction: every entry fails loudly until implemented.
#include "ftk_tc.cuh"

namespace ftk {

int tc_plan_init(TcPlan& tc, const PlanMath&, const std::vector<float>&, const std::vector<int>&,
                 const std::vector<float>&, int, std::string& msg) {
  tc.ready = false;
  msg = "tensor-core engine (engine=0) not available in this build; use engine=1";
  return FTK_EINVAL;
}
void tc_plan_free(TcPlan&) {}
int tc_prepare_images(TcPlan&, const float2*, int64_t, const DevPlan&, cudaStream_t, std::string& msg) {
  msg = "tensor-core engine not available";
  return FTK_EINVAL;
}
int tc_prepare_templates(TcPlan&, const float2*, int64_t, const DevPlan&, cudaStream_t, std::string& msg) {
  msg = "tensor-core engine not available";
  return FTK_EINVAL;
}
size_t tc_bytes_per_pair(const TcPlan&, const DevPlan& P) {
  return (size_t)P.H_plus * P.n_psi * 8 + (size_t)P.K3p * P.n_psi * 4;
}
ftk_status_t tc_block_shape(const TcPlan&, const DevPlan&, int, int64_t, int64_t, int64_t, int64_t&, int64_t&) {
  return FTK_OK;
}
int tc_run_block(TcPlan&, const PairBlock&, const DevPlan&, void*, size_t, int, unsigned long long*,
                 unsigned long long*, int, float*, cudaStream_t, prof_cb_t, void*, std::string& msg) {
  msg = "tensor-core engine not available";
  return FTK_EINVAL;
}

}  // namespace ftk
