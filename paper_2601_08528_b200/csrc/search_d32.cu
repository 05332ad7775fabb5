// K-S instantiations for rows of 32 float4 (0 = generic runtime geometry).  See search_impl.cuh.
#include "search_impl.cuh"

namespace svf {
cudaError_t launch_search_d32(SearchArgs a, int kpl, int cpl, int num_sms, cudaStream_t st) {
  return launch_search_dq<32>(a, kpl, cpl, num_sms, st);
}
}  // namespace svf
