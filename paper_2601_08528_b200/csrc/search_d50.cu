// K-S instantiations for rows of 50 float4 (0 = generic runtime geometry).  See search_impl.cuh.
#include "search_impl.cuh"

namespace svf {
cudaError_t launch_search_d50(SearchArgs a, int kpl, int cpl, int num_sms, cudaStream_t st) {
  return launch_search_dq<50>(a, kpl, cpl, num_sms, st);
}
}  // namespace svf
