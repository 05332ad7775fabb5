// K-S instantiations for rows of 0 float4 (0 = generic runtime geometry).  See search_impl.cuh.
#include "search_impl.cuh"

namespace svf {
cudaError_t launch_search_d0(SearchArgs a, int kpl, int cpl, int num_sms, cudaStream_t st) {
  return launch_search_dq<0>(a, kpl, cpl, num_sms, st);
}
// dynamic shared memory of one search block (checked against the device's opt-in limit before any launch)
size_t search_smem_bytes(int hbits, int kpl, int cpl, int L, int large_pool, int vc_bits, int Dp, int lp_slots) {
  (void)kpl;
  if (large_pool) return search_lp_smem_bytes(lp_slots, L, cpl, vc_bits > 0, Dp);
  switch (cpl) {
    case 1: return Smem<1>::block_bytes(hbits);
    case 2: return Smem<2>::block_bytes(hbits);
    case 4: return Smem<4>::block_bytes(hbits);
    default: return Smem<8>::block_bytes(hbits);
  }
}
}  // namespace svf
