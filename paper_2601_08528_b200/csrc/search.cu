// K-S dispatch: specialised instantiations for the configs' row lengths (D = 96, 128, 200), generic otherwise.
#include "kernels.h"

namespace svf {

cudaError_t launch_search_d0(SearchArgs a, int kpl, int cpl, int num_sms, cudaStream_t st);
cudaError_t launch_search_d24(SearchArgs a, int kpl, int cpl, int num_sms, cudaStream_t st);
cudaError_t launch_search_d32(SearchArgs a, int kpl, int cpl, int num_sms, cudaStream_t st);
cudaError_t launch_search_d50(SearchArgs a, int kpl, int cpl, int num_sms, cudaStream_t st);

cudaError_t launch_search(SearchArgs a, int kpl, int cpl, int num_sms, cudaStream_t st) {
  switch (a.dq) {
    case 24: return launch_search_d24(a, kpl, cpl, num_sms, st);   // D = 96 (Deep-shaped)
    case 32: return launch_search_d32(a, kpl, cpl, num_sms, st);   // D = 128 (SIFT-shaped)
    case 50: return launch_search_d50(a, kpl, cpl, num_sms, st);   // D = 200 (Text2Image-shaped)
  }
  return launch_search_d0(a, kpl, cpl, num_sms, st);
}

}  // namespace svf
