// verify_tc_n16.cu — the N = 16 instantiations of verify_tc_kernel (verify_tc.cuh); one translation
// unit per MMA width so the 8 instantiations of each compile in parallel.
#include "verify_tc.cuh"

namespace sa {
cudaError_t launch_verify_tc_n16(int mr, const VerifyParams& p, const CUtensorMap& tk, const CUtensorMap& tv,
                                 cudaStream_t s) {
  return launch_mr<16>(mr, p, tk, tv, s);
}
}  // namespace sa
