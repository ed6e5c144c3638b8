// verify_tc_n32.cu — the N = 32 instantiations of verify_tc_kernel (verify_tc.cuh); one translation
// unit per MMA width so the 8 instantiations of each compile in parallel.
#include "verify_tc.cuh"

namespace sa {
cudaError_t launch_verify_tc_n32(int mr, const VerifyParams& p, const CUtensorMap& tk, const CUtensorMap& tv,
                                 cudaStream_t s) {
  return launch_mr<32>(mr, p, tk, tv, s);
}
}  // namespace sa
