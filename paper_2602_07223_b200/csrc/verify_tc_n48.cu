// verify_tc_n48.cu — the N = 48 instantiations of verify_tc_kernel (verify_tc.cuh); one translation
// unit per MMA width so the 8 instantiations of each compile in parallel.
#include "verify_tc.cuh"

namespace sa {
cudaError_t launch_verify_tc_n48(int mr, const VerifyParams& p, const CUtensorMap& tk, const CUtensorMap& tv,
                                 cudaStream_t s) {
  return launch_mr<48>(mr, p, tk, tv, s);
}
}  // namespace sa
