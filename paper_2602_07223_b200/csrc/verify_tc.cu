// verify_tc.cu — dispatch of the tcgen05 verify kernel (verify_tc.cuh) over its MMA widths.
#include "verify_tc.cuh"

namespace sa {
cudaError_t launch_verify_tc_n16(int, const VerifyParams&, const CUtensorMap&, const CUtensorMap&, cudaStream_t);
cudaError_t launch_verify_tc_n32(int, const VerifyParams&, const CUtensorMap&, const CUtensorMap&, cudaStream_t);
cudaError_t launch_verify_tc_n48(int, const VerifyParams&, const CUtensorMap&, const CUtensorMap&, cudaStream_t);
cudaError_t launch_verify_tc_n64(int, const VerifyParams&, const CUtensorMap&, const CUtensorMap&, cudaStream_t);

int verify_tc_merge_capacity(int M) {
  switch ((M + 2 + 15) / 16 * 16) {
    case 16: return TCfg<16>::kOffBar;
    case 32: return TCfg<32>::kOffBar;
    case 48: return TCfg<48>::kOffBar;
    default: return TCfg<64>::kOffBar;
  }
}

cudaError_t launch_verify_tc(const VerifyParams& p, const CUtensorMap& tk, const CUtensorMap& tv, cudaStream_t s) {
  const int n = (p.M + 15) / 16 * 16;
  const int mr = p.full_rows ? n : (p.M + 3) / 4 * 4;  // softmax rows: M rounded up to 4 (<= N)
  switch (n) {
    case 16: return launch_verify_tc_n16(mr, p, tk, tv, s);
    case 32: return launch_verify_tc_n32(mr, p, tk, tv, s);
    case 48: return launch_verify_tc_n48(mr, p, tk, tv, s);
    case 64: return launch_verify_tc_n64(mr, p, tk, tv, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace sa
