// Instantiations of the tcgen05 GEMM, 3xTF32 (fp32-accurate).
#include "gemm_tc.cuh"

namespace wapgemm {
template <int CG>
static int by_bn(const Plan& p, cudaStream_t st) {
  switch (p.bn) {
    case 64: return launch_majors<64, 3, CG>(p, st);
    case 128: return launch_majors<128, 3, CG>(p, st);
    default: return launch_majors<192, 3, CG>(p, st);  // 3xTF32: BN <= 192 (TMEM: acc + S + A slots)
  }
}
int launch_prec3(const Plan& p, cudaStream_t st) { return p.cg == 2 ? by_bn<2>(p, st) : by_bn<1>(p, st); }
}  // namespace wapgemm

#ifdef WAP_GEMM_TRACE
// Diagnostic builds only: copy block 0's role/wait trace (5 roles x 4 slots).
extern "C" int wap_gemm_trace_read(unsigned long long* host, int n) {
  if (n > 64) n = 64;
  return (int)cudaMemcpyFromSymbol(host, wapgemm::g_gemm_trace, n * sizeof(unsigned long long));
}
#endif
