// Instantiations of the tcgen05 GEMM, single-pass TF32.
#include "gemm_tc.cuh"

namespace wapgemm {
template <int CG>
static int by_bn(const Plan& p, cudaStream_t st) {
  switch (p.bn) {
    case 64: return launch_majors<64, 1, CG>(p, st);
    case 128: return launch_majors<128, 1, CG>(p, st);
    case 192: return launch_majors<192, 1, CG>(p, st);
    default: return launch_majors<256, 1, CG>(p, st);
  }
}
int launch_prec1(const Plan& p, cudaStream_t st) { return p.cg == 2 ? by_bn<2>(p, st) : by_bn<1>(p, st); }
}  // namespace wapgemm
