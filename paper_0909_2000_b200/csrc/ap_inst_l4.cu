// Comb-kernel instantiations for L = 4 lanes per strip pair.  Split by L so the
// build compiles them in parallel; ap_capi.cu reaches them through the host
// launch-stub pointers returned here (see kShapes there).
#include "ap_kernels.cuh"

namespace apk {

template <int R, int K>
static KernelFn pick(bool dense, bool xm) {
  if (dense) return xm ? &comb_kernel<4, R, K, true, true, false> : &comb_kernel<4, R, K, true, false, false>;
  return xm ? &comb_kernel<4, R, K, false, true, false> : &comb_kernel<4, R, K, false, false, false>;
}

KernelFn pick_l4(int r, int k, bool dense, bool xm) {
  if (r == 32 && k == 2) return pick<32, 2>(dense, xm);
  if (r == 32 && k == 4) return pick<32, 4>(dense, xm);
  return nullptr;
}

}  // namespace apk
