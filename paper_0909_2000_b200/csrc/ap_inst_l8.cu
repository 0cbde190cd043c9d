// Comb-kernel instantiations for L = 8 lanes per strip pair.  Split by L so the
// build compiles them in parallel; ap_capi.cu reaches them through the host
// launch-stub pointers returned here (see kShapes there).
#include "ap_kernels.cuh"

namespace apk {

template <int R, int K>
static KernelFn pick(bool dense, bool xm) {
  if (dense) return xm ? &comb_kernel<8, R, K, true, true, false> : &comb_kernel<8, R, K, true, false, false>;
  return xm ? &comb_kernel<8, R, K, false, true, false> : &comb_kernel<8, R, K, false, false, false>;
}

KernelFn pick_l8(int r, int k, bool dense, bool xm) {
  if (r == 8 && k == 2) return pick<8, 2>(dense, xm);
  if (r == 16 && k == 2) return pick<16, 2>(dense, xm);
  if (r == 16 && k == 4) return pick<16, 4>(dense, xm);
  if (r == 24 && k == 2) return pick<24, 2>(dense, xm);
  if (r == 32 && k == 2) return pick<32, 2>(dense, xm);
  if (r == 32 && k == 4) return pick<32, 4>(dense, xm);
  return nullptr;
}

}  // namespace apk
