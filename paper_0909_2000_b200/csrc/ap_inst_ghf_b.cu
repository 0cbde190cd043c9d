// fp16-key (HF) instantiations of the generic comb kernel (table masks), part b:
// V' = (V - d) + T on the FMA pipe for one row of every four (ap_kernels.cuh, kHfBase).
// Used when W + L*K <= kHfMaxSpan (checked by the host); see kShapes in ap_capi.cu.
#include "ap_kernels.cuh"

namespace apk {

template <int L, int R, int K>
static KernelFn pick(bool dense) {
  return dense ? &comb_kernel<L, R, K, true, false, true> : &comb_kernel<L, R, K, false, false, true>;
}

KernelFn pick_ghf_b(int l, int r, int k, bool dense) {
#define AP_G(L, R, K) \
  if (l == L && r == R && k == K) return pick<L, R, K>(dense);
  AP_G(16, 8, 2) AP_G(16, 16, 2) AP_G(16, 16, 4) AP_G(16, 24, 2) AP_G(16, 32, 2) AP_G(16, 32, 4)
#undef AP_G
  return nullptr;
}

}  // namespace apk
