// fp16-key (HF) instantiations of the r = 2 kernel for the RR >= 8 shapes: one
// mismatch min per real row as two HADD2s on the FMA pipe (ap_kernels.cuh,
// kHfBase).  Usable when W + 2*VB <= kHfMaxSpan (checked by the host).
#include "ap_kernels.cuh"

namespace apk {

template <int L, int RR, int K>
static KernelFn pick(bool dense) {
  return dense ? &comb2_kernel<L, RR, K, true, true> : &comb2_kernel<L, RR, K, false, true>;
}

KernelFn pick_r2_hf(int l, int rr, int k, bool dense) {
#define AP_R2(L, RR, K) \
  if (l == L && rr == RR && k == K) return pick<L, RR, K>(dense);
  AP_R2(4, 25, 5) AP_R2(8, 8, 2) AP_R2(8, 8, 4) AP_R2(16, 8, 4) AP_R2(32, 8, 4)
  AP_R2(8, 16, 4) AP_R2(16, 16, 4) AP_R2(32, 16, 4)
  AP_R2(8, 20, 4) AP_R2(16, 10, 2) AP_R2(4, 25, 1)
  AP_R2(10, 10, 2) AP_R2(5, 20, 4) AP_R2(10, 10, 1) AP_R2(5, 20, 1)
#undef AP_R2
  return nullptr;
}

}  // namespace apk
