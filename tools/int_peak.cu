// Integer-pipe issue-rate microbenchmark for the roofline denominator
// (P_int = N_SM x int32 ops/clk/SM x clock).
// Each kernel runs 8 independent dependency chains of one SASS op per thread;
// ops/clk/SM is computed from per-CTA clock64 deltas, so it is clock-free.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o int_peak int_peak.cu
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <vector>
#include <algorithm>

#define ITERS 4096
#define CHAINS 8

struct Rec { long long t0, t1; };

template <int OP>
__device__ __forceinline__ uint32_t op(uint32_t a, uint32_t b, uint32_t c, int parity) {
  if constexpr (OP == 0) {  // LOP3
    uint32_t d; asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d;
  } else if constexpr (OP == 1) {  // IADD3
    return a + b + c;
  } else if constexpr (OP == 2) {  // VIMNMX.U16x2 (alternate max / min so nothing folds)
    return parity ? __vmaxu2(a, b) : __vminu2(a, b);
  } else if constexpr (OP == 3) {  // VIADDMNMX.U16x2
    return parity ? __viaddmax_u16x2(a, b, c) : __viaddmin_u16x2(a, b, c);
  } else if constexpr (OP == 4) {  // PRMT
    return __byte_perm(a, b, c);
  } else if constexpr (OP == 5) {  // HMNMX2
    __half2 x = *reinterpret_cast<__half2*>(&a), y = *reinterpret_cast<__half2*>(&b);
    __half2 r = parity ? __hmax2(x, y) : __hmin2(x, y); return *reinterpret_cast<uint32_t*>(&r);
  } else if constexpr (OP == 6) {  // HMUL2
    __half2 x = *reinterpret_cast<__half2*>(&a), y = *reinterpret_cast<__half2*>(&b);
    __half2 r = __hmul2(x, y); return *reinterpret_cast<uint32_t*>(&r);
  } else if constexpr (OP == 7) {  // IMAD
    return a * b + c;
  } else {  // 8: the comb cell triple: D = max(V, T & NF); R = V ^ T ^ D
    uint32_t t = b & c;
    uint32_t d = __vmaxu2(a, t);
    return a ^ b ^ d;
  }
}

template <int OP>
__global__ void k_ops(uint32_t* out, Rec* rec, uint32_t seed) {
  uint32_t v[CHAINS];
  uint32_t b = seed ^ threadIdx.x, c = seed * 3u + blockIdx.x;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) v[i] = seed + i * 77u + threadIdx.x;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) v[i] = op<OP>(v[i], v[(i + 1) % CHAINS], (OP == 4 ? (b + i) & 0x7777u : c), 1);
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) v[i] = op<OP>(v[i], v[(i + 3) % CHAINS], (OP == 4 ? (c + i) & 0x7777u : b), 0);
  }
  __syncthreads();
  long long t1 = clock64();
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) acc ^= v[i];
  if (acc == 0x12345678u) out[0] = acc;
  if (threadIdx.x == 0) rec[blockIdx.x] = {t0, t1};
}

__global__ void k_shfl(uint32_t* out, Rec* rec, uint32_t seed) {
  uint32_t v[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) v[i] = seed + i + threadIdx.x;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) v[i] = __shfl_up_sync(0xffffffffu, v[i], 1, 8);
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) v[i] = __shfl_up_sync(0xffffffffu, v[i], 1, 8);
  }
  __syncthreads();
  long long t1 = clock64();
  uint32_t acc = 0;
  for (int i = 0; i < CHAINS; ++i) acc ^= v[i];
  if (acc == 0x12345678u) out[0] = acc;
  if (threadIdx.x == 0) rec[blockIdx.x] = {t0, t1};
}

__global__ void k_lds128(uint32_t* out, Rec* rec, uint32_t seed) {
  __shared__ uint4 tab[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) tab[i] = make_uint4(i, i + 1, i + 2, (i * 7) & 3);
  __syncthreads();
  uint32_t idx = (seed + threadIdx.x) & 3;
  uint32_t acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      uint4 q = tab[(idx * 512 + (threadIdx.x & 31) + i * 32) & 2047];
      acc += q.x ^ q.y ^ q.z; idx = q.w;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (acc == 0x12345678u) out[0] = acc;
  if (threadIdx.x == 0) rec[blockIdx.x] = {t0, t1};
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  const int nsm = p.multiProcessorCount;
  const int threads = 256, per_sm = 4, blocks = nsm * per_sm;
  uint32_t* out; Rec* rec; cudaMalloc(&out, 4); cudaMalloc(&rec, blocks * sizeof(Rec));
  std::vector<Rec> h(blocks);
  auto report = [&](const char* name, double ops_per_thread) {
    cudaDeviceSynchronize();
    cudaMemcpy(h.data(), rec, blocks * sizeof(Rec), cudaMemcpyDeviceToHost);
    // all blocks resident at once (4 x 256 threads per SM): cycles = median CTA span
    std::vector<double> d; for (auto& r : h) d.push_back(double(r.t1 - r.t0));
    std::sort(d.begin(), d.end());
    double cyc = d[d.size() / 2];
    double per_sm_ops = ops_per_thread * threads * per_sm;
    printf("{\"op\": \"%s\", \"lane_ops_per_clk_per_sm\": %.2f, \"cycles\": %.0f}\n", name, per_sm_ops / cyc, cyc);
  };
  const double ops = 2.0 * ITERS * CHAINS;
#define RUN(OP, NAME, MULT) k_ops<OP><<<blocks, threads>>>(out, rec, 1); report(NAME, ops * MULT);
  for (int rep = 0; rep < 2; ++rep) {
    RUN(0, "LOP3", 1) RUN(1, "IADD3", 1) RUN(2, "VIMNMX.U16x2", 1) RUN(3, "VIADDMNMX.U16x2", 1)
    RUN(4, "PRMT", 1) RUN(5, "HMNMX2", 1) RUN(6, "HMUL2", 1) RUN(7, "IMAD", 1) RUN(8, "comb_triple(3 ops)", 3)
    k_shfl<<<blocks, threads>>>(out, rec, 1); report("SHFL", ops);
    k_lds128<<<blocks, threads>>>(out, rec, 1); report("LDS.128", 16.0 * ITERS);
  }
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"sms\": %d, \"clock_khz_attr\": %d, \"name\": \"%s\"}\n", nsm, clk, p.name);
  return 0;
}
