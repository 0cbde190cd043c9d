// Build the generic kernel's step loop up from the bare cell pattern, one
// component at a time, to see which one costs throughput:
//   V0 cells (4 bands x 4 rows, registers) + STS of the bottom seaweed (one lane)
//   V1 + SHFL of the seaweed (lane j-1 -> j)   V2 + SHFL of the y code   V4 + LDS.128 table quad per band
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/loop_peak.bin tools/loop_peak.cu
#include <cstdint>
#include <cstdio>
#include <vector>
#include <algorithm>
#include <map>

#define STEPS 2048
struct Rec { long long t0, t1; int sm; };
__device__ __forceinline__ uint32_t smid() { uint32_t s; asm volatile("mov.u32 %0, %%smid;" : "=r"(s)); return s; }
__device__ __forceinline__ uint32_t lop3x(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d; asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d; }
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v; asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr)); return v; }

template <int V>
__global__ void __launch_bounds__(128, 4) k_loop(uint32_t* out, Rec* rec, uint32_t seed) {
  constexpr int K = 4, RB = 4, L = 8;
  __shared__ __align__(16) uint4 tbl[4 /*warps*/][4 /*codes*/][4 /*quads*/][32];
  __shared__ uint32_t ring[4][64];
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, j = lane % L;
  for (int i = threadIdx.x; i < 4 * 4 * 4 * 32; i += blockDim.x)
    (&tbl[0][0][0][0])[i] = make_uint4(seed * i & 0x80008000u, (seed + i) & 0x8000u, i & 0x80000000u, 0u);
  __syncthreads();
  uint32_t Vr[K * RB], tb[K], cd[K];
#pragma unroll
  for (int i = 0; i < K * RB; ++i) Vr[i] = (seed * (i + 3) + threadIdx.x) & 0x3FFF3FFFu;
#pragma unroll
  for (int b = 0; b < K; ++b) { tb[b] = seed + b; cd[b] = (lane + b) & 3; }
  const uint32_t tbase = uint32_t(__cvta_generic_to_shared(&tbl[warp][0][0][lane]));
  uint32_t fresh = seed;
  long long t0 = clock64();
  for (int s = 0; s < STEPS; ++s) {
    uint4 nfq[K];
#pragma unroll
    for (int b = 0; b < K; ++b) {
      if constexpr (V >= 4) nfq[b] = lds128(tbase + cd[b] * (4 * 32 * 16) + b * (32 * 16));
      else nfq[b] = make_uint4(cd[b] << 15, cd[b] << 31, (cd[b] ^ 1) << 15, (cd[b] ^ 2) << 31);
    }
    uint32_t tin[K];
    if constexpr (V >= 1) {
      const uint32_t sh = __shfl_up_sync(0xFFFFFFFFu, tb[K - 1], 1, L);
      tin[0] = j == 0 ? fresh : sh;
    } else {
      tin[0] = fresh;
    }
#pragma unroll
    for (int b = 1; b < K; ++b) tin[b] = tb[b - 1];
    fresh += 0x10001u;
#pragma unroll
    for (int b = 0; b < K; ++b) {
      uint32_t t = tin[b];
      const uint32_t m[4] = {nfq[b].x, nfq[b].y, nfq[b].z, nfq[b].w};
#pragma unroll
      for (int k = 0; k < RB; ++k) {
        uint32_t& v = Vr[b * RB + k];
        const uint32_t d = __viaddmax_s16x2(t, m[k], v);
        v = lop3x(v, t, d);
        t = d;
      }
      tb[b] = t;
    }
    if (j == L - 1) ring[warp][s & 63] = tb[K - 1];   // always on: pins the loop
    {
      const uint32_t ynew = (s * 2654435761u >> 30);
      uint32_t sh = cd[K - 1];
      if constexpr (V >= 2) sh = __shfl_up_sync(0xFFFFFFFFu, cd[K - 1], 1, L);
#pragma unroll
      for (int b = K - 1; b > 0; --b) cd[b] = cd[b - 1];
      cd[0] = j == 0 ? ynew : (sh & 3);
    }
  }
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < K * RB; ++i) acc ^= Vr[i];
  asm volatile("" : "+r"(acc) :: "memory");   // the loop's results exist before the second clock read
  long long t1 = clock64();
  if (acc == 0x12345678u) out[0] = acc + ring[warp][lane];
  if (threadIdx.x == 0) rec[blockIdx.x] = {t0, t1, (int)smid()};
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  const int nsm = p.multiProcessorCount;
  uint32_t* out; Rec* rec; cudaMalloc(&out, 64); cudaMalloc(&rec, 64 * nsm * sizeof(Rec));
  std::vector<Rec> h(64 * nsm);
  auto run = [&](auto kern, const char* name, int warps_per_sm) {
    const int threads = 128, blocks = nsm * warps_per_sm / 4;
    kern<<<blocks, threads>>>(out, rec, 7); kern<<<blocks, threads>>>(out, rec, 7);
    cudaDeviceSynchronize();
    cudaMemcpy(h.data(), rec, blocks * sizeof(Rec), cudaMemcpyDeviceToHost);
    std::map<int, std::pair<long long, long long>> span; std::map<int, int> nb;
    for (int i = 0; i < blocks; ++i) {
      auto it = span.find(h[i].sm);
      if (it == span.end()) span[h[i].sm] = {h[i].t0, h[i].t1};
      else { it->second.first = std::min(it->second.first, h[i].t0); it->second.second = std::max(it->second.second, h[i].t1); }
      nb[h[i].sm]++;
    }
    std::vector<double> r;
    for (auto& kv : span) r.push_back(double(nb[kv.first]) * threads * 16.0 * STEPS / double(kv.second.second - kv.second.first));
    std::sort(r.begin(), r.end());
    printf("{\"variant\": \"%s\", \"warps_per_sm\": %d, \"cell_pairs_per_clk_per_sm\": %.2f}\n", name, warps_per_sm, r[r.size() / 2]);
  };
  for (int w : {16}) {
    run(k_loop<0>, "V0 cells + sts ring", w);
    run(k_loop<1>, "V1 +shfl seaweed", w);
    run(k_loop<2>, "V2 +shfl code", w);
    run(k_loop<4>, "V4 +lds.128 table", w);
  }
  return 0;
}
