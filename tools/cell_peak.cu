// Throughput of the comb-cell instruction patterns with independent chains
// (like the kernels' K bands), operands in registers: which limit applies --
// the ALU pipe (2 ALU ops per cell pair) or operand/issue bandwidth?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/cell_peak.bin tools/cell_peak.cu
#include <cstdint>
#include <cstdio>
#include <vector>
#include <algorithm>
#include <map>

#define ITERS 512
struct Rec { long long t0, t1; int sm; };
__device__ __forceinline__ uint32_t smid() { uint32_t s; asm volatile("mov.u32 %0, %%smid;" : "=r"(s)); return s; }
__device__ __forceinline__ uint32_t lop3x(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d; asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d; }
__device__ __forceinline__ uint32_t vam(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d; asm volatile("{.reg .b32 t; add.s16x2 t, %1, %2; max.s16x2 %0, t, %3;}" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d; }

__device__ __forceinline__ uint32_t hadd2x(uint32_t a, uint32_t b) {
  uint32_t d; asm volatile("add.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b)); return d; }
__device__ __forceinline__ uint32_t hsub2x(uint32_t a, uint32_t b) {
  uint32_t d; asm volatile("sub.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b)); return d; }

// NCH chains, each RB cells deep per step; V[NCH*RB] state, M[NCH*RB] masks (registers)
template <int NCH, int RB, int VAR>
__global__ void k_cell(uint32_t* out, Rec* rec, uint32_t seed) {
  uint32_t V[NCH * RB], M[NCH * RB], T[NCH];
#pragma unroll
  for (int i = 0; i < NCH * RB; ++i) { V[i] = (seed * (i + 3) + threadIdx.x) & 0x3FFF3FFFu; M[i] = (seed >> (i & 7)) & 0x80008000u; }
#pragma unroll
  for (int c = 0; c < NCH; ++c) T[c] = seed + c;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      uint32_t t = T[c];
#pragma unroll
      for (int k = 0; k < RB; ++k) {
        uint32_t& v = V[c * RB + k];
        if constexpr (VAR == 0) {           // VIADDMNMX + LOP3 (the generic kernel's cell)
          const uint32_t d = __viaddmax_s16x2(t, M[c * RB + k], v);
          v = lop3x(v, t, d);
          t = d;
        } else if constexpr (VAR == 1) {    // same, LOP3 operand order t first (reuse of t)
          const uint32_t d = __viaddmax_s16x2(t, M[c * RB + k], v);
          v = lop3x(t, v, d);
          t = d;
        } else if constexpr (VAR >= 3 && VAR <= 6) {
          // V' = (V - d) + T as fp16 values (keys 0x6400 + k = 1024 + k: exact), on the FMA pipe,
          // for the first F rows of each group of 4 (F = 4, 2, 3, 1 for VAR 3..6)
          constexpr int F = VAR == 3 ? 4 : VAR == 4 ? 2 : VAR == 5 ? 3 : 1;
          const uint32_t d = __viaddmax_s16x2(t, M[c * RB + k], v);
          if ((k & 3) < F) v = hadd2x(hsub2x(v, d), t);
          else v = lop3x(v, t, d);
          t = d;
        } else if constexpr (VAR == 7) {    // max + fp16 (v - d) + t
          const uint32_t d = __vmaxu2(v, t);
          v = hadd2x(hsub2x(v, d), t);
          t = d;
        } else {                            // mismatch-only comparator: max + min (2-operand ops)
          const uint32_t d = __vmaxu2(v, t);
          v = __vminu2(v, t);
          t = d;
        }
      }
      T[c] = t;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < NCH * RB; ++i) acc ^= V[i];
#pragma unroll
  for (int c = 0; c < NCH; ++c) acc ^= T[c];
  if (acc == 0x12345678u) out[0] = acc;
  if (threadIdx.x == 0) rec[blockIdx.x] = {t0, t1, (int)smid()};
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  const int nsm = p.multiProcessorCount;
  uint32_t* out; Rec* rec; cudaMalloc(&out, 64); cudaMalloc(&rec, 64 * nsm * sizeof(Rec));
  std::vector<Rec> h(64 * nsm);
  auto run = [&](auto kern, const char* name, int warps_per_sm, int cells) {
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
    for (auto& kv : span) r.push_back(double(nb[kv.first]) * threads * cells * double(ITERS) / double(kv.second.second - kv.second.first));
    std::sort(r.begin(), r.end());
    printf("{\"pattern\": \"%s\", \"warps_per_sm\": %d, \"cell_pairs_per_clk_per_sm\": %.2f}\n", name, warps_per_sm, r[r.size() / 2]);
  };
  for (int w : {8, 16, 32}) {
    run(k_cell<4, 4, 0>, "viaddmax+lop3 4x4", w, 16);
    run(k_cell<4, 4, 1>, "viaddmax+lop3(t first) 4x4", w, 16);
    run(k_cell<8, 2, 0>, "viaddmax+lop3 8x2", w, 16);
    run(k_cell<2, 8, 0>, "viaddmax+lop3 2x8", w, 16);
    run(k_cell<4, 4, 2>, "vmax+vmin 4x4", w, 16);
    run(k_cell<4, 4, 3>, "viaddmax+hsub2+hadd2 (all rows) 4x4", w, 16);
    run(k_cell<4, 4, 4>, "viaddmax + 2/4 rows hadd2, 2/4 lop3 4x4", w, 16);
    run(k_cell<4, 4, 5>, "viaddmax + 3/4 rows hadd2, 1/4 lop3 4x4", w, 16);
    run(k_cell<4, 4, 6>, "viaddmax + 1/4 rows hadd2, 3/4 lop3 4x4", w, 16);
    run(k_cell<4, 4, 7>, "vmax + hsub2+hadd2 4x4", w, 16);
  }
  return 0;
}
