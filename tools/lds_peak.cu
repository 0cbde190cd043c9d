// Shared-memory load issue/throughput microbenchmark: does a warp's LDS cost depend on how
// many distinct words it touches (broadcast / overlap) or only on the instruction width?
// Decides whether the generic comb kernel's table loads (LSU-bound, C3/C5) can be cut by
// letting lane groups share table words.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lds_peak.bin tools/lds_peak.cu
#include <cstdint>
#include <cstdio>
#include <vector>

#define ITERS 2048
#define CH 8

__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.volatile.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ uint2 lds64(uint32_t a) {
  uint2 v;
  asm volatile("ld.volatile.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}

// P: address pattern (byte offset of lane l):
//  0 distinct consecutive 16 B (lane*16)       1 all lanes one address
//  2 groups of 4 lanes share 16 B (8 distinct)  3 groups of 8 lanes share (4 distinct)
//  4 lanes of group g (4 lanes) at g*8 + j*128 (overlapping, 8-B shifted: the shared-table layout)
//  5-10 the dual-pair kernel's table layouts: is an LDS.128 conflict-free when every aligned
//       group of 8 lanes (a quarter warp) covers 8 different 16-B bank groups?
// W: 32, 64, 128-bit loads
template <int P, int W>
__global__ void k(uint32_t* out, long long* cyc) {
  __shared__ __align__(16) uint32_t sm[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = i * 2654435761u;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t off;
  if (P == 0) off = lane * 16;
  else if (P == 1) off = 0;
  else if (P == 2) off = (lane >> 2) * 16;
  else if (P == 3) off = (lane >> 3) * 16;
  else if (P == 4) off = (lane >> 2) * 8 + (lane & 3) * 128;
  // dual-pair table layouts (ap_dual_kernels.cuh): lane (g, j) at chunk PJ * j + g
  else if (P == 5) off = ((lane & 3) * 17 + (lane >> 2)) * 16;    // L = 4, PJ = 17
  else if (P == 6) off = ((lane & 3) * 18 + (lane >> 2)) * 16;    // L = 4, PJ = 18
  else if (P == 7) off = ((lane & 7) * 13 + (lane >> 3)) * 16;    // L = 8, PJ = 13
  else if (P == 8) off = ((lane & 7) * 12 + (lane >> 3)) * 16;    // L = 8, PJ = 12 (even)
  else if (P == 9) off = ((lane % 10) * 9 + (lane / 10 < 3 ? lane / 10 : 2)) * 16;   // L = 10, PJ = 9
  else if (P == 10) off = ((lane % 5) * 13 + (lane / 5 < 6 ? lane / 5 : 5)) * 16;    // L = 5, PJ = 13
  else {   // L = 10, R = 20 with per-run bank residues (dual_base): runs at quads 0, 9, 20, 31, 42, 53, 67, 78, 92, 103
    const int base[10] = {0, 9, 20, 31, 42, 53, 67, 78, 92, 103};
    off = (base[lane % 10] + (lane / 10 < 3 ? lane / 10 : 2)) * 16;
  }
  if (W == 32) off = P == 0 ? lane * 4 : off / 4 * 4;
  const uint32_t base = uint32_t(__cvta_generic_to_shared(sm)) + off + (warp & 7) * 512;
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const uint32_t a = base + ((it * CH + c) & 3) * 4096;
      if (W == 128) { uint4 v = lds128(a); acc += v.x ^ v.y ^ v.z ^ v.w; }
      else if (W == 64) { uint2 v = lds64(a); acc += v.x ^ v.y; }
      else acc += lds32(a);
    }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int P, int W>
void run(const char* name, int warps) {
  uint32_t* out;
  long long* cyc;
  const int blocks = 148;
  cudaMalloc(&out, blocks * warps * 32 * 4);
  cudaMalloc(&cyc, blocks * 8);
  k<P, W><<<blocks, warps * 32>>>(out, cyc);
  k<P, W><<<blocks, warps * 32>>>(out, cyc);
  cudaDeviceSynchronize();
  std::vector<long long> h(blocks);
  cudaMemcpy(h.data(), cyc, blocks * 8, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (auto v : h) avg += double(v);
  avg /= blocks;
  const double instr = double(ITERS) * CH * warps;   // warp-level LDS per SM (one CTA per SM)
  std::printf("{\"pattern\": \"%s\", \"bits\": %d, \"warps_per_sm\": %d, \"cycles_per_warp_lds\": %.3f, "
              "\"bytes_per_clk_per_sm_nominal\": %.1f}\n",
              name, W, warps, avg / instr, instr * 32 * (W / 8) / avg);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {8, 16, 32}) {
    run<0, 128>("distinct", w);
    run<1, 128>("broadcast", w);
    run<2, 128>("8 distinct (4 lanes each)", w);
    run<3, 128>("4 distinct (8 lanes each)", w);
    run<0, 64>("distinct", w);
    run<1, 64>("broadcast", w);
    run<4, 64>("shared table (8-B group shift)", w);
    run<5, 128>("dual table L=4 PJ=17 (2 lanes per bank group in a quarter warp)", w);
    run<6, 128>("dual table L=4 PJ=18", w);
    run<7, 128>("dual table L=8 PJ=13", w);
    run<8, 128>("dual table L=8 PJ=12 (even)", w);
    run<9, 128>("dual table L=10 PJ=9", w);
    run<10, 128>("dual table L=5 PJ=13", w);
    run<11, 128>("dual table L=10, runs placed by bank residue", w);
    run<0, 32>("distinct", w);
    run<1, 32>("broadcast", w);
  }
  return 0;
}
