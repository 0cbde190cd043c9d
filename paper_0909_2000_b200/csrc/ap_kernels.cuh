// ap_kernels.cuh — sm_100a kernels of the alignment-plot engine.
//
// The hot path of the reference:
//   blowup (scoring.cpp:5-17)                       -> fused into the code streams (K1)
//   comb_strip_lanes / sweep<T> (lane_kernel.cpp:28-128)
//   to_bottom_events (lane_kernel.cpp:5-18)
//   window_llcs_from_events (seaweed_scalar.cpp:65-99)
//   llcs_to_half / recover_score (runner.cpp:31-35, scoring.cpp:26-28)
//   PlotGrid fill / apply_threshold (runner.cpp:108, scoring.cpp:30-39)
// all fused into one combing kernel (K2) per launch.
//
// Seaweed representation.  The reference keeps, per lane, the *distance* of a
// seaweed from its start column and saturates it (lane_kernel.cpp:66-77).  We
// keep the seaweed's *start key* instead: key = start_column - kbase, a 16-bit
// unsigned value, two strips packed per 32-bit register (x-windows A and B of
// the same grid-row pair share every y character).  Left-boundary seaweeds
// have key 0 (they start left of everything, seaweed_scalar.cpp:21-22).  The
// cell rule "exchange iff match or start(V) > start(T)"
// (seaweed_scalar.cpp:26-32) becomes, with NF = 0 on a match and all-ones on a
// mismatch (per 16-bit half):
//     d      = max_u16x2(V, T & NF)      // seaweed leaving downwards
//     V'     = V ^ T ^ d                 // seaweed leaving to the right
// i.e. LOP3 + VIMNMX.U16x2 + LOP3 for two cells: no increment, no saturation
// in the inner loop.  Keys are rebased (saturating at 0) every ~32K columns;
// a rebased-to-0 seaweed is provably older than any window.
//
// NF comes from a per-warp shared-memory table indexed by the y code: the
// x-window characters are fixed for a strip, so table[code][row] holds the
// mismatch mask of both strips; one LDS.128 serves four rows.
//
// Mapping.  A warp holds 32/L groups; a group of L lanes combs one strip pair,
// lane j owning R consecutive rows [j*R, j*R+R).  Lane j processes column
// s - j at step s (antidiagonal wavefront across lanes); the seaweed leaving
// the bottom of lane j and the y code move to lane j+1 with one SHFL each.
//
// Extraction without a heap.  For the bottom event at column e with start st
// (countable iff e - st < W), the window count obeys
//     count(K+1) = count(K) + [event e=K+W countable] - [seaweed starting at K
//                  ended inside [K, K+W-1]]
// (DESIGN.md §4), evaluated 32 columns at a time by a segmented warp scan;
// LLCS(K) = W - count(K), reported at K = 0 mod r (seaweed_scalar.cpp:85-96).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace apk {

constexpr int kWarpsPerCta = 4;
constexpr int kChunk = 32;          // steps per extraction batch
constexpr uint32_t kRebaseAt = 0xF000u;
constexpr uint32_t kRebaseBy = 0x8000u;

struct CombParams {
  const uint8_t* xcode;   // mapped x codes (0xFF = absent from y), local row 0 at xcode[0]
  const uint8_t* ycode;   // effective y codes, N entries + >=128 pad bytes, 16-B aligned
  uint32_t rows;          // grid rows in this launch
  uint32_t h, w, r, W, N; // step, window, blowup, blown window, effective y length
  uint32_t sigma;         // table codes (incl. the sentinel code when r = 2)
  uint32_t sent_code;     // code of the $ sentinel (r = 2)
  uint32_t S;             // column segment width (effective columns), multiple of 8
  uint32_t nseg;          // number of column segments
  uint32_t ring;          // ok-flag ring size (power of two >= W + 64)
  uint32_t cols;          // grid columns
  uint32_t row_global0;   // global grid row of local row 0
  // dense output
  uint16_t* out;          // [rows][cols]
  // thresholded output
  int32_t t_half;
  uint4* stage;                   // {row, col, half, rank} records
  unsigned long long* cursor;     // staging append cursor
  unsigned long long stage_cap;
  uint32_t* seg_counts;           // [rows][nseg] hits per (row, segment)
};

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

// PRMT with sign replication (selector nibble bit 3); __byte_perm masks it off.
__device__ __forceinline__ uint32_t prmt_sign(uint32_t a, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, 0, %2;" : "=r"(d) : "r"(a), "r"(sel));
  return d;
}

// Shared memory bytes per warp for a (L, R) instantiation.
__host__ __device__ inline size_t comb_smem_per_warp(int L, int R, uint32_t sigma, uint32_t ring) {
  const int G = 32 / L;
  return size_t(128) * sigma * R          // mismatch table (sigma = 0 when masks are computed)
       + size_t(G) * kChunk * 4           // bottom-key ring per group
       + size_t(G) * 2 * ring;            // ok flags per group (strip A, strip B)
}

// XM = false: mismatch masks from the shared-memory table (small alphabets).
// XM = true : masks computed in registers from the x-code pairs (any alphabet):
//   e = (xpair ^ y*0x10001) + 0x7FFF7FFF has bit 15 of a half set iff the codes
//   differ; PRMT's sign-replicate mode (selector 0xBB99) widens it to 0xFFFF.
template <int L, int R, bool DENSE, bool XM>
__global__ void __launch_bounds__(kWarpsPerCta * 32)
comb_kernel(const CombParams p) {
  static_assert(32 % L == 0 && R % 4 == 0, "bad shape");
  constexpr int G = 32 / L;
  constexpr int Q = R / 4;
  extern __shared__ __align__(16) unsigned char smem[];

  const uint32_t lane = lane_id();
  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t g = lane / L;     // group within warp
  const uint32_t j = lane % L;     // lane within group
  const size_t per_warp = comb_smem_per_warp(L, R, p.sigma, p.ring);
  unsigned char* wbase = smem + warp * per_warp;
  uint4* tbl = reinterpret_cast<uint4*>(wbase);                       // [G][sigma][Q][L]
  uint32_t* ringB = reinterpret_cast<uint32_t*>(wbase + size_t(128) * p.sigma * R) + g * kChunk;
  uint8_t* okA = wbase + size_t(128) * p.sigma * R + G * kChunk * 4 + size_t(g) * 2 * p.ring;
  uint8_t* okB = okA + p.ring;
  const uint32_t rmask = p.ring - 1;

  const uint32_t npairs = (p.rows + 1) / 2;
  const uint32_t ngroups = (npairs + G - 1) / G;
  const uint64_t ntasks = uint64_t(ngroups) * p.nseg;
  const uint64_t wstride = uint64_t(gridDim.x) * kWarpsPerCta;

  for (uint64_t task = uint64_t(blockIdx.x) * kWarpsPerCta + warp; task < ntasks; task += wstride) {
    const uint32_t pg = uint32_t(task / p.nseg);
    const uint32_t seg = uint32_t(task % p.nseg);
    const uint32_t pair = pg * G + g;
    const uint32_t rA = 2 * pair, rB = 2 * pair + 1;
    const bool hasA = rA < p.rows, hasB = rB < p.rows;
    const uint32_t c0 = seg * p.S;                       // first effective column of the segment
    const uint32_t nseg_cols = min(p.S + p.W - 1, p.N - c0);
    const uint32_t nsteps = nseg_cols + L - 1;
    const uint32_t nch = (nsteps + kChunk - 1) / kChunk;

    // ---- mismatch table for this strip pair (fused $-interleave, scoring.cpp:5-17)
    __syncwarp();
    uint32_t xpair[XM ? R : 1];
    {
      uint32_t xa[R], xb[R];
#pragma unroll
      for (int rho = 0; rho < R; ++rho) {
        const uint32_t i = j * R + rho;
        uint32_t ca = 0x1FFu, cb = 0x1FFu;  // 0x1FF: never equals a code
        if (i < p.W) {
          if (p.r == 2 && !(i & 1u)) {
            ca = hasA ? p.sent_code : 0x1FFu;
            cb = hasB ? p.sent_code : 0x1FFu;
          } else {
            const uint32_t xi = (p.r == 2) ? (i >> 1) : i;
            if (hasA) ca = p.xcode[size_t(rA) * p.h + xi];
            if (hasB) cb = p.xcode[size_t(rB) * p.h + xi];
            if (ca == 0xFFu) ca = 0x1FFu;   // byte absent from y: never matches
            if (cb == 0xFFu) cb = 0x1FFu;
          }
        }
        xa[rho] = ca;
        xb[rho] = cb;
      }
      if constexpr (XM) {
#pragma unroll
        for (int rho = 0; rho < R; ++rho) xpair[rho] = xa[rho] | (xb[rho] << 16);
      }
      uint4* tg = tbl + size_t(g) * p.sigma * Q * L;
      for (uint32_t a = 0; a < (XM ? 0u : p.sigma); ++a) {
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          uint32_t wv[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int rho = 4 * q + k;
            wv[k] = (xa[rho] == a ? 0u : 0x0000FFFFu) | (xb[rho] == a ? 0u : 0xFFFF0000u);
          }
          tg[(a * Q + q) * L + j] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
        }
      }
      for (uint32_t k = j; k < 2 * p.ring; k += L) okA[k] = 0;
    }
    __syncwarp();

    const uint4* tl = tbl + size_t(g) * p.sigma * Q * L + j;
    const uint64_t* yw = reinterpret_cast<const uint64_t*>(p.ycode + c0);

    uint32_t V[R];
#pragma unroll
    for (int rho = 0; rho < R; ++rho) V[rho] = 0u;   // left-boundary seaweeds: key 0
    uint32_t tout = 0u;                              // virtual columns carry key 0 (harmless)
    uint32_t yprev = 0u;
    int32_t kbase = -int32_t(p.W) - 1;               // key(c) = c - kbase > W for every top seaweed
    uint32_t fresh = uint32_t(-kbase) * 0x00010001u;
    uint32_t run = 0u;                               // packed window counts (A | B << 16)
    uint32_t hitsA = 0u, hitsB = 0u;

    uint64_t ycur = __ldg(yw);
    for (uint32_t ch = 0; ch < nch; ++ch) {
#pragma unroll 1
      for (int sub = 0; sub < kChunk / 8; ++sub) {
        const uint32_t s0 = ch * kChunk + sub * 8;
        const uint64_t ynext = __ldg(yw + (s0 >> 3) + 1);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint32_t y0 = uint32_t(ycur >> (8 * u)) & 0xFFu;
          uint32_t yc = __shfl_up_sync(0xFFFFFFFFu, yprev, 1, L);
          uint32_t tin = __shfl_up_sync(0xFFFFFFFFu, tout, 1, L);
          if (j == 0) { yc = y0; tin = fresh; }
          fresh += 0x00010001u;
          const uint4* tp = tl + yc * (Q * L);
          const uint32_t yrep = yc * 0x00010001u;
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            uint32_t nfv[4];
            if constexpr (XM) {
#pragma unroll
              for (int k = 0; k < 4; ++k)
                nfv[k] = prmt_sign((xpair[4 * q + k] ^ yrep) + 0x7FFF7FFFu, 0xBB99u);
            } else {
              const uint4 nf = tp[q * L];
              nfv[0] = nf.x; nfv[1] = nf.y; nfv[2] = nf.z; nfv[3] = nf.w;
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint32_t t = tin & nfv[k];
              const uint32_t d = __vmaxu2(V[4 * q + k], t);
              V[4 * q + k] = V[4 * q + k] ^ tin ^ d;
              tin = d;
            }
          }
          tout = tin;
          if (j == L - 1) ringB[sub * 8 + u] = tout;
          yprev = yc;
        }
        ycur = ynext;
      }
      __syncwarp();

      // ---- window extraction for bottom columns [E0, E0 + 32)
      const int32_t E0 = int32_t(ch * kChunk) - (L - 1);
#pragma unroll 1
      for (int rd = 0; rd < kChunk / L; ++rd) {
        const int32_t e = E0 + rd * L + int32_t(j);
        const bool valid = e >= 0 && e < int32_t(nseg_cols);
        const uint32_t k = ringB[rd * L + j];
        const int32_t thr = e - kbase - int32_t(p.W);
        const int32_t kA = int32_t(k & 0xFFFFu), kB = int32_t(k >> 16);
        const bool cA = valid && kA > thr;
        const bool cB = valid && kB > thr;
        if (cA) okA[uint32_t(kA + kbase) & rmask] = 1;
        if (cB) okB[uint32_t(kB + kbase) & rmask] = 1;
        __syncwarp();
        uint32_t oA = 0, oB = 0;
        if (valid) {
          const uint32_t slot = uint32_t(e - int32_t(p.W)) & rmask;
          oA = okA[slot];
          oB = okB[slot];
          okA[slot] = 0;
          okB[slot] = 0;
        }
        uint32_t dl = (uint32_t(cA) + 1u - oA) | ((uint32_t(cB) + 1u - oB) << 16);
#pragma unroll
        for (int off = 1; off < L; off <<= 1) {
          const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, dl, off, L);
          if (j >= uint32_t(off)) dl += v;
        }
        const uint32_t cnt = run + dl - (j + 1) * 0x00010001u;
        run = __shfl_sync(0xFFFFFFFFu, cnt, L - 1, L);

        const int32_t kp = e - int32_t(p.W) + 1;   // window start (segment-relative)
        const bool out_ok = valid && kp >= 0 && kp < int32_t(p.S) && (p.r == 1 || !(kp & 1));
        const uint32_t gcol = (c0 + uint32_t(kp)) / p.r;
        const int32_t llA = int32_t(p.W) - int32_t(cnt & 0xFFFFu);
        const int32_t llB = int32_t(p.W) - int32_t(cnt >> 16);
        const int32_t hA = p.r == 1 ? 2 * llA : 2 * llA - 2 * int32_t(p.w);
        const int32_t hB = p.r == 1 ? 2 * llB : 2 * llB - 2 * int32_t(p.w);
        if constexpr (DENSE) {
          if (out_ok && hasA) p.out[size_t(rA) * p.cols + gcol] = uint16_t(hA);
          if (out_ok && hasB) p.out[size_t(rB) * p.cols + gcol] = uint16_t(hB);
        } else {
          const bool hitA = out_ok && hasA && hA >= p.t_half;
          const bool hitB = out_ok && hasB && hB >= p.t_half;
          const uint32_t bA = __ballot_sync(0xFFFFFFFFu, hitA);
          const uint32_t bB = __ballot_sync(0xFFFFFFFFu, hitB);
          if (bA | bB) {
            const uint32_t gmask = (L == 32 ? 0xFFFFFFFFu : ((1u << L) - 1u)) << (g * L);
            const uint32_t lt = (1u << lane) - 1u;
            const uint32_t total = __popc(bA) + __popc(bB);
            unsigned long long basepos = 0;
            if (lane == 0) basepos = atomicAdd(p.cursor, (unsigned long long)total);
            basepos = __shfl_sync(0xFFFFFFFFu, basepos, 0);
            if (hitA) {
              const unsigned long long pos = basepos + __popc(bA & lt);
              const uint32_t rank = hitsA + __popc(bA & gmask & lt);
              if (pos < p.stage_cap)
                p.stage[pos] = make_uint4(p.row_global0 + rA, gcol, uint32_t(hA), rank);
            }
            if (hitB) {
              const unsigned long long pos = basepos + __popc(bA) + __popc(bB & lt);
              const uint32_t rank = hitsB + __popc(bB & gmask & lt);
              if (pos < p.stage_cap)
                p.stage[pos] = make_uint4(p.row_global0 + rB, gcol, uint32_t(hB), rank);
            }
            hitsA += __popc(bA & gmask);
            hitsB += __popc(bB & gmask);
          }
        }
        __syncwarp();
      }

      // ---- key rebase (saturating at 0): keeps fresh keys below 2^16
      if (uint32_t(int32_t((ch + 1) * kChunk + kChunk) - kbase) >= kRebaseAt) {
        const uint32_t by = kRebaseBy * 0x00010001u;
#pragma unroll
        for (int rho = 0; rho < R; ++rho) V[rho] = __vmaxu2(V[rho], by) - by;
        tout = __vmaxu2(tout, by) - by;
        fresh -= by;
        kbase += int32_t(kRebaseBy);
      }
    }
    if constexpr (!DENSE) {
      if (j == 0) {
        if (hasA) p.seg_counts[size_t(rA) * p.nseg + seg] = hitsA;
        if (hasB) p.seg_counts[size_t(rB) * p.nseg + seg] = hitsB;
      }
    }
  }
}

// K1: effective y code stream (fused $-interleave, scoring.cpp:5-17):
// ycode[c] = r == 2 ? (c odd ? map[y[c/2]] : sent) : map[y[c]]; pad with 0.
__global__ void ycode_kernel(const uint8_t* __restrict__ y, size_t n, uint32_t r, uint32_t sent,
                             const uint8_t* __restrict__ map, uint8_t* __restrict__ ycode,
                             size_t total) {
  for (size_t c = blockIdx.x * size_t(blockDim.x) + threadIdx.x; c < total;
       c += size_t(gridDim.x) * blockDim.x) {
    const size_t N = n * r;
    uint8_t v = 0;
    if (c < N) v = (r == 2) ? ((c & 1) ? map[y[c >> 1]] : uint8_t(sent)) : map[y[c]];
    ycode[c] = v;
  }
}

// x codes: map[x[i]] (0xFF for bytes absent from y).
__global__ void xcode_kernel(const uint8_t* __restrict__ x, size_t m, const uint8_t* __restrict__ map,
                             uint8_t* __restrict__ xcode) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < m;
       i += size_t(gridDim.x) * blockDim.x)
    xcode[i] = map[x[i]];
}

// Alphabet of y: presence bitmap -> dense codes (map[b] = rank of b among the
// bytes present in y, 0xFF if absent), sigma -> out[256].  One CTA.
__global__ void alphabet_kernel(const uint8_t* __restrict__ y, size_t n, uint8_t* __restrict__ map,
                                uint32_t* __restrict__ sigma_out, uint32_t* __restrict__ zero_flag) {
  __shared__ uint32_t present[256];
  for (int b = threadIdx.x; b < 256; b += blockDim.x) present[b] = 0;
  __syncthreads();
  for (size_t i = threadIdx.x; i < n; i += blockDim.x) present[y[i]] = 1;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t k = 0;
    for (int b = 0; b < 256; ++b) {
      map[b] = present[b] ? uint8_t(k) : uint8_t(0xFF);
      k += present[b];
    }
    *sigma_out = k;
    *zero_flag = present[0];
  }
}

// Deterministic row-major placement of staged threshold records:
// final index = offset[row * nseg + seg] + rank.
__global__ void place_kernel(const uint4* __restrict__ stage, unsigned long long nrec,
                             const unsigned long long* __restrict__ offsets, uint32_t nseg,
                             uint32_t seg_cols, uint32_t r, uint32_t row_global0,
                             uint32_t* __restrict__ orow, uint32_t* __restrict__ ocol,
                             uint16_t* __restrict__ ohalf, unsigned long long cap) {
  for (unsigned long long i = blockIdx.x * 1ull * blockDim.x + threadIdx.x; i < nrec;
       i += 1ull * gridDim.x * blockDim.x) {
    const uint4 rec = stage[i];
    const uint32_t seg = (rec.y * r) / seg_cols;
    const unsigned long long pos = offsets[size_t(rec.x - row_global0) * nseg + seg] + rec.w;
    if (pos < cap) {
      orow[pos] = rec.x;
      ocol[pos] = rec.y;
      ohalf[pos] = uint16_t(rec.z);
    }
  }
}

}  // namespace apk
