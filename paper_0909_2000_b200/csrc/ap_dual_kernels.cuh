// ap_dual_kernels.cuh — generic comb kernel with two strip pairs per lane group.
//
// Same path as comb_kernel (ap_kernels.cuh): comb_strip_lanes / sweep<T>
// (lane_kernel.cpp:28-128), to_bottom_events (lane_kernel.cpp:5-18),
// window_llcs_from_events (seaweed_scalar.cpp:65-99), apply_threshold
// (scoring.cpp:30-39), for LCS plots (r = 1) with step h = 1 whose window is
// exactly L*R rows.
//
// Why.  comb_kernel's long-lane shapes (C3, C5) spend 91% of the shared-memory
// wavefronts on the mask table: one 32-bit mask word per (row, column) and strip
// pair, 8 cells per LDS.128 (ncu r02; halving the loads in a timing ablation
// gave -8.4% on C3).  With h = 1 the strip pair (rows 4g+2, 4g+3) sees the
// x-window of the pair (4g, 4g+1) shifted by two characters, so its mask word
// of strip row i is the first pair's word of row i + 2: a lane that holds rows
// [jR, jR+R) of BOTH pairs reads R + 2 words (R/4 LDS.128 + one LDS.64 per
// band: the first half of the quad below it) for 4R cells instead of 2R —
// 1.8x fewer table wavefronts per cell, four independent seaweed chains per
// lane (K = 2 bands x 2 pairs), and the per-step overhead (shuffles, code feed,
// table addresses) shared by twice the cells.
//
// One table per warp.  Group g's rows are group 0's shifted by 4g characters = g quads, so
// all groups of a warp read one table: per code and lane index j a run of G + R/4 quads
// (group g, quad q at position g + q), runs PJ quads apart with PJ chosen so that every quarter
// warp of an LDS.128 covers all 8 bank groups.  2.5-4 KB per warp instead of 16 (C3),
// which lifts the shared-memory limit on resident warps.
//
// The ok-flag ring is shared too: byte 0/2 of a slot are pair 0's strips, byte
// 1/3 pair 1's (extract_scatter's BYTE).
#pragma once
#include "ap_kernels.cuh"

namespace apk {

KernelFn pick_dual(int l, int r, int k, bool dense, bool hf);

// Quads between the table runs of consecutive lane indices j.  An LDS.128 is served a quarter
// warp (8 lanes, 128 B) at a time, so PJ is the smallest run length for which the chunks
// PJ*j + g of every aligned group of 8 lanes fall on 8 different bank groups (PJ odd for L >= 8,
// PJ = 2 mod 4 for L = 4, 13 for L = 5; lane groups of 10, 15 or 20 lanes straddle the quarters and
// no single stride serves them: dual_base below).
__host__ __device__ constexpr int dual_pj_conflicts(int L, int PJ) {
  const int G = 32 / L;
  int worst = 0;
  for (int a = 0; a < 32; ++a) {
    const int ga = a / L < G ? a / L : G - 1, ca = PJ * (a % L) + ga;
    int n = 1;
    for (int b = (a / 8) * 8; b < (a / 8) * 8 + 8; ++b) {
      const int gb = b / L < G ? b / L : G - 1, cb = PJ * (b % L) + gb;
      bool first = true;   // count each distinct conflicting chunk once
      for (int c = (a / 8) * 8; c < b; ++c) {
        const int gc = c / L < G ? c / L : G - 1;
        if (PJ * (c % L) + gc == cb) first = false;
      }
      if (b != a && cb != ca && cb % 8 == ca % 8 && first) ++n;
    }
    if (n > worst) worst = n;
  }
  return worst;
}
__host__ __device__ constexpr int dual_pj(int L, int R) {
  const int need = 32 / L + R / 4 + (32 % L ? 1 : 0);
  int best = need, bc = 99;
  for (int pj = need; pj < need + 9; ++pj) {
    const int c = dual_pj_conflicts(L, pj);
    if (c < bc) { bc = c; best = pj; }
  }
  return best;
}
// First quad of lane index j's run.  Regular layouts: j * PJ.  Lane groups of 10 and 15 lanes
// straddle the quarter warps, and no single stride is conflict-free for them (an LDS.128 cost 7
// cycles instead of 4 with the best one, tools/lds_peak.cu); a search over the runs' bank groups
// (base mod 8, every quarter warp all-different) gives the residues below, and each run starts at
// the first quad with its residue after the previous run.
__host__ __device__ constexpr int dual_base(int L, int R, int j) {
  if (L != 10 && L != 15) return j * dual_pj(L, R);
  constexpr int b10[10] = {0, 1, 4, 7, 2, 5, 3, 6, 4, 7};
  constexpr int b15[15] = {0, 1, 2, 3, 4, 5, 6, 7, 0, 2, 3, 4, 5, 6, 7};
  const int need = 32 / L + R / 4 + 1;
  int base = 0;
  for (int i = 1; i <= j; ++i) {
    const int want = L == 10 ? b10[i] : b15[i];
    base += need;
    base += (want - base % 8 + 8) % 8;
  }
  return base;
}
// the same for a run-time lane index inside the kernels: the regular stride is folded at compile
// time (dual_pj's search must not run per task)
template <int L, int R>
__device__ __forceinline__ uint32_t dual_base_rt(uint32_t j) {
  if constexpr (L == 10 || L == 15) {
    return uint32_t(dual_base(L, R, int(j)));
  } else {
    constexpr int kPj = dual_pj(L, R);
    return j * uint32_t(kPj);
  }
}
// table quads per code: the L runs, rounded up to 8 quads (128 B) so that lanes holding different
// codes (lane j is at column s - j*K - b) keep their bank group
__host__ __device__ constexpr int dual_cs(int L, int R) {
  return (dual_base(L, R, L - 1) + 32 / L + R / 4 + 1 + 7) / 8 * 8;
}

// Shared memory per warp (one-warp CTAs): the mask table [sigma][CS] quads, two bottom-key rings
// per group, one ok-flag ring per group; lane groups that do not tile the warp (L = 5, 10, 20)
// add an idle "phantom" group with its own rings and a 64-byte flag scratch (as comb2_kernel).
__host__ __device__ inline size_t combd_smem_per_warp(int L, int R, int K, uint32_t sigma, uint32_t ring) {
  const int G = 32 / L, Ga = groups_alloc(L);
  const size_t bytes = size_t(16) * sigma * dual_cs(L, R)
       + ((size_t(2) * Ga * ring_stride(L, kChunk) * 4 + 15) & ~size_t(15))
       + size_t(G) * ok_stride(ring) + (Ga > G ? 64 : 0);
  return (bytes + 15) & ~size_t(15);
}

__device__ __forceinline__ uint2 lds64(uint32_t addr) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
}

#ifndef AP_DUAL_HF_ROWS
#define AP_DUAL_HF_ROWS AP_HF_ROWS   // fp16 keys: rows of each quad whose V' is formed by two HADD2s
#endif
#ifndef AP_DUAL_MINB32
#define AP_DUAL_MINB32 12  // resident warps per SM the R = 32 dual shapes are compiled for
#endif
#ifndef AP_DUAL_MINB32_L8
#define AP_DUAL_MINB32_L8 9   // 9 and 12 both mean 3 warps per scheduler (168 registers); ptxas schedules
#endif                        // the L = 8 shapes ~2% better with 9 (C5 136.4 vs 139.3 ms per 8192 rows)
#ifndef AP_DUAL_MINB16
#define AP_DUAL_MINB16 12  // same for the R = 16 shapes
#endif
#ifndef AP_DUAL_HF_MOD
#define AP_DUAL_HF_MOD 4      // ... of every AP_DUAL_HF_MOD rows (1 in 4: 3, 5, 6, 8 and 3 in 8 measured slower or equal)
#endif
#ifndef AP_DUAL_HF_PHASE0
#define AP_DUAL_HF_PHASE0 0   // which row of every four takes the fp16 form, pair 0 / pair 1
#endif
#ifndef AP_DUAL_HF_PHASE1
#define AP_DUAL_HF_PHASE1 0
#endif
#ifndef AP_DUAL_SUBUNROLL
#define AP_DUAL_SUBUNROLL 1
#endif

template <int L, int R, int K, bool DENSE, bool HF>
__global__ void __launch_bounds__(32, R <= 8 ? 16 : (R <= 24 ? AP_DUAL_MINB16 : (L == 32 ? 8 : (L >= 8 ? AP_DUAL_MINB32_L8 : AP_DUAL_MINB32))))
combd_kernel(const CombParams p) {
  constexpr int kHfRows = HF ? AP_DUAL_HF_ROWS : 0;
  constexpr int kSU = AP_DUAL_SUBUNROLL;
  static_assert(L >= 4 && L <= 32, "lane groups of 4..32 lanes");
  static_assert(R % (4 * K) == 0, "bands must hold whole LDS.128 quads");
  constexpr int G = 32 / L;          // real groups; lanes >= G*L form an idle phantom group
  constexpr int Ga = groups_alloc(L);
  constexpr int CS = dual_cs(L, R);
  constexpr int Q = R / 4;
  constexpr int RB = R / K;
  constexpr int QB = RB / 4;
  constexpr int VB = L * K;
  extern __shared__ __align__(16) unsigned char smem[];

  const uint32_t lane = lane_id();
  const uint32_t g = lane / L;
  const uint32_t j = lane % L;
  uint4* tbl = reinterpret_cast<uint4*>(smem);                        // [sigma][CS]: L runs of quads (dual_base)
  const size_t tbytes = size_t(p.sigma) * CS * 16;
  constexpr int RSG = ring_stride(L, kChunk);
  uint32_t* ring0 = reinterpret_cast<uint32_t*>(smem + tbytes) + g * RSG;
  uint32_t* ring1 = ring0 + Ga * RSG;
  const uint32_t okb = uint32_t(__cvta_generic_to_shared(smem + tbytes)) +
                       ((2 * Ga * RSG * 4 + 15) & ~15u) + g * uint32_t(ok_stride(p.ring));
  // the phantom group folds every ok slot onto its 64-byte scratch
  const uint32_t okmask = g < uint32_t(G) ? p.ring - 1 : 0u;

  const uint32_t npairs = (p.rows + 1) / 2;
  const uint32_t ngroups = (npairs + 2 * G - 1) / (2 * G);
  const uint32_t gsplit = min(p.g_split, ngroups);
  const uint64_t split_tasks = uint64_t(gsplit) * p.nseg;
  const uint64_t ntasks = split_tasks + uint64_t(ngroups - gsplit) * p.nseg2;
  const uint64_t wstride = uint64_t(gridDim.x);
  if (p.sigma_cap != 0xFFFFFFFFu && *p.sigma_dev > p.sigma_cap) {   // speculative plan too small
    if (threadIdx.x == 0) *p.abort_flag = 1u;
    return;
  }

  for (uint64_t task = blockIdx.x; task < ntasks; task = next_task(p, task, wstride, lane, ntasks)) {
    CombParams pt = p;
    uint32_t pg, seg;
    if (task < split_tasks) {
      pg = uint32_t(task / p.nseg);
      seg = uint32_t(task % p.nseg);
    } else {
      pg = gsplit + uint32_t((task - split_tasks) / p.nseg2);
      seg = uint32_t((task - split_tasks) % p.nseg2);
      pt.S = p.S2;
    }
    const uint32_t r0 = 4 * (pg * G + g);   // grid rows r0, r0+1 (pair 0) and r0+2, r0+3 (pair 1)
    const bool real_g = g < uint32_t(G);
    const bool has0 = real_g && r0 < p.rows, has1 = real_g && r0 + 1 < p.rows, has2 = real_g && r0 + 2 < p.rows,
               has3 = real_g && r0 + 3 < p.rows;
    const uint32_t c0 = seg * pt.S;
    const uint32_t nseg_cols = min(pt.S + p.W - 1, p.N - c0);
    const uint32_t nsteps = nseg_cols + VB - 1;
    const uint32_t nch = (nsteps + kChunk - 1) / kChunk;

    // ---- mask table: word of warp row i = (x[rw+i] == a) | (x[rw+1+i] == a) << 16 with rw the
    // first grid row of the warp's group 0; group g's strip row i is warp row 4g + i
    __syncwarp();
    {
      const uint32_t rw = 4 * pg * G;   // h = 1: strip s starts at x[s]
      for (uint32_t e = lane; e < uint32_t(L * (G + Q)); e += 32) {
        const uint32_t jj = e / (G + Q), c = e % (G + Q);
        const uint32_t jbase = dual_base_rt<L, R>(jj);
        uint32_t xc[5];
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          const uint32_t idx = rw + jj * R + 4 * c + k;
          uint32_t cv = 0x1FFu;                  // never equals a code
          if (idx < p.xlen) {
            cv = p.xcode[idx];
            if (cv == 0xFFu) cv = 0x1FFu;        // byte absent from y
          }
          xc[k] = cv;
        }
        for (uint32_t a = 0; a < p.sigma; ++a) {
          uint32_t wv[4];
#pragma unroll
          for (int k = 0; k < 4; ++k)
            wv[k] = (xc[k] == a ? 0x00008000u : 0u) | (xc[k + 1] == a ? 0x80000000u : 0u);
          tbl[a * CS + jbase + c] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
        }
      }
      for (uint32_t k = j; k <= okmask; k += L) sts_u32(okb + 4 * k, 0u);
    }
    __syncwarp();

    const uint32_t tlb = uint32_t(__cvta_generic_to_shared(tbl + dual_base_rt<L, R>(j) + (real_g ? g : uint32_t(G - 1))));
    const uint4* yq = reinterpret_cast<const uint4*>((j == 0 ? p.ycol : p.ycol_zero) + c0);
    const uint32_t nz = j != 0 ? 1u : 0u;
    const uint32_t finc = j == 0 ? 0x00010001u : 0u;

    uint32_t V0[R], V1[R];
#pragma unroll
    for (int rho = 0; rho < R; ++rho) { V0[rho] = 0u; V1[rho] = 0u; }
    uint32_t tb0[K], tb1[K], cd[K];
    uint32_t tb0_prev = 0u, tb1_prev = 0u;
#pragma unroll
    for (int b = 0; b < K; ++b) { tb0[b] = 0u; tb1[b] = 0u; cd[b] = 0u; }
    int32_t kbase = -int32_t(p.W) - 1 - (HF ? int32_t(kHfBase) : 0);
    uint32_t fresh = j == 0 ? uint32_t(-kbase) * 0x00010001u : 0u;
    const uint32_t rebase_by = HF ? (kHfRebaseAt - kHfBase - 2 * kChunk - VB - p.W) : kRebaseBy;
    const uint32_t one = p.one;
    uint32_t run0 = 0u, run1 = 0u;
    uint32_t hits0 = 0u, hits1 = 0u, hits2 = 0u, hits3 = 0u;

    uint4 qa = __ldg(yq), qb = __ldg(yq + 1);   // this sub's 8 column words; the next 8 load during it
    cd[0] = qa.x;
    uint32_t nsub = 0;

    for (uint32_t ch = 0; ch < nch; ++ch) {
#pragma unroll kSU
      for (int sub = 0; sub < kChunk / 8; ++sub, ++nsub) {
        const uint4 na = __ldg(yq + 2 * nsub + 2), nb = __ldg(yq + 2 * nsub + 3);
        uint32_t* rs0 = ring0 + sub * 8;
        uint32_t* rs1 = ring1 + sub * 8;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          uint4 nfq[Q];
          uint2 nfx[K];
#pragma unroll
          for (int b = 0; b < K; ++b) {
            const uint32_t tbase = imad(cd[b], one, tlb);   // column word = the code's table offset
#pragma unroll
            for (int qq = 0; qq < QB; ++qq) nfq[b * QB + qq] = lds128(tbase + (b * QB + qq) * 16);
            nfx[b] = lds64(tbase + (b + 1) * QB * 16);        // first two words of the quad below the band
          }
          uint32_t tin0[K], tin1[K];
          {
            const uint32_t s0 = shfl_up1<L>(tb0[K - 1]);
            const uint32_t s1 = shfl_up1<L>(tb1[K - 1]);
            tin0[0] = imad(s0, nz, fresh);
            tin1[0] = imad(s1, nz, fresh);
#pragma unroll
            for (int b = 1; b < K; ++b) { tin0[b] = tb0[b - 1]; tin1[b] = tb1[b - 1]; }
          }
          fresh = imad(fresh, one, finc);
#pragma unroll
          for (int b = 0; b < K; ++b) {
            uint32_t m[RB + 2];
#pragma unroll
            for (int qq = 0; qq < QB; ++qq) {
              const uint4 w4 = nfq[b * QB + qq];
              m[4 * qq] = w4.x; m[4 * qq + 1] = w4.y; m[4 * qq + 2] = w4.z; m[4 * qq + 3] = w4.w;
            }
            m[RB] = nfx[b].x;
            m[RB + 1] = nfx[b].y;
            uint32_t t0 = tin0[b], t1 = tin1[b];
#pragma unroll
            for (int i = 0; i < RB; ++i) {
              {
                uint32_t& v = V0[b * RB + i];
                const uint32_t d = __viaddmax_s16x2(t0, m[i], v);
                if (((i + AP_DUAL_HF_PHASE0) % AP_DUAL_HF_MOD) < kHfRows) v = hadd2u(hsub2u(v, d), t0);
                else v = lop3_xor(v, t0, d);
                t0 = d;
              }
              {
                uint32_t& v = V1[b * RB + i];
                const uint32_t d = __viaddmax_s16x2(t1, m[i + 2], v);
                if (((i + AP_DUAL_HF_PHASE1) % AP_DUAL_HF_MOD) < kHfRows) v = hadd2u(hsub2u(v, d), t1);
                else v = lop3_xor(v, t1, d);
                t1 = d;
              }
            }
            tb0[b] = t0;
            tb1[b] = t1;
          }
          if (u & 1) {
            if (j == L - 1) {
              *reinterpret_cast<uint2*>(rs0 + u - 1) = make_uint2(tb0_prev, tb0[K - 1]);
              *reinterpret_cast<uint2*>(rs1 + u - 1) = make_uint2(tb1_prev, tb1[K - 1]);
            }
          } else {
            tb0_prev = tb0[K - 1];
            tb1_prev = tb1[K - 1];
          }
          {
            const uint32_t ynew = u == 0 ? qa.y : u == 1 ? qa.z : u == 2 ? qa.w : u == 3 ? qb.x :
                                  u == 4 ? qb.y : u == 5 ? qb.z : u == 6 ? qb.w : na.x;
            const uint32_t sh = shfl_up1<L>(cd[K - 1]);
#pragma unroll
            for (int b = K - 1; b > 0; --b) cd[b] = cd[b - 1];
            cd[0] = imad(sh, nz, ynew);
          }
        }
        qa = na; qb = nb;
      }
      __syncwarp();

      // ---- window extraction of both pairs (shared ok-flag ring: bytes 0/2 and 1/3)
      {
        constexpr int CPL = (kChunk + L - 1) / L;
        const int32_t E0 = int32_t(ch * kChunk) - (VB - 1);
        const uint32_t rmask = okmask;
        const bool interior = E0 >= int32_t(p.W) - 1 &&
                              E0 + kChunk <= min(int32_t(nseg_cols), int32_t(pt.S + p.W) - 1);
        uint32_t cab0[CPL], cab1[CPL], o[CPL], o0[CPL], o1[CPL];
        if (interior) {
          extract_scatter<L, kChunk, false, 0>(pt, ring0, okb, rmask, j, E0, nseg_cols, kbase, cab0);
          extract_scatter<L, kChunk, false, 1>(pt, ring1, okb, rmask, j, E0, nseg_cols, kbase, cab1);
          __syncwarp();
          extract_flags<L, kChunk, false>(pt, okb, rmask, j, E0, nseg_cols, o);
        } else {
          extract_scatter<L, kChunk, true, 0>(pt, ring0, okb, rmask, j, E0, nseg_cols, kbase, cab0);
          extract_scatter<L, kChunk, true, 1>(pt, ring1, okb, rmask, j, E0, nseg_cols, kbase, cab1);
          __syncwarp();
          extract_flags<L, kChunk, true>(pt, okb, rmask, j, E0, nseg_cols, o);
        }
        extract_clear<L, kChunk>(pt, okb, rmask, j, E0);
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          o0[c] = o[c] & 0x00010001u;
          o1[c] = (o[c] >> 8) & 0x00010001u;
        }
        if (interior) {
          extract_out<L, kChunk, DENSE, false>(pt, j, g, lane, E0, nseg_cols, c0, cab0, o0, r0, r0 + 1, has0, has1,
                                               run0, hits0, hits1);
          extract_out<L, kChunk, DENSE, false>(pt, j, g, lane, E0, nseg_cols, c0, cab1, o1, r0 + 2, r0 + 3, has2, has3,
                                               run1, hits2, hits3);
        } else {
          extract_out<L, kChunk, DENSE, true>(pt, j, g, lane, E0, nseg_cols, c0, cab0, o0, r0, r0 + 1, has0, has1,
                                              run0, hits0, hits1);
          extract_out<L, kChunk, DENSE, true>(pt, j, g, lane, E0, nseg_cols, c0, cab1, o1, r0 + 2, r0 + 3, has2, has3,
                                              run1, hits2, hits3);
        }
      }

      // ---- key rebase (saturating at 0)
      if (uint32_t(int32_t((ch + 2) * kChunk) - kbase) >= (HF ? kHfRebaseAt : kRebaseAt)) {
        const uint32_t by = rebase_by * 0x00010001u;
        const uint32_t fl = (HF ? kHfBase : 0u) * 0x00010001u + by;
#pragma unroll
        for (int rho = 0; rho < R; ++rho) {
          V0[rho] = __vmaxu2(V0[rho], fl) - by;
          V1[rho] = __vmaxu2(V1[rho], fl) - by;
        }
#pragma unroll
        for (int b = 0; b < K; ++b) {
          tb0[b] = __vmaxu2(tb0[b], fl) - by;
          tb1[b] = __vmaxu2(tb1[b], fl) - by;
        }
        tb0_prev = __vmaxu2(tb0_prev, fl) - by;
        tb1_prev = __vmaxu2(tb1_prev, fl) - by;
        if (j == 0) fresh -= by;
        kbase += int32_t(rebase_by);
      }
    }
    if constexpr (!DENSE) {
      if (j == 0) {
        if (has0) p.seg_counts[size_t(r0) * p.seg_stride + seg] = hits0;
        if (has1) p.seg_counts[size_t(r0 + 1) * p.seg_stride + seg] = hits1;
        if (has2) p.seg_counts[size_t(r0 + 2) * p.seg_stride + seg] = hits2;
        if (has3) p.seg_counts[size_t(r0 + 3) * p.seg_stride + seg] = hits3;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Dual-pair alignment-score kernel (r = 2, h = 1, w = 4*L): comb2_kernel's cell classes
// (ap_kernels.cuh: ($,$) swap free, ($,real) / (real,$) compare-exchange, real x real table
// cell) with two strip pairs per lane group.  A lane holds RR = 4 real rows (8 blown rows) of
// both pairs; pair 1's mask word of real row i is pair 0's of row i + 2, so a step reads 6
// words.  One linear table per warp, T[code][warp real row / 4]: group g's rows are group 0's
// shifted by 4 = one quad, lane (g, j) reads quad g + j, so every quarter warp of an LDS.128
// reads 8 consecutive quads (conflict-free) and the table is 16 * (G + L) bytes per code, rounded
// up to 128, instead of 512 (C4, 20 codes: 7.7 KB per warp).  The per-step overhead of comb2_kernel (code
// feed, table address, shuffles, ring stores: 16 of 44 issue slots on C4) is shared by twice
// the cells.
KernelFn pick_r2_dual(int l, int k, bool dense);

// table quads per code: G + L, rounded up to 8 quads (128 B) so that lanes holding different
// codes (lane j is at column s - j) still fall on bank group (g + j) mod 8
__host__ __device__ constexpr int r2d_nq(int L) { return (32 / L + L + 7) / 8 * 8; }
__host__ __device__ inline size_t comb2d_smem_per_warp(int L, uint32_t sigma, uint32_t ring) {
  const int G = 32 / L;
  const size_t bytes = size_t(16) * sigma * r2d_nq(L)
       + ((size_t(2) * G * ring_stride(L, 2 * kChunk) * 4 + 15) & ~size_t(15))
       + size_t(G) * ok_stride(ring);
  return (bytes + 15) & ~size_t(15);
}

#ifndef AP_R2D_MINB
#define AP_R2D_MINB 16
#endif
#ifndef AP_R2D_SUBUNROLL
#define AP_R2D_SUBUNROLL 2
#endif

template <int L, int K, bool DENSE>
__global__ void __launch_bounds__(32, AP_R2D_MINB)
comb2d_kernel(const CombParams p) {
  static_assert(32 % L == 0 && L >= 4 && (K == 1 || K == 2), "bad shape");
  constexpr int G = 32 / L;
  constexpr int RR = 4;            // real rows per lane
  constexpr int R = 2 * RR;        // blown rows per lane
  constexpr int RRB = RR / K;      // real rows per band
  constexpr int NB = 2 * kChunk;   // blown bottom columns per chunk
  constexpr int kSU2 = AP_R2D_SUBUNROLL;
  constexpr int NQ = r2d_nq(L);    // table quads per code (G + L used)
  constexpr int VB = L * K;
  extern __shared__ __align__(16) unsigned char smem[];

  const uint32_t lane = lane_id();
  const uint32_t g = lane / L;
  const uint32_t j = lane % L;
  uint4* tbl = reinterpret_cast<uint4*>(smem);                        // [sigma][NQ]
  const size_t tbytes = size_t(p.sigma) * NQ * 16;
  constexpr int RS = ring_stride(L, NB);
  uint32_t* ring0 = reinterpret_cast<uint32_t*>(smem + tbytes) + g * RS;
  uint32_t* ring1 = ring0 + G * RS;
  const uint32_t okb = uint32_t(__cvta_generic_to_shared(smem + tbytes)) +
                       ((2 * G * RS * 4 + 15) & ~15u) + g * uint32_t(ok_stride(p.ring));

  const uint32_t npairs = (p.rows + 1) / 2;
  const uint32_t ngroups = (npairs + 2 * G - 1) / (2 * G);
  const uint32_t gsplit = min(p.g_split, ngroups);
  const uint64_t split_tasks = uint64_t(gsplit) * p.nseg;
  const uint64_t ntasks = split_tasks + uint64_t(ngroups - gsplit) * p.nseg2;
  const uint64_t wstride = uint64_t(gridDim.x);
  if (p.sigma_cap != 0xFFFFFFFFu && *p.sigma_dev > p.sigma_cap) {   // speculative plan too small
    if (threadIdx.x == 0) *p.abort_flag = 1u;
    return;
  }

  for (uint64_t task = blockIdx.x; task < ntasks; task = next_task(p, task, wstride, lane, ntasks)) {
    CombParams pt = p;
    uint32_t pg, seg;
    if (task < split_tasks) {
      pg = uint32_t(task / p.nseg);
      seg = uint32_t(task % p.nseg);
    } else {
      pg = gsplit + uint32_t((task - split_tasks) / p.nseg2);
      seg = uint32_t((task - split_tasks) % p.nseg2);
      pt.S = p.S2;
    }
    const uint32_t r0 = 4 * (pg * G + g);
    const bool has0 = r0 < p.rows, has1 = r0 + 1 < p.rows, has2 = r0 + 2 < p.rows, has3 = r0 + 3 < p.rows;
    const uint32_t c0 = seg * pt.S;                        // blown, multiple of 64
    const uint32_t c0r = c0 >> 1;                          // raw, multiple of 32
    const uint32_t nseg_cols = min(pt.S + p.W - 1, p.N - c0);
    const uint32_t nraw = (nseg_cols + 1) >> 1;
    const uint32_t nsteps = nraw + VB - 1;
    const uint32_t nch = (nsteps + kChunk - 1) / kChunk;

    // ---- mask table (real rows, real codes): word of warp real row u = (x[rw+u] == a) |
    // (x[rw+1+u] == a) << 16, rw = the first grid row of the warp's group 0
    __syncwarp();
    {
      const uint32_t rw = 4 * pg * G;
      for (uint32_t c = lane; c < uint32_t(G + L); c += 32) {
        uint32_t xc[5];
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          const uint32_t idx = rw + 4 * c + k;
          uint32_t cv = 0x1FFu;
          if (idx < p.xlen) {
            cv = p.xcode[idx];
            if (cv == 0xFFu) cv = 0x1FFu;
          }
          xc[k] = cv;
        }
        for (uint32_t a = 0; a < p.sigma; ++a) {
          uint32_t wv[4];
#pragma unroll
          for (int k = 0; k < 4; ++k)
            wv[k] = (xc[k] == a ? 0x00008000u : 0u) | (xc[k + 1] == a ? 0x80000000u : 0u);
          tbl[a * NQ + c] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
        }
      }
      for (uint32_t k = j; k < p.ring; k += L) sts_u32(okb + 4 * k, 0u);
    }
    __syncwarp();

    const uint32_t tlb = uint32_t(__cvta_generic_to_shared(tbl + g + j));
    const uint4* yq = reinterpret_cast<const uint4*>((j == 0 ? p.ycol : p.ycol_zero) + c0r);
    const uint32_t nz = j != 0 ? 1u : 0u;
    const uint32_t finc = j == 0 ? 0x00020002u : 0u;
    const uint32_t one = p.one;

    uint32_t V0[R], V1[R];
#pragma unroll
    for (int i = 0; i < R; ++i) { V0[i] = 0u; V1[i] = 0u; }
    uint32_t tbD0[K], tbR0[K], tbD1[K], tbR1[K], cd[K];
#pragma unroll
    for (int b = 0; b < K; ++b) { tbD0[b] = 0u; tbR0[b] = 0u; tbD1[b] = 0u; tbR1[b] = 0u; cd[b] = 0u; }
    int32_t kbase = -int32_t(p.W) - 1;
    uint32_t freshD = j == 0 ? uint32_t(-kbase) * 0x00010001u : 0u;   // key of blown column 2s (lane 0)
    uint32_t freshR = j == 0 ? freshD + 0x00010001u : 0u;             // ... and of 2s + 1
    uint32_t run0 = 0u, run1 = 0u, hits0 = 0u, hits1 = 0u, hits2 = 0u, hits3 = 0u;

    uint4 qa = __ldg(yq), qb = __ldg(yq + 1);
    cd[0] = qa.x;
    uint32_t nsub = 0;

    for (uint32_t ch = 0; ch < nch; ++ch) {
#pragma unroll kSU2
      for (int sub = 0; sub < kChunk / 8; ++sub, ++nsub) {
        const uint4 na = __ldg(yq + 2 * nsub + 2), nb = __ldg(yq + 2 * nsub + 3);
        uint32_t* rs0 = ring0 + sub * 16;
        uint32_t* rs1 = ring1 + sub * 16;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          // mask words of this step: band b needs real rows [b*RRB, b*RRB + RRB + 2)
          uint32_t m[K][RRB + 2];
          if constexpr (K == 1) {
            const uint32_t tbase = imad(cd[0], one, tlb);
            const uint4 w4 = lds128(tbase);
            const uint2 w2 = lds64(tbase + 16);
            m[0][0] = w4.x; m[0][1] = w4.y; m[0][2] = w4.z; m[0][3] = w4.w; m[0][4] = w2.x; m[0][5] = w2.y;
          } else {
            const uint4 w4 = lds128(imad(cd[0], one, tlb));
            m[0][0] = w4.x; m[0][1] = w4.y; m[0][2] = w4.z; m[0][3] = w4.w;
            const uint32_t tb1 = imad(cd[K - 1], one, tlb);
            const uint2 wa = lds64(tb1 + 8), wb = lds64(tb1 + 16);
            m[K - 1][0] = wa.x; m[K - 1][1] = wa.y; m[K - 1][2] = wb.x; m[K - 1][3] = wb.y;
          }
          uint32_t tinD0[K], tinR0[K], tinD1[K], tinR1[K];
          {
            const uint32_t a0 = shfl_up1<L>(tbD0[K - 1]);
            const uint32_t a1 = shfl_up1<L>(tbR0[K - 1]);
            const uint32_t a2 = shfl_up1<L>(tbD1[K - 1]);
            const uint32_t a3 = shfl_up1<L>(tbR1[K - 1]);
            tinD0[0] = imad(a0, nz, freshD);
            tinR0[0] = imad(a1, nz, freshR);
            tinD1[0] = imad(a2, nz, freshD);
            tinR1[0] = imad(a3, nz, freshR);
#pragma unroll
            for (int b = 1; b < K; ++b) {
              tinD0[b] = tbD0[b - 1]; tinR0[b] = tbR0[b - 1];
              tinD1[b] = tbD1[b - 1]; tinR1[b] = tbR1[b - 1];
            }
          }
          freshD = imad(freshD, one, finc);
          freshR = imad(freshR, one, finc);
#pragma unroll
          for (int b = 0; b < K; ++b) {
#pragma unroll
            for (int pr = 0; pr < 2; ++pr) {
              uint32_t* V = pr ? V1 : V0;
              uint32_t t = pr ? tinD1[b] : tinD0[b];           // blown column 2c: $
#pragma unroll
              for (int i = 0; i < RRB; ++i) {
                uint32_t& vs = V[b * 2 * RRB + 2 * i];         // $ row: match -> swap
                const uint32_t sw = vs;
                vs = t;
                t = sw;
                uint32_t& vr = V[b * 2 * RRB + 2 * i + 1];     // real row: mismatch
                const uint32_t d = __vmaxu2(vr, t);
                vr = __vminu2(vr, t);
                t = d;
              }
              (pr ? tbD1[b] : tbD0[b]) = t;
              t = pr ? tinR1[b] : tinR0[b];                    // blown column 2c+1: real character
#pragma unroll
              for (int i = 0; i < RRB; ++i) {
                uint32_t& vs = V[b * 2 * RRB + 2 * i];         // $ row: mismatch; min on the FMA pipe
                const uint32_t d0 = __vmaxu2(vs, t);
                vs = imad(d0, p.minus_one, imad(vs, one, t));  // vs + t - max (16-bit halves never carry)
                t = d0;
                uint32_t& vr = V[b * 2 * RRB + 2 * i + 1];     // real x real: table
                const uint32_t d1 = __viaddmax_s16x2(t, m[b][i + 2 * pr], vr);
                vr = lop3_xor(vr, t, d1);
                t = d1;
              }
              (pr ? tbR1[b] : tbR0[b]) = t;
            }
          }
          if (j == L - 1) {
            *reinterpret_cast<uint2*>(rs0 + 2 * u) = make_uint2(tbD0[K - 1], tbR0[K - 1]);
            *reinterpret_cast<uint2*>(rs1 + 2 * u) = make_uint2(tbD1[K - 1], tbR1[K - 1]);
          }
          {
            const uint32_t ynew = u == 0 ? qa.y : u == 1 ? qa.z : u == 2 ? qa.w : u == 3 ? qb.x :
                                  u == 4 ? qb.y : u == 5 ? qb.z : u == 6 ? qb.w : na.x;
            const uint32_t sh = shfl_up1<L>(cd[K - 1]);
#pragma unroll
            for (int b = K - 1; b > 0; --b) cd[b] = cd[b - 1];
            cd[0] = imad(sh, nz, ynew);
          }
        }
        qa = na; qb = nb;
      }
      __syncwarp();

      // ---- window extraction of both pairs (shared ok-flag ring: bytes 0/2 and 1/3)
      {
        constexpr int CPL = NB / L;
        const int32_t E0 = 2 * (int32_t(ch * kChunk) - int32_t(VB - 1));
        const uint32_t rmask = p.ring - 1;
        const bool interior = E0 >= int32_t(p.W) - 1 &&
                              E0 + NB <= min(int32_t(nseg_cols), int32_t(pt.S + p.W) - 1);
        uint32_t cab0[CPL], cab1[CPL], o[CPL], o0[CPL], o1[CPL];
        if (interior) {
          extract_scatter<L, NB, false, 0>(pt, ring0, okb, rmask, j, E0, nseg_cols, kbase, cab0);
          extract_scatter<L, NB, false, 1>(pt, ring1, okb, rmask, j, E0, nseg_cols, kbase, cab1);
          __syncwarp();
          extract_flags<L, NB, false>(pt, okb, rmask, j, E0, nseg_cols, o);
        } else {
          extract_scatter<L, NB, true, 0>(pt, ring0, okb, rmask, j, E0, nseg_cols, kbase, cab0);
          extract_scatter<L, NB, true, 1>(pt, ring1, okb, rmask, j, E0, nseg_cols, kbase, cab1);
          __syncwarp();
          extract_flags<L, NB, true>(pt, okb, rmask, j, E0, nseg_cols, o);
        }
        extract_clear<L, NB>(pt, okb, rmask, j, E0);
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          o0[c] = o[c] & 0x00010001u;
          o1[c] = (o[c] >> 8) & 0x00010001u;
        }
        if (interior) {
          extract_out<L, NB, DENSE, false>(pt, j, g, lane, E0, nseg_cols, c0, cab0, o0, r0, r0 + 1, has0, has1,
                                           run0, hits0, hits1);
          extract_out<L, NB, DENSE, false>(pt, j, g, lane, E0, nseg_cols, c0, cab1, o1, r0 + 2, r0 + 3, has2, has3,
                                           run1, hits2, hits3);
        } else {
          extract_out<L, NB, DENSE, true>(pt, j, g, lane, E0, nseg_cols, c0, cab0, o0, r0, r0 + 1, has0, has1,
                                          run0, hits0, hits1);
          extract_out<L, NB, DENSE, true>(pt, j, g, lane, E0, nseg_cols, c0, cab1, o1, r0 + 2, r0 + 3, has2, has3,
                                          run1, hits2, hits3);
        }
      }

      if (uint32_t(int32_t((ch + 2) * NB) - kbase) >= kRebaseAt) {
        const uint32_t by = kRebaseBy * 0x00010001u;
#pragma unroll
        for (int i = 0; i < R; ++i) {
          V0[i] = __vmaxu2(V0[i], by) - by;
          V1[i] = __vmaxu2(V1[i], by) - by;
        }
#pragma unroll
        for (int b = 0; b < K; ++b) {
          tbD0[b] = __vmaxu2(tbD0[b], by) - by; tbR0[b] = __vmaxu2(tbR0[b], by) - by;
          tbD1[b] = __vmaxu2(tbD1[b], by) - by; tbR1[b] = __vmaxu2(tbR1[b], by) - by;
        }
        if (j == 0) { freshD -= by; freshR -= by; }
        kbase += int32_t(kRebaseBy);
      }
    }
    if constexpr (!DENSE) {
      if (j == 0) {
        if (has0) p.seg_counts[size_t(r0) * p.seg_stride + seg] = hits0;
        if (has1) p.seg_counts[size_t(r0 + 1) * p.seg_stride + seg] = hits1;
        if (has2) p.seg_counts[size_t(r0 + 2) * p.seg_stride + seg] = hits2;
        if (has3) p.seg_counts[size_t(r0 + 3) * p.seg_stride + seg] = hits3;
      }
    }
  }
}

}  // namespace apk
