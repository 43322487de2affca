// Persistent, warp-specialised 3M complex FP64 GEMM with TMA staging (sm_100a).
//
// Same work lists, warp tiling (8 MMA warps of 32 x 16 on a 64 x 64 CTA tile), Gauss products
// (T1 = Ar Br, T2 = Ai Bi, T3 = (Ar + Ai)(Br + Bi) on DMMA.8x8x4), sub-tile skipping at ragged
// edges and epilogues as zgemm3m_kernel (zgemm.cuh); the operand staging and scheduling differ:
//
//   * one CTA per SM (grid = min(tiles, SMs)) takes tiles from a list ordered by cost (largest
//     first), claimed dynamically through a global counter: list scheduling that lets faster SMs
//     (e.g. those closer to the L2 half holding the operands) absorb the tail;
//   * a producer warp streams every K stage (8 complex k) of op(A) and op(B) of the CTA's tiles into
//     a ring of S stages by TMA (cp.async.bulk.tensor, one lane) from per-item tensor maps --
//     out-of-range rows, columns and k are zero-filled by the TMA unit, so ragged edges need no
//     predication -- running up to S stages ahead across tile boundaries, so the next tile's operands
//     land while the MMA warps run the current tile's epilogue; the tile index rides with the first
//     stage of each tile;
//   * a "full" mbarrier per stage (armed with the 16 KB byte count) and an "empty" mbarrier (one
//     arrival per MMA warp): no block-wide barrier in the main loop, warps drift within the ring;
//   * dense 128-byte rows with the 128B swizzle (16-byte chunk c of row r stored at c ^ (r & 7)).
//     Row-major operands ([m][k], op(B) = B^dag as [n][k]) are one 64-row box; k-major operands
//     ([k][n], op(A) = A^dag as [k][m]) are eight 8 x 8 boxes, one per 8-column block.  With the
//     swizzle, lane (r, c) of a DMMA fragment reads k = 2c + s for k-step s: every 8-lane phase
//     of an LDS.128 touches 8 distinct 16-byte bank groups (conflict-free), for both layouts.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "zgemm.cuh"

namespace sqoc {

// Operand-sum planes (build with -DSQOC_PT_SUMS=1; default off): two helper warps form the Gauss operand
// sums Re + Im of every landed stage once per CTA (512 per operand) and store them beside the tiles, so
// the MMA warps issue no DADDs (each of the 8 warps forms the sums of its own fragments otherwise:
// 3072 DADD lanes per stage; the bare loop loses 8% to them, profiles/r02_dmma_loop_probe.txt v1 vs
// v2).  Measured and rejected (r02, cfg 3, GEMM ms per 6 slices, same day): 329.0 with the DADDs,
// 371.1 with the planes (434.0 before the helper's 16 loads were batched) -- the 9-stage ring, the
// extra full -> ready hop and 12 more LDS.64 per MMA warp and stage cost more than the DADDs did.
#ifndef SQOC_PT_SUMS
#define SQOC_PT_SUMS 0
#endif
constexpr bool kPtSums = SQOC_PT_SUMS != 0;
#ifndef SQOC_PT_STAGES
#define SQOC_PT_STAGES (SQOC_PT_SUMS ? 9 : 12)
#endif
constexpr int PT_STAGES = SQOC_PT_STAGES;
constexpr int TMA_STAGE_BYTES = 2 * GBM * 8 * 16;  // A + B tiles: 64 x 8 complex each (the TMA byte count)
constexpr int PT_SUM_BYTES = GBM * 8 * 8;           // one operand's sums: 64 x 8 doubles
constexpr int PT_SLOT_BYTES = TMA_STAGE_BYTES + (kPtSums ? 2 * PT_SUM_BYTES : 0);  // ring slot stride
constexpr int PT_HELPERS = kPtSums ? 2 : 0;         // helper warps (A sums, B sums)
constexpr size_t PT_SMEM = (size_t)PT_STAGES * PT_SLOT_BYTES + 3 * PT_STAGES * 8 + 1024;  // ring + barriers + align

// per work-list item and K segment: tensor maps of A and B in both staging orientations
// (m[6 seg + 0] A as [m][k], + 1 A as [k][m] (op = conj-transpose), + 2 B as [k][n], + 3 B as [n][k],
//  + 4 / + 5: the k-major views of A / B again as 3-D maps (8 columns, k, column block) whose one
//  16 x 8 x 8 box lands as the same eight swizzled 8 x 8 blocks that eight 2-D boxes write -- one TMA
//  instruction instead of eight for tiles whose 64 columns are all inside the full column blocks;
//  the column-block extent is floor(cols / 8), so no box reads past a row's end); unused ones zero
struct alignas(64) ItemMaps {
  CUtensorMap m[12];
  unsigned has3d;  // bit 2 seg + 0 / + 1: the 3-D map of A / B of segment seg was encoded
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_s(uint32_t b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(b) : "memory");
}
__device__ __forceinline__ void mbar_wait_s(uint32_t b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(b),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// Tensor maps live in global memory (uploaded per work list): before the async proxy reads a map whose
// bytes the host wrote, the generic -> tensormap proxy acquire fence of the CUDA programming guide is
// required, or an SM may use a stale cached descriptor of a map that used to live at the same address
// (an earlier engine's list): r02 found first evaluations of fresh engines reading slightly wrong
// operands that way (tools/repeat_check.py).
__device__ __forceinline__ void tensormap_acquire(const CUtensorMap* map) {
  asm volatile("fence.proxy.tensormap::generic.acquire.sys [%0], 128;\n" ::"l"(map) : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

// Issue the TMA copies of K stage kt (segment and k0 from kt) into ring slot `st`.
template <int TA, int TB>
__device__ __forceinline__ void tma_issue_stage(const ItemMaps* mp, const GemmItem& it, int kt, int kt_per_seg,
                                                int m0, int n0, bool a3d, bool b3d, uint8_t* slot, uint64_t* full) {
  const int seg = kt / kt_per_seg;
  const int k0 = (kt - seg * kt_per_seg) * GBK;
  const CUtensorMap* ma = &mp->m[6 * seg + (TA == OP_N ? 0 : 1)];
  const CUtensorMap* mb = &mp->m[6 * seg + (TB == OP_N ? 2 : 3)];
  uint8_t* sA = slot;
  uint8_t* sB = slot + GBM * 8 * 16;
  mbar_arrive_expect(full, TMA_STAGE_BYTES);
  if (TA == OP_N) tma_load_2d(sA, ma, 2 * k0, m0, full);  // [m][k]: one 64-row box
  else if (a3d && (mp->has3d >> (2 * seg) & 1u)) tma_load_3d(sA, &mp->m[6 * seg + 4], 0, k0, m0 >> 3, full);  // [k][m]: 8 blocks, one box
  else
#pragma unroll
    for (int b = 0; b < GBM / 8; ++b) tma_load_2d(sA + b * 1024, ma, 2 * (m0 + 8 * b), k0, full);  // [k][m] blocks
  if (TB != OP_N) tma_load_2d(sB, mb, 2 * k0, n0, full);  // [n][k]: one 64-row box
  else if (b3d && (mp->has3d >> (2 * seg + 1) & 1u)) tma_load_3d(sB, &mp->m[6 * seg + 5], 0, k0, n0 >> 3, full);  // [k][n]: 8 blocks, one box
  else
#pragma unroll
    for (int b = 0; b < GBN / 8; ++b) tma_load_2d(sB + b * 1024, mb, 2 * (n0 + 8 * b), k0, full);  // [k][n] blocks
}

// Warp layout of a tile with R x Cc valid 8 x 8 sub-tiles (R, Cc <= 8): the 8 MMA warps form a
// (8 / WC) x WC grid of th x tw sub-tile warp tiles (th <= 4, tw <= 2: the accumulator array).  Full
// tiles use 2 x 4 warps of 4 x 2; a ragged edge tile picks the grid with the smallest per-warp work
// th * tw that still covers it (d = 1179: the 27-wide edge tiles run 4 x 2 warps of 2 x 2, half the
// DMMAs per warp of the full layout, which would leave 4 of 8 warps idle).
__host__ __device__ inline void pt_layout(int R, int Cc, int& th, int& tw, int& WC) {
  th = 4; tw = 2; WC = 4;
  int best = 8;
  for (int wc = 1; wc <= 8; wc *= 2) {
    const int wr = 8 / wc;
    const int h = (R + wr - 1) / wr, w = (Cc + wc - 1) / wc;
    if (h <= 4 && w <= 2 && h * w < best) {
      best = h * w; th = h; tw = w; WC = wc;
    }
  }
}

struct TileRef {
  int item, m0, n0, local;  // work-list item, tile origin, tile index inside the item (trace partials)
};

// One k-step's fragments (k = 2 lc + s of a stage) with the Gauss operand sums precomputed.
template <int MC, int NC>
struct Frag {
  double ar[MC > 0 ? MC : 1], ai[MC > 0 ? MC : 1], as[MC > 0 ? MC : 1];
  double br[NC > 0 ? NC : 1], bi[NC > 0 ? NC : 1], bs[NC > 0 ? NC : 1];
};

// 16-byte fragment load by 32-bit shared address (LDS.128; a generic pointer derived from the aligned
// dynamic-smem base compiles to generic LD.E.128 with 64-bit address arithmetic)
__device__ __forceinline__ double2 lds_c128(uint32_t addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}

__device__ __forceinline__ double lds_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts_c128(uint32_t addr, double x, double y) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};\n" ::"r"(addr), "d"(x), "d"(y) : "memory");
}

// Sum plane of one operand: [index 0..63][k 0..7] doubles, 64-byte rows, index = the tile row (column
// for k-major operands); k is stored at k ^ ((index >> 1) & 1) so that the 16 lanes of an LDS.64 phase
// (4 rows x 4 k) hit 16 different 8-byte bank pairs.
__device__ __forceinline__ int sum_off(int idx, int k) { return idx * 64 + ((k ^ ((idx >> 1) & 1)) << 3); }

template <int TA, int TB, int MC, int NC>
__device__ __forceinline__ void frag_load(Frag<MC, NC>& f, uint32_t stage, int oa, int ob, int osa, int osb) {
  constexpr int A_MI = (TA == OP_N) ? 8 * 128 : 1024;  // byte stride between the warp's 8-row sub-tiles
  constexpr int B_NI = (TB == OP_N) ? 1024 : 8 * 128;
  const uint32_t sA = stage + oa;
  const uint32_t sB = stage + GBM * 8 * 16 + ob;
#pragma unroll
  for (int mi = 0; mi < MC; ++mi) {
    double2 a = lds_c128(sA + mi * A_MI);
    if (TA == OP_C) a.y = -a.y;
    f.ar[mi] = a.x; f.ai[mi] = a.y;
    if constexpr (kPtSums) f.as[mi] = lds_f64(stage + TMA_STAGE_BYTES + osa + mi * 512);
    else f.as[mi] = a.x + a.y;
  }
#pragma unroll
  for (int ni = 0; ni < NC; ++ni) {
    double2 b = lds_c128(sB + ni * B_NI);
    if (TB == OP_C) b.y = -b.y;
    f.br[ni] = b.x; f.bi[ni] = b.y;
    if constexpr (kPtSums) f.bs[ni] = lds_f64(stage + TMA_STAGE_BYTES + PT_SUM_BYTES + osb + ni * 512);
    else f.bs[ni] = b.x + b.y;
  }
}

// Helper warp: the 512 sums Re +- Im (conjugated operands: Re - Im) of one operand tile of a landed
// stage.  Lane handles tile indices lane and lane + 32.  At step q index idx works on the k pair
// pi((idx >> 1) & 3) ^ q with pi = (0, 2, 3, 1): both pi(a) and pi(a) ^ a are permutations of 0..3, so
// the 8 lanes of a phase read 8 different swizzled 16-byte chunks (chunk = k ^ (idx & 7)) and store
// to 8 different bank groups (group = 4 (idx & 1) + pair).  kmajor: the tile is eight
// [k][8 columns] blocks, else [index][k] rows.
template <bool KMAJOR, bool CONJ>
__device__ __forceinline__ void sum_tile(uint32_t src, uint32_t dst, int lane) {
  double2 v[2][4][2];  // all 16 loads in flight before the first sum (one shared-memory latency per stage)
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int idx = lane + 32 * j;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int p = ((0x78 >> (2 * ((idx >> 1) & 3))) & 3) ^ q;  // k pair (2p, 2p + 1)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int k = 2 * p + h;
        const uint32_t a = KMAJOR ? src + (idx >> 3) * 1024 + k * 128 + ((((idx & 7) ^ k)) << 4)
                                  : src + idx * 128 + (((k ^ (idx & 7))) << 4);
        v[j][q][h] = lds_c128(a);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int idx = lane + 32 * j;
    const int b = (idx >> 1) & 1;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int p = ((0x78 >> (2 * ((idx >> 1) & 3))) & 3) ^ q;
      const double s0 = CONJ ? v[j][q][0].x - v[j][q][0].y : v[j][q][0].x + v[j][q][0].y;
      const double s1 = CONJ ? v[j][q][1].x - v[j][q][1].y : v[j][q][1].x + v[j][q][1].y;
      sts_c128(dst + idx * 64 + p * 16, b ? s1 : s0, b ? s0 : s1);
    }
  }
}

// SQOC_MMA_ORDER 1: the two Gauss products that need no operand sums first, for every sub-tile, then
// the third ones -- the DADDs that form the sums complete behind 2 MC NC DMMAs instead of stalling
// the first sub-tile's third product (the asm statements keep their program order).
#ifndef SQOC_MMA_ORDER
#define SQOC_MMA_ORDER 0
#endif
template <int MC, int NC>
__device__ __forceinline__ void frag_mma(double (&acc)[4][2][3][2], const Frag<MC, NC>& f) {
#if SQOC_MMA_ORDER
#pragma unroll
  for (int mi = 0; mi < MC; ++mi)
#pragma unroll
    for (int ni = 0; ni < NC; ++ni) {
      dmma(acc[mi][ni][0][0], acc[mi][ni][0][1], f.ar[mi], f.br[ni]);
      dmma(acc[mi][ni][1][0], acc[mi][ni][1][1], f.ai[mi], f.bi[ni]);
    }
#pragma unroll
  for (int mi = 0; mi < MC; ++mi)
#pragma unroll
    for (int ni = 0; ni < NC; ++ni) dmma(acc[mi][ni][2][0], acc[mi][ni][2][1], f.as[mi], f.bs[ni]);
#else
#pragma unroll
  for (int mi = 0; mi < MC; ++mi)
#pragma unroll
    for (int ni = 0; ni < NC; ++ni) {
      dmma(acc[mi][ni][0][0], acc[mi][ni][0][1], f.ar[mi], f.br[ni]);
      dmma(acc[mi][ni][1][0], acc[mi][ni][1][1], f.ai[mi], f.bi[ni]);
      dmma(acc[mi][ni][2][0], acc[mi][ni][2][1], f.as[mi], f.bs[ni]);
    }
#endif
}

// kt_total K stages of one tile for a warp whose valid output is MC x NC DMMA sub-tiles; every warp
// waits for and releases every stage (8 releases per slot).  r02 same-box A/B (cfg 3 / cfg 4 ms per
// slice): this plain loop 102.1 / 83.0; a two-deep register pipeline of the fragments 106.2 / 87.0
// (the 168-register cap of 9 warps spills); the producer fused into thread 0 (256 threads) 142 / 112.
template <int TA, int TB, int MC, int NC>
__device__ __forceinline__ void pt_mainloop(double (&acc)[4][2][3][2], uint32_t ring, uint32_t full, uint32_t empty,
                                            uint32_t& slot, uint32_t& phase, int kt_total, const int (&offa)[2],
                                            const int (&offb)[2], const int (&osa)[2], const int (&osb)[2], int lane) {
  for (int kt = 0; kt < kt_total; ++kt) {
    mbar_wait_s(full + 8 * slot, phase);  // `full` is the helpers' ready barrier when the sum planes are on
    if constexpr (MC > 0 && NC > 0) {
      Frag<MC, NC> f;
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        frag_load<TA, TB>(f, ring + slot * PT_SLOT_BYTES, offa[s], offb[s], osa[s], osb[s]);
        frag_mma(acc, f);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive_s(empty + 8 * slot);
    if (++slot == PT_STAGES) { slot = 0; phase ^= 1; }
  }
}

constexpr int PT_THREADS = G3THREADS + 32 + 32 * PT_HELPERS;  // 8 MMA warps + 1 producer warp + helper warps

template <int TA, int TB, int EPI>
__global__ void __launch_bounds__(PT_THREADS, 1) zgemm3m_pt_kernel(const GemmItem* __restrict__ items,
                                                                   const ItemMaps* __restrict__ maps,
                                                                   const TileRef* __restrict__ tiles, int ntiles,
                                                                   int* __restrict__ counter, GemmArgs args) {
  extern __shared__ uint8_t tsm_raw[];
  __shared__ double2 red[G3THREADS / 32][4];
  __shared__ int stage_tile[PT_STAGES];  // tile index announced with a tile's first stage; -1 = done
  __shared__ int stage_info[PT_STAGES][8];  // with it: item, m0, n0, K stages, item m, item n, local (no global loads
                                            // between a tile's announcement and its first DMMA)
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(tsm_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + PT_STAGES * PT_SLOT_BYTES);
  uint64_t* empty = full + PT_STAGES;
  uint64_t* ready = empty + PT_STAGES;  // sum planes written (one arrival per helper warp)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < PT_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], G3THREADS / 32);
      mbar_init(&ready[s], PT_HELPERS > 0 ? PT_HELPERS : 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp == G3THREADS / 32) {
    // ---- producer warp: one lane streams every stage of every tile this CTA takes.  Tiles are
    // claimed dynamically (first blockIdx.x, then gridDim.x + atomicAdd) from the cost-ordered list,
    // so faster SMs take more of the tail (largest-first list scheduling) ----
    if (lane == 0) {
      uint32_t g = 0;
      int t = blockIdx.x;
      while (true) {
        if (t >= ntiles) {  // announce the end through one more (empty) stage
          const uint32_t slot = g % PT_STAGES;
          if (g >= PT_STAGES) mbar_wait(&empty[slot], ((g / PT_STAGES) - 1) & 1);
          stage_tile[slot] = -1;
          mbar_arrive(&full[slot]);
          break;
        }
        const TileRef tr = tiles[t];
        const GemmItem& it = items[tr.item];
        const ItemMaps* mp = maps + tr.item;
        const int kt_per_seg = (it.k + GBK - 1) / GBK;
        const int kt_total = kt_per_seg * it.nseg;
        const bool a3d = tr.m0 + GBM <= (it.m & ~7), b3d = tr.n0 + GBN <= (it.n & ~7);  // all 8 blocks full
        for (int seg = 0; seg < it.nseg; ++seg) {  // the maps this tile's stages use
          const bool a3 = TA != OP_N && a3d && (mp->has3d >> (2 * seg) & 1u);
          const bool b3 = TB == OP_N && b3d && (mp->has3d >> (2 * seg + 1) & 1u);
          tensormap_acquire(&mp->m[6 * seg + (TA == OP_N ? 0 : a3 ? 4 : 1)]);
          tensormap_acquire(&mp->m[6 * seg + (TB != OP_N ? 3 : b3 ? 5 : 2)]);
        }
        for (int kt = 0; kt < kt_total; ++kt, ++g) {
          const uint32_t slot = g % PT_STAGES;
          if (g >= PT_STAGES) mbar_wait(&empty[slot], ((g / PT_STAGES) - 1) & 1);
          if (kt == 0) {
            stage_tile[slot] = t;
            stage_info[slot][0] = tr.item; stage_info[slot][1] = tr.m0; stage_info[slot][2] = tr.n0;
            stage_info[slot][3] = kt_total; stage_info[slot][4] = it.m; stage_info[slot][5] = it.n;
            stage_info[slot][6] = tr.local;
          }
          tma_issue_stage<TA, TB>(mp, it, kt, kt_per_seg, tr.m0, tr.n0, a3d, b3d, ring + slot * PT_SLOT_BYTES,
                                  &full[slot]);
        }
        t = gridDim.x + atomicAdd(counter, 1);
      }
    }
    return;
  }
  if (warp > G3THREADS / 32) {
    // ---- helper warps (sum planes): warp 9 the A tile, warp 10 the B tile of every landed stage ----
    const bool isB = warp == G3THREADS / 32 + 2;
    const uint32_t ring_h = smem_u32(ring), full_h = smem_u32(full), ready_h = smem_u32(ready);
    uint32_t slot = 0, phase = 0;
    while (true) {
      mbar_wait_s(full_h + 8 * slot, phase);
      const int t = *reinterpret_cast<volatile int*>(&stage_tile[slot]);
      if (t < 0) {  // pass the end marker on to the MMA warps
        if (lane == 0) mbar_arrive_s(ready_h + 8 * slot);
        break;
      }
      const GemmItem& it = items[tiles[t].item];
      const int kt_total = ((it.k + GBK - 1) / GBK) * it.nseg;
      for (int kt = 0; kt < kt_total; ++kt) {
        if (kt) mbar_wait_s(full_h + 8 * slot, phase);
        const uint32_t st = ring_h + slot * PT_SLOT_BYTES;
        if (!isB) sum_tile<TA != OP_N, TA == OP_C>(st, st + TMA_STAGE_BYTES, lane);
        else sum_tile<TB == OP_N, TB == OP_C>(st + GBM * 8 * 16, st + TMA_STAGE_BYTES + PT_SUM_BYTES, lane);
        __syncwarp();
        if (lane == 0) mbar_arrive_s(ready_h + 8 * slot);
        if (++slot == PT_STAGES) { slot = 0; phase ^= 1; }
      }
    }
    return;
  }
  const int lr = lane >> 2, lc = lane & 3;
  int rowmaj[2], kmaj[2];  // fragment byte offsets of this lane inside an 8-row / 8-column group, k-steps 0 and 1
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int k = 2 * lc + s;
    rowmaj[s] = lr * 128 + ((k ^ lr) << 4);  // [row][k]: row * 128 + ((k ^ (row & 7)) * 16)
    kmaj[s] = k * 128 + ((lr ^ k) << 4);     // [k][col] 8 x 8 blocks: k * 128 + (((col & 7) ^ k) * 16)
  }
  const uint32_t ring_s = smem_u32(ring), full_s = smem_u32(kPtSums ? ready : full), empty_s = smem_u32(empty);
  int sumo[2];  // sum-plane byte offsets of this lane inside an 8-index group (k-steps 0 and 1)
#pragma unroll
  for (int s = 0; s < 2; ++s) sumo[s] = sum_off(lr, 2 * lc + s);
  uint32_t slot = 0, phase = 0;
  while (true) {
    mbar_wait_s(full_s + 8 * slot, phase);
    const int t = *reinterpret_cast<volatile int*>(&stage_tile[slot]);
    if (t < 0) break;
#ifndef SQOC_TILE_INFO
#define SQOC_TILE_INFO 1
#endif
#if SQOC_TILE_INFO
    volatile const int* info = stage_info[slot];
    const GemmItem& it = items[info[0]];
    const int m0 = info[1], n0 = info[2];
    const int kt_total = info[3];
    const int it_m = info[4], it_n = info[5], tile_local = info[6];
#else
    const TileRef tr = tiles[t];
    const GemmItem& it = items[tr.item];
    const int m0 = tr.m0, n0 = tr.n0;
    const int kt_total = ((it.k + GBK - 1) / GBK) * it.nseg;
    const int it_m = it.m, it_n = it.n, tile_local = tr.local;
#endif
    double acc[4][2][3][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int c = 0; c < 3; ++c) acc[a][b][c][0] = acc[a][b][c][1] = 0.0;
    int th, tw, WC;
    const int R = min(8, (it_m - m0 + 7) / 8), Cc = min(8, (it_n - n0 + 7) / 8);
    pt_layout(R, Cc, th, tw, WC);
    const int wri = warp / WC, wci = warp - wri * WC;
    const int wm = wri * th * 8, wn = wci * tw * 8;
    const int mc = max(0, min(th, R - wri * th));
    const int nc = max(0, min(tw, Cc - wci * tw));
    int offa[2], offb[2], osa[2], osb[2];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      offa[s] = (TA == OP_N ? rowmaj[s] + wm * 128 : kmaj[s] + (wm >> 3) * 1024);
      offb[s] = (TB == OP_N ? kmaj[s] + (wn >> 3) * 1024 : rowmaj[s] + wn * 128);
      osa[s] = sumo[s] + wm * 64;
      osb[s] = sumo[s] + wn * 64;
    }
    switch ((mc == 0 || nc == 0) ? -1 : (mc - 1) * 2 + (nc - 1)) {
      case 7: pt_mainloop<TA, TB, 4, 2>(acc, ring_s, full_s, empty_s, slot, phase, kt_total, offa, offb, osa, osb, lane); break;
      case 6: pt_mainloop<TA, TB, 4, 1>(acc, ring_s, full_s, empty_s, slot, phase, kt_total, offa, offb, osa, osb, lane); break;
      case 5: pt_mainloop<TA, TB, 3, 2>(acc, ring_s, full_s, empty_s, slot, phase, kt_total, offa, offb, osa, osb, lane); break;
      case 4: pt_mainloop<TA, TB, 3, 1>(acc, ring_s, full_s, empty_s, slot, phase, kt_total, offa, offb, osa, osb, lane); break;
      case 3: pt_mainloop<TA, TB, 2, 2>(acc, ring_s, full_s, empty_s, slot, phase, kt_total, offa, offb, osa, osb, lane); break;
      case 2: pt_mainloop<TA, TB, 2, 1>(acc, ring_s, full_s, empty_s, slot, phase, kt_total, offa, offb, osa, osb, lane); break;
      case 1: pt_mainloop<TA, TB, 1, 2>(acc, ring_s, full_s, empty_s, slot, phase, kt_total, offa, offb, osa, osb, lane); break;
      case 0: pt_mainloop<TA, TB, 1, 1>(acc, ring_s, full_s, empty_s, slot, phase, kt_total, offa, offb, osa, osb, lane); break;
      default: pt_mainloop<TA, TB, 0, 0>(acc, ring_s, full_s, empty_s, slot, phase, kt_total, offa, offb, osa, osb, lane); break;
    }
    const bool trace = EPI == EPI_TRACE || (EPI == EPI_MIXED && it.nF > 0);  // uniform per tile
    if (!trace) {
      // the epilogue's item fields in registers: through the reference every store to C forces the
      // pointers to be loaded again (they may alias), 16 dependent global loads per thread and tile
#ifndef SQOC_EP_COPY
#define SQOC_EP_COPY 1
#endif
#if SQOC_EP_COPY
      GemmItem ep{};
      ep.C = it.C; ep.C2 = it.C2; ep.E0 = it.E0; ep.E1 = it.E1; ep.E2 = it.E2; ep.E3 = it.E3;
      ep.ldc = it.ldc; ep.diag = it.diag;
#else
      const GemmItem& ep = it;
#endif
      const int im = it_m, in = it_n;
      const bool mirror = it.herm && n0 > m0;
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni)
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            const int m = m0 + wm + mi * 8 + lr;
            const int n = n0 + wn + ni * 8 + 2 * lc + v;
            if (mi < mc && ni < nc && m < im && n < in) {
              const double t1 = acc[mi][ni][0][v], t2 = acc[mi][ni][1][v], t3 = acc[mi][ni][2][v];
              epi_store(ep, args, m, n, t1 - t2, t3 - t1 - t2);
            }
          }
      if (mirror) {  // Hermitian product, tile above the diagonal: (n, m) = conj (m, n)
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int ni = 0; ni < 2; ++ni)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
              const int m = m0 + wm + mi * 8 + lr;
              const int n = n0 + wn + ni * 8 + 2 * lc + v;
              if (mi < mc && ni < nc && m < im && n < in) {
                const double t1 = acc[mi][ni][0][v], t2 = acc[mi][ni][1][v], t3 = acc[mi][ni][2][v];
                epi_store(ep, args, n, m, t1 - t2, t1 + t2 - t3);
              }
            }
      }
    } else {
      const int nF = it.nF;
      for (int f = 0; f < nF; ++f) {
        const double2* F = it.F + f * it.fstride;
        double sx = 0.0, sy = 0.0;
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int ni = 0; ni < 2; ++ni)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
              const int p = m0 + wm + mi * 8 + lr;
              const int q = n0 + wn + ni * 8 + 2 * lc + v;
              if (mi < mc && ni < nc && p < it_m && q < it_n) {
                const double2 e = F[(size_t)q * it.ldc + p];
                const double t1 = acc[mi][ni][0][v], t2 = acc[mi][ni][1][v], t3 = acc[mi][ni][2][v];
                const double cr = args.alpha * (t1 - t2), ci = args.alpha * (t3 - t1 - t2);
                sx += cr * e.x - ci * e.y;
                sy += cr * e.y + ci * e.x;
              }
            }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          sx += __shfl_xor_sync(0xffffffffu, sx, o);
          sy += __shfl_xor_sync(0xffffffffu, sy, o);
        }
        if (lane == 0) red[warp][f] = make_double2(sx, sy);
      }
      asm volatile("bar.sync 1, %0;\n" ::"n"(G3THREADS) : "memory");
      if (threadIdx.x < nF) {
        double2 s = make_double2(0.0, 0.0);
        for (int w = 0; w < G3THREADS / 32; ++w) { s.x += red[w][threadIdx.x].x; s.y += red[w][threadIdx.x].y; }
        it.tr_out[(size_t)tile_local * nF + threadIdx.x] = s;
      }
      asm volatile("bar.sync 1, %0;\n" ::"n"(G3THREADS) : "memory");  // red[] reused by the next trace tile
    }
  }
}

}  // namespace sqoc
