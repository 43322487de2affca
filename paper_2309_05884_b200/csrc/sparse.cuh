// Sparse-generator products of the large path (sm_100a, FP64 CUDA cores).
//
// The block generators a_k = -i dt H_k of local Hamiltonians are sparse in the symmetry-adapted
// basis: a spin flip or a flip-flop links a D_n orbit to ~n others, so the union pattern of
// a_0..a_K has ~19-41 entries per row at d = 495..1179 (cfg 3) and ~19 at d = 4096 (cfg 4).  The
// slice generator A_j = 2^-s (a_0 + sum_k u_kj a_k) shares that pattern, so every product of the
// propagator scheme with A as a factor -- A2 = A A, A3 = A2 A and the derivative terms A dA, dA A,
// dA2 A -- costs nnz(A) d instead of d^3 (~30x less at d = 1170), and so does the gradient trace
// Tr(U^dag N a_k).  The kernels stage the dense operand's panel in shared memory once per CTA, so
// each dense matrix is read from HBM/L2 about once per product; no tensor cores.
//
//   sp_values_kernel    per slice: values of A_j on the pattern (a CSR value array per block)
//   spmm_cols_kernel    S L: a CTA owns W columns [c0, c0 + W) of an item's output and holds the
//                       panel L[:, c0:c0+W] in shared memory; thread per row i (row-ELL entries):
//                       acc[w] = sum_{e in row i} S_e L[col_e][c0 + w]  (+ X[i][c0 + w])
//   spmm_rows_kernel    R S: a CTA owns W rows [i0, i0 + W) and holds R[i0:i0+W, :] in shared
//                       memory; thread per column c (column-ELL entries):
//                       acc[w] = sum_{e in col c} R[i0 + w][row_e] S_e (+ X)
//   both then apply the GEMM epilogue (alpha acc + sum beta_t E_t + gamma I, optional second output)
//   sp_trace_kernel     a CTA owns W rows l of U and N (conj(U) rows in shared memory); thread per q:
//                       partial[l][k] = sum_q N_lq sum_{p in row q} (a_k)_qp conj(U_lp), so
//                       sum_l partial[l][k] = Tr(N a_k U^dag) = Tr(U^dag N a_k)
#pragma once
#include <cuda_runtime.h>

#include "zgemm.cuh"

namespace sqoc {

constexpr int kSpMaxW = 8;       // columns / rows per CTA (fewer when a panel would not fit)
constexpr int kSpThreads = 512;  // 16 warps: one CTA per SM (panel smem), latency hidden by warps

// Union pattern of a block's generators in two padded (ELL) layouts.  Rows (columns) are sorted by
// their entry count, longest first: entry e of the row at sorted position t sits at [e * d + t], so
// a warp's threads (consecutive t) read consecutive addresses and the 32 rows of a warp chunk have
// nearly equal counts -- a chunk loops to its own maximum r_cnt[t / 32] instead of the block's
// (d = 1179: 27.7 entries on average against 41).  Padding entries carry index 0 and value 0.
// Chunks are claimed by the warps of a CTA through a shared counter, longest first.
struct SpBlockDev {
  int d, wr, wc;          // dimension, entries per row / column (max, rounded up to a multiple of 4)
  const int* r_perm;      // [d] row at sorted position t
  const int* c_perm;      // [d] column at sorted position t
  const int* r_cnt;       // [ceil(d / 32)] entries of the longest row of each 32-chunk
  const int* c_cnt;
  const int* r_idx;       // [wr][d] column of row entry e
  const int* c_idx;       // [wc][d] row of column entry e
  const double2* r_gv;    // [(K+1)][wr][d] unscaled a_0..a_K, row layout
  const double2* c_gv;    // [(K+1)][wc][d] unscaled a_0..a_K, column layout
  double2* r_sv;          // [wr][d] the current slice's A_j, row layout
  double2* c_sv;          // [wc][d] the current slice's A_j, column layout
  // A2 = A A as a sparse x sparse product on its fixed pattern (spgemm_a2_kernel): nonzero z of A2 at
  // dense offset a2_out[z] is the sum over pairs a2_ptr[z] .. a2_ptr[z + 1] of r_sv[x] * r_sv[y]
  int a2_nnz;
  const int* a2_ptr;      // [a2_nnz + 1]
  const int* a2_out;      // [a2_nnz] row * d + column, ascending
  const int2* a2_pairs;   // offsets into r_sv of A_ij and A_jk, j ascending
};

struct SpItem {
  int blk;         // index into the SpBlockDev array
  int add_x;       // acc += X
  int diag;        // gamma I applies
  int tile_start;  // first CTA of this item in the launch
  const double2* D;  // the dense factor: L (cols kernel) or R (rows kernel)
  const double2* X;
  double2* C;
  double2* C2;
  const double2* E[4];
};

static __global__ void sp_values_kernel(int j, int K, int N, const double* __restrict__ u, double scale,
                                        const SpBlockDev* __restrict__ blocks) {
  const SpBlockDev bd = blocks[blockIdx.y];
  double uk[4];
  for (int k = 0; k < 4; ++k) uk[k] = k < K ? u[k * N + j] : 0.0;
  const int nr = bd.wr * bd.d, nc = bd.wc * bd.d;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nr + nc; t += gridDim.x * blockDim.x) {
    const bool row = t < nr;
    const int e = row ? t : t - nr;
    const int n = row ? nr : nc;
    const double2* gv = row ? bd.r_gv : bd.c_gv;
    double2 a = gv[e];
    for (int k = 0; k < K; ++k) {
      const double2 g = gv[(size_t)(k + 1) * n + e];
      a.x = fma(uk[k], g.x, a.x);
      a.y = fma(uk[k], g.y, a.y);
    }
    (row ? bd.r_sv : bd.c_sv)[e] = make_double2(a.x * scale, a.y * scale);
  }
}

__device__ __forceinline__ void cmac(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, fma(-a.y, b.y, acc.x));
  acc.y = fma(a.x, b.y, fma(a.y, b.x, acc.y));
}

// A2 = A_j A_j on the fixed pattern of the square of the union pattern (~400 of 1179 columns per row
// at cfg 3, ~730 multiply-adds per row instead of the 32,000 of S x dense): one thread per nonzero of
// A2, its contributing (A_ij, A_jk) pairs listed at setup; entries outside the pattern stay the exact
// zeros the workspace was created with (every other writer of A2 stores exact zeros there too).
static __global__ void spgemm_a2_kernel(const SpBlockDev* __restrict__ blocks, const size_t* __restrict__ off,
                                        double2* __restrict__ A2) {
  const SpBlockDev bd = blocks[blockIdx.y];
  double2* out = A2 + off[blockIdx.y];
  for (int z = blockIdx.x * blockDim.x + threadIdx.x; z < bd.a2_nnz; z += gridDim.x * blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
    const int p1 = bd.a2_ptr[z + 1];
    for (int p = bd.a2_ptr[z]; p < p1; ++p) {
      const int2 pr = bd.a2_pairs[p];
      cmac(acc, bd.r_sv[pr.x], bd.r_sv[pr.y]);
    }
    out[bd.a2_out[z]] = acc;
  }
}

// next 32-chunk of sorted rows / columns for this warp (-1: none left)
__device__ __forceinline__ int sp_claim(int* next, int nchunks, int lane) {
  int c = 0;
  if (lane == 0) c = atomicAdd(next, 1);
  c = __shfl_sync(0xffffffffu, c, 0);
  return c < nchunks ? c : -1;
}

__device__ __forceinline__ int sp_find(const SpItem* items, int nitems, int tile) {
  int lo = 0, hi = nitems - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (items[mid].tile_start <= tile) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ GemmItem sp_epi(const SpItem& it, int d) {
  GemmItem g{};
  g.C = it.C;
  g.C2 = it.C2;
  g.E0 = it.E[0];
  g.E1 = it.E[1];
  g.E2 = it.E[2];
  g.E3 = it.E[3];
  g.ldc = d;
  g.diag = it.diag;
  return g;
}

// Thread mapping: one thread per sparse row (cols kernel, trace) or column (rows kernel), so an entry's
// index and value are loaded once and used for W complex multiply-adds.  The shared-memory operand
// keeps the W values of one sparse index contiguous ([index][W], 128 bytes at W = 8) and thread t
// visits them rotated by t: at step w it handles slot (w + t) % W, so the 8 lanes of an LDS.128 phase
// read 8 different 16-byte bank groups (conflict-free for any indices); accumulator w belongs to
// output column / row (w + t) % W, a static register index.

// C[:, c0:c0+W] = S L[:, c0:c0+W] (+ X), epilogue.  Dynamic smem: d x W double2 (the L panel).
// WT > 0: the panel width as a compile-time constant (the usual 8: no width guards, shifts for the
// panel index arithmetic); WT = 0: the run-time width Wrt (panels narrowed to fit shared memory).
template <int WT>
static __global__ void __launch_bounds__(kSpThreads) spmm_cols_kernel(const SpItem* __restrict__ items, int nitems,
                                                               const SpBlockDev* __restrict__ blocks, int Wrt,
                                                               GemmArgs args) {
  const int W = WT ? WT : Wrt;
  extern __shared__ double2 panel[];  // [d][W]
  __shared__ int next;
  const int idx = sp_find(items, nitems, blockIdx.x);
  const SpItem& it = items[idx];
  const SpBlockDev& bd = blocks[it.blk];
  const int d = bd.d;
  const int c0 = (blockIdx.x - it.tile_start) * W;
  const int w_here = min(W, d - c0);
  if (threadIdx.x == 0) next = 0;
  for (int t0 = threadIdx.x; t0 < d * W; t0 += 4 * blockDim.x) {  // 4 independent loads in flight per thread
    double2 v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int t = t0 + q * blockDim.x;
      const int r = t / W, w = t - r * W;
      v[q] = (t < d * W && w < w_here) ? it.D[(size_t)r * d + c0 + w] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int t = t0 + q * blockDim.x;
      if (t < d * W) panel[t] = v[q];
    }
  }
  __syncthreads();
  const GemmItem g = sp_epi(it, d);
  const double2* addX = it.add_x ? it.X : nullptr;  // in a register: the stores below may alias the item
  const int lane = threadIdx.x & 31;
  int sl[kSpMaxW];  // rotated slot of step w
#pragma unroll
  for (int w = 0; w < kSpMaxW; ++w) sl[w] = (w + lane) % W;
  const int nchunks = (d + 31) >> 5;
  for (int ch = sp_claim(&next, nchunks, lane); ch >= 0; ch = sp_claim(&next, nchunks, lane)) {
    const int t = min(ch * 32 + lane, d - 1);  // the last chunk's spare lanes repeat row d - 1 (not stored)
    const bool live = ch * 32 + lane < d;
    const int i = bd.r_perm[t];
    const int cnt = bd.r_cnt[ch];
    double2 acc[kSpMaxW];
#pragma unroll
    for (int w = 0; w < kSpMaxW; ++w) acc[w] = make_double2(0.0, 0.0);
    // groups of 4 entries, the next group's values and indices loaded (L2) while this one multiplies;
    // the ELL height is padded to a multiple of 4 with zero entries, so a group never reads past it
    const double2* sv = bd.r_sv + t;
    const int* si = bd.r_idx + t;
    double2 cs[4];
    int ci[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      cs[q] = sv[(size_t)q * d];
      ci[q] = si[(size_t)q * d];
    }
    for (int e = 0; e < cnt; e += 4) {
      double2 ns[4];
      int ni[4];
      const bool more = e + 4 < cnt;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        ns[q] = more ? sv[(size_t)(e + 4 + q) * d] : make_double2(0.0, 0.0);
        ni[q] = more ? si[(size_t)(e + 4 + q) * d] : 0;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double2* pr = panel + ci[q] * W;
#pragma unroll
        for (int w = 0; w < kSpMaxW; ++w)
          if (w < W) cmac(acc[w], cs[q], pr[sl[w]]);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        cs[q] = ns[q];
        ci[q] = ni[q];
      }
    }
    if (!live) continue;
#pragma unroll
    for (int w = 0; w < kSpMaxW; ++w) {
      if (w >= W) break;
      const int cw = sl[w];
      if (cw >= w_here) continue;
      if (addX) {
        const double2 x = addX[(size_t)i * d + c0 + cw];
        acc[w].x += x.x;
        acc[w].y += x.y;
      }
      epi_store(g, args, i, c0 + cw, acc[w].x, acc[w].y);
    }
  }
}

// C[i0:i0+W, :] = R[i0:i0+W, :] S (+ X), epilogue.  Dynamic smem: d x W double2 (R rows, transposed).
template <int WT>
static __global__ void __launch_bounds__(kSpThreads) spmm_rows_kernel(const SpItem* __restrict__ items, int nitems,
                                                               const SpBlockDev* __restrict__ blocks, int Wrt,
                                                               GemmArgs args) {
  const int W = WT ? WT : Wrt;
  extern __shared__ double2 rowsT[];  // [d][W]: rowsT[r][w] = R[i0 + w][r]
  __shared__ int next;
  const int idx = sp_find(items, nitems, blockIdx.x);
  const SpItem& it = items[idx];
  const SpBlockDev& bd = blocks[it.blk];
  const int d = bd.d;
  const int i0 = (blockIdx.x - it.tile_start) * W;
  const int w_here = min(W, d - i0);
  if (threadIdx.x == 0) next = 0;
  for (int t0 = threadIdx.x; t0 < d * W; t0 += 4 * blockDim.x) {  // 4 independent loads in flight per thread
    double2 v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int t = t0 + q * blockDim.x;
      const int w = t / d, r = t - w * d;  // coalesced global reads along r
      v[q] = (t < d * W && w < w_here) ? it.D[(size_t)(i0 + w) * d + r] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int t = t0 + q * blockDim.x;
      const int w = t / d, r = t - w * d;
      if (t < d * W) rowsT[r * W + w] = v[q];
    }
  }
  __syncthreads();
  const GemmItem g = sp_epi(it, d);
  const double2* addX = it.add_x ? it.X : nullptr;  // in a register: the stores below may alias the item
  const int lane = threadIdx.x & 31;
  int sl[kSpMaxW];
#pragma unroll
  for (int w = 0; w < kSpMaxW; ++w) sl[w] = (w + lane) % W;
  const int nchunks = (d + 31) >> 5;
  for (int ch = sp_claim(&next, nchunks, lane); ch >= 0; ch = sp_claim(&next, nchunks, lane)) {
    const int t = min(ch * 32 + lane, d - 1);
    const bool live = ch * 32 + lane < d;
    const int c = bd.c_perm[t];
    const int cnt = bd.c_cnt[ch];
    double2 acc[kSpMaxW];
#pragma unroll
    for (int w = 0; w < kSpMaxW; ++w) acc[w] = make_double2(0.0, 0.0);
    const double2* sv = bd.c_sv + t;  // entry groups of 4 with the next group prefetched (see the cols kernel)
    const int* si = bd.c_idx + t;
    double2 cs[4];
    int ci[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      cs[q] = sv[(size_t)q * d];
      ci[q] = si[(size_t)q * d];
    }
    for (int e = 0; e < cnt; e += 4) {
      double2 ns[4];
      int ni[4];
      const bool more = e + 4 < cnt;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        ns[q] = more ? sv[(size_t)(e + 4 + q) * d] : make_double2(0.0, 0.0);
        ni[q] = more ? si[(size_t)(e + 4 + q) * d] : 0;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double2* rr = rowsT + ci[q] * W;
#pragma unroll
        for (int w = 0; w < kSpMaxW; ++w)
          if (w < W) cmac(acc[w], rr[sl[w]], cs[q]);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        cs[q] = ns[q];
        ci[q] = ni[q];
      }
    }
    if (!live) continue;
#pragma unroll
    for (int w = 0; w < kSpMaxW; ++w) {
      if (w >= W) break;
      const int rw = sl[w];
      if (rw >= w_here) continue;
      if (addX) {
        const double2 x = addX[(size_t)(i0 + rw) * d + c];
        acc[w].x += x.x;
        acc[w].y += x.y;
      }
      epi_store(g, args, i0 + rw, c, acc[w].x, acc[w].y);
    }
  }
}

// partial[l][k] for l in [l0, l0 + W): sum_q N[l][q] sum_{e in row q} (a_{k+1})_e conj(U[l][col_e]).
// With the dense path's convention (the trace epilogue of U^dag N against a_{k+1}) the per-block sum
// over l is Tr(U^dag N a_{k+1}).
struct SpTraceItem {
  int blk;
  int tile_start;
  const double2* U;
  const double2* N;
  double2* part;  // [d][K] of this block
};

template <int WT>
static __global__ void __launch_bounds__(kSpThreads) sp_trace_kernel(const SpTraceItem* __restrict__ items, int nitems,
                                                              const SpBlockDev* __restrict__ blocks, int K, int Wrt) {
  const int W = WT ? WT : Wrt;
  extern __shared__ double2 uT[];  // [d][W]: uT[p][w] = conj(U[l0 + w][p])
  __shared__ double2 red[kSpMaxW][kSpThreads / 32];
  int lo = 0, hi = nitems - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (items[mid].tile_start <= (int)blockIdx.x) lo = mid;
    else hi = mid - 1;
  }
  const SpTraceItem& it = items[lo];
  const SpBlockDev& bd = blocks[it.blk];
  const int d = bd.d;
  const int l0 = (blockIdx.x - it.tile_start) * W;
  const int w_here = min(W, d - l0);
  for (int t0 = threadIdx.x; t0 < d * W; t0 += 4 * blockDim.x) {  // 4 independent loads in flight per thread
    double2 v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int t = t0 + q * blockDim.x;
      const int w = t / d, p = t - w * d;
      v[q] = (t < d * W && w < w_here) ? it.U[(size_t)(l0 + w) * d + p] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int t = t0 + q * blockDim.x;
      const int w = t / d, p = t - w * d;
      if (t < d * W) uT[p * W + w] = make_double2(v[q].x, -v[q].y);
    }
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int sl[kSpMaxW];
#pragma unroll
  for (int w = 0; w < kSpMaxW; ++w) sl[w] = (w + lane) % W;
  const size_t nr = (size_t)bd.wr * d;
  const int nchunks = (d + 31) >> 5;
  for (int k = 0; k < K; ++k) {
    const double2* gv = bd.r_gv + (size_t)(k + 1) * nr;
    double2 acc[kSpMaxW];
#pragma unroll
    for (int w = 0; w < kSpMaxW; ++w) acc[w] = make_double2(0.0, 0.0);
    // static chunk -> warp map: the reduction order below must not depend on which warp claimed what,
    // so that repeated evaluations are bit-identical
    const int nw = (int)(blockDim.x >> 5);
    for (int ps = 0; ps * nw < nchunks; ++ps) {  // serpentine over the count-sorted chunks: balanced warps
      const int ch = ps * nw + ((ps & 1) ? nw - 1 - warp : warp);
      if (ch >= nchunks) continue;
      const int tq = min(ch * 32 + lane, d - 1);
      const bool live = ch * 32 + lane < d;
      const int q = bd.r_perm[tq];
      const int cnt = bd.r_cnt[ch];
      double2 t[kSpMaxW];
#pragma unroll
      for (int w = 0; w < kSpMaxW; ++w) t[w] = make_double2(0.0, 0.0);
#pragma unroll 4
      for (int e = 0; e < cnt; ++e) {
        const double2 a = gv[(size_t)e * d + tq];
        const double2* ur = uT + bd.r_idx[(size_t)e * d + tq] * W;
#pragma unroll
        for (int w = 0; w < kSpMaxW; ++w)
          if (w < W) cmac(t[w], a, ur[sl[w]]);
      }
      if (!live) continue;
#pragma unroll
      for (int w = 0; w < kSpMaxW; ++w) {
        if (w >= W) break;
        const int lw = sl[w];
        if (lw < w_here) cmac(acc[w], it.N[(size_t)(l0 + lw) * d + q], t[w]);
      }
    }
    // rows of this thread's accumulators are rotated: route acc[w] to row (w + rot) % W, then a
    // fixed-order reduction per row (warp shuffles, then warps in order): deterministic
#pragma unroll
    for (int r = 0; r < kSpMaxW; ++r) {
      if (r >= W) break;
      double sx = 0.0, sy = 0.0;
#pragma unroll
      for (int w = 0; w < kSpMaxW; ++w)
        if (w < W && sl[w] == r) {
          sx = acc[w].x;
          sy = acc[w].y;
        }
      for (int o = 16; o > 0; o >>= 1) {
        sx += __shfl_xor_sync(0xffffffffu, sx, o);
        sy += __shfl_xor_sync(0xffffffffu, sy, o);
      }
      if (lane == 0) red[r][warp] = make_double2(sx, sy);
    }
    __syncthreads();
    if (threadIdx.x < w_here) {
      double2 s = make_double2(0.0, 0.0);
      for (int v = 0; v < (int)(blockDim.x >> 5); ++v) {
        s.x += red[threadIdx.x][v].x;
        s.y += red[threadIdx.x][v].y;
      }
      it.part[(size_t)(l0 + threadIdx.x) * K + k] = s;
    }
    __syncthreads();
  }
}

}  // namespace sqoc
