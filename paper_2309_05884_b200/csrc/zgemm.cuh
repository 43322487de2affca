// Batched complex FP64 GEMM on the sm_100a FP64 tensor path (mma.sync m8n8k4 -> DMMA.8x8x4).
//
// tcgen05/UMMA has no FP64 kind, so the FP64 tensor cores are reached through
// warp-level mma.sync; on B200 DMMA runs at 64 FMA/clk/SM (36.9 TFLOP/s measured,
// profiles/r01_fp64_peak.txt).  Complex products use 4 real DMMAs (re*re - im*im,
// re*im + im*re) on interleaved (re, im) tiles: one LDS.128 gives both parts of
// a fragment element.
//
// Work list: an array of GemmItem (one independent GEMM each, possibly with two
// K segments C = A0 B0 + A1 B1), tiles mapped by a prefix sum so blocks of
// different sizes share one launch.  Operands may be conjugate-transposed.
// Epilogues: C = alpha acc + beta0 E0 + beta1 E1 + gamma [diag] I, or a fused
// trace sum_pq acc[p][q] F_k[q][p] written as per-tile partials (no C store); EPI_MIXED
// lets one launch hold both kinds of items (trace iff the item has nF > 0).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace sqoc {

enum { OP_N = 0, OP_C = 1 };
enum { EPI_STORE = 0, EPI_TRACE = 1, EPI_MIXED = 2 };  // MIXED: per item, trace iff it.nF > 0

struct GemmItem {
  const double2* A0;
  const double2* B0;
  const double2* A1;
  const double2* B1;
  double2* C;
  const double2* E0;
  const double2* E1;
  const double2* E2;
  const double2* E3;
  double2* C2;        // optional second output (same product, its own linear combination)
  const double2* F;   // trace epilogue: nF matrices, F + f * fstride
  double2* tr_out;    // trace epilogue: [tiles][nF] partials
  long fstride;
  int m, n, k, nseg;
  int lda, ldb, ldc;
  int diag;           // gamma applies to this item
  int tile_start, tiles_n;
  int nF;
  int herm;           // the product is Hermitian (X X with X = -X^dag): the persistent kernel computes the tiles on
                      // and above the diagonal and stores the conjugate mirror of the ones above it
};

// C  = alpha  acc + sum_t beta_t  E_t + gamma  [diag] I
// C2 = alpha2 acc + sum_t beta2_t E_t + gamma2 [diag] I   (when it.C2)
struct GemmArgs {
  double alpha, beta0, beta1, gamma;
  double beta2, beta3;
  double alpha2, beta2_0, beta2_1, beta2_2, beta2_3, gamma2;
};

__device__ __forceinline__ void epi_store(const GemmItem& it, const GemmArgs& a, int m, int n, double re, double im) {
  const size_t off = (size_t)m * it.ldc + n;
  const double2* E[4] = {it.E0, it.E1, it.E2, it.E3};
  const double b1[4] = {a.beta0, a.beta1, a.beta2, a.beta3};
  const double b2[4] = {a.beta2_0, a.beta2_1, a.beta2_2, a.beta2_3};
  double2 c = make_double2(a.alpha * re, a.alpha * im);
  double2 c2 = make_double2(a.alpha2 * re, a.alpha2 * im);
#pragma unroll
  for (int t = 0; t < 4; ++t)
    if (E[t]) {
      const double2 e = E[t][off];
      c.x += b1[t] * e.x;
      c.y += b1[t] * e.y;
      c2.x += b2[t] * e.x;
      c2.y += b2[t] * e.y;
    }
  if (it.diag && m == n) {
    c.x += a.gamma;
    c2.x += a.gamma2;
  }
  it.C[off] = c;
  if (it.C2) it.C2[off] = c2;
}

// K depth per pipeline stage and stage count (build-time knobs; r01 cfg 2: GBK 8 x 4 stages 39.4 ms,
// 16 x 3 stages (1 CTA / SM) 55.6 ms, 16 x 2 stages 39.5 ms)
#ifndef SQOC_GBK
#define SQOC_GBK 8
#endif
#ifndef SQOC_GSTAGES
#define SQOC_GSTAGES 4
#endif
constexpr int GBM = 64, GBN = 64, GBK = SQOC_GBK, GSTAGES = SQOC_GSTAGES, GTHREADS = 128;
constexpr int LD_KMAJ = GBK + 4;  // tiles stored [row][k]: ld = 12 (== 4 mod 8, conflict-free)
constexpr int LD_NMAJ = GBM + 2;  // tiles stored [k][col]: ld = 66 (== 2 mod 8, conflict-free)
constexpr int G_A_ELEMS = (GBM * LD_KMAJ > GBK * LD_NMAJ) ? GBM * LD_KMAJ : GBK * LD_NMAJ;  // 768 vs 528
constexpr size_t G_SMEM = sizeof(double2) * GSTAGES * 2 * G_A_ELEMS;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int n = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

#ifndef SQOC_DMMA_NV
#define SQOC_DMMA_NV 0
#endif
#if SQOC_DMMA_NV
#define SQOC_DMMA_ASM asm
#else
#define SQOC_DMMA_ASM asm volatile
#endif
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  SQOC_DMMA_ASM("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Load one K-step (GBK) of op(A) (rows m0.., k0..) and op(B) (k0.., cols n0..) into a stage.
template <int TA, int TB, int NT = GTHREADS>
__device__ __forceinline__ void gemm_load_stage(double2* sA, double2* sB, const double2* A, const double2* B,
                                                const GemmItem& it, int m0, int n0, int k0) {
  const int tid = threadIdx.x;
#pragma unroll
  for (int r = 0; r < (GBM * GBK) / NT; ++r) {
    const int i = tid + r * NT;
    if (TA == OP_N) {  // A[m][k] row-major; smem [m][k]
      const int row = i / GBK, col = i % GBK;
      const int gm = m0 + row, gk = k0 + col;
      const bool ok = gm < it.m && gk < it.k;
      cp_async16(sA + row * LD_KMAJ + col, ok ? A + (size_t)gm * it.lda + gk : A, ok);
    } else {  // op(A)[m][k] = conj(A[k][m]); smem [k][m]
      const int row = i / GBM, col = i % GBM;
      const int gk = k0 + row, gm = m0 + col;
      const bool ok = gm < it.m && gk < it.k;
      cp_async16(sA + row * LD_NMAJ + col, ok ? A + (size_t)gk * it.lda + gm : A, ok);
    }
    if (TB == OP_N) {  // B[k][n]; smem [k][n]
      const int row = i / GBN, col = i % GBN;
      const int gk = k0 + row, gn = n0 + col;
      const bool ok = gn < it.n && gk < it.k;
      cp_async16(sB + row * LD_NMAJ + col, ok ? B + (size_t)gk * it.ldb + gn : B, ok);
    } else {  // op(B)[k][n] = conj(B[n][k]); smem [n][k]
      const int row = i / GBK, col = i % GBK;
      const int gn = n0 + row, gk = k0 + col;
      const bool ok = gn < it.n && gk < it.k;
      cp_async16(sB + row * LD_KMAJ + col, ok ? B + (size_t)gn * it.ldb + gk : B, ok);
    }
  }
}

template <int TA, int TB, int EPI>
__global__ void __launch_bounds__(GTHREADS) zgemm_kernel(const GemmItem* __restrict__ items, int nitems,
                                                         GemmArgs args) {
  extern __shared__ double2 gsm[];
  // ---- locate the item owning this tile (items sorted by tile_start) ----
  int lo = 0, hi = nitems - 1;
  const int tile = blockIdx.x;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (items[mid].tile_start <= tile) lo = mid;
    else hi = mid - 1;
  }
  const GemmItem it = items[lo];
  const int local = tile - it.tile_start;
  const int m0 = (local / it.tiles_n) * GBM;
  const int n0 = (local % it.tiles_n) * GBN;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  const int lr = lane >> 2, lc = lane & 3;

  double acc[4][4][4];  // [mi][ni][re0, re1, im0, im1]
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[a][b][c] = 0.0;

  const int kt_per_seg = (it.k + GBK - 1) / GBK;
  const int kt_total = kt_per_seg * it.nseg;
  double2* sAbase = gsm;
  double2* sBbase = gsm + GSTAGES * G_A_ELEMS;

  auto issue = [&](int kt) {
    if (kt < kt_total) {
      const int seg = kt / kt_per_seg;
      const int k0 = (kt - seg * kt_per_seg) * GBK;
      const int st = kt % GSTAGES;
      gemm_load_stage<TA, TB>(sAbase + st * G_A_ELEMS, sBbase + st * G_A_ELEMS, seg ? it.A1 : it.A0,
                              seg ? it.B1 : it.B0, it, m0, n0, k0);
    }
    cp_async_commit();
  };

#pragma unroll
  for (int s = 0; s < GSTAGES - 1; ++s) issue(s);

  for (int kt = 0; kt < kt_total; ++kt) {
    cp_async_wait<GSTAGES - 2>();
    __syncthreads();
    issue(kt + GSTAGES - 1);
    const int st = kt % GSTAGES;
    const double2* sA = sAbase + st * G_A_ELEMS;
    const double2* sB = sBbase + st * G_A_ELEMS;
#pragma unroll
    for (int kk = 0; kk < GBK; kk += 4) {
      double ar[4], ai[4], nai[4], br[4], bi[4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) {
        const int m = wm + mi * 8 + lr, k = kk + lc;
        double2 a;
        if (TA == OP_N) a = sA[m * LD_KMAJ + k];
        else { a = sA[k * LD_NMAJ + m]; a.y = -a.y; }
        ar[mi] = a.x; ai[mi] = a.y; nai[mi] = -a.y;
      }
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        const int n = wn + ni * 8 + lr, k = kk + lc;
        double2 b;
        if (TB == OP_N) b = sB[k * LD_NMAJ + n];
        else { b = sB[n * LD_KMAJ + k]; b.y = -b.y; }
        br[ni] = b.x; bi[ni] = b.y;
      }
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) {
          dmma(acc[mi][ni][0], acc[mi][ni][1], ar[mi], br[ni]);
          dmma(acc[mi][ni][0], acc[mi][ni][1], nai[mi], bi[ni]);
          dmma(acc[mi][ni][2], acc[mi][ni][3], ar[mi], bi[ni]);
          dmma(acc[mi][ni][2], acc[mi][ni][3], ai[mi], br[ni]);
        }
    }
  }
  cp_async_wait<0>();

  const bool trace = EPI == EPI_TRACE || (EPI == EPI_MIXED && it.nF > 0);  // uniform per CTA
  if (!trace) {
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int m = m0 + wm + mi * 8 + lr;
          const int n = n0 + wn + ni * 8 + 2 * lc + v;
          if (m < it.m && n < it.n) epi_store(it, args, m, n, acc[mi][ni][v], acc[mi][ni][2 + v]);
        }
  } else {
    // fused trace: partial_f = sum_{p,q in tile} alpha acc[p][q] F_f[q][p]
    __shared__ double2 red[GTHREADS / 32][4];
    for (int f = 0; f < it.nF; ++f) {
      const double2* F = it.F + f * it.fstride;
      double sx = 0.0, sy = 0.0;
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            const int p = m0 + wm + mi * 8 + lr;
            const int q = n0 + wn + ni * 8 + 2 * lc + v;
            if (p < it.m && q < it.n) {
              const double2 e = F[(size_t)q * it.ldc + p];
              const double cr = args.alpha * acc[mi][ni][v], ci = args.alpha * acc[mi][ni][2 + v];
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
    __syncthreads();
    if (threadIdx.x < it.nF) {
      double2 s = make_double2(0.0, 0.0);
      for (int w = 0; w < GTHREADS / 32; ++w) { s.x += red[w][threadIdx.x].x; s.y += red[w][threadIdx.x].y; }
      it.tr_out[(size_t)local * it.nF + threadIdx.x] = s;
    }
  }
}

// ---------------------------------------------------------------------------
// 3M (Gauss) variant: T1 = Ar Br, T2 = Ai Bi, T3 = (Ar + Ai)(Br + Bi);
// C = (T1 - T2) + i (T3 - T1 - T2).  Three DMMAs per complex k-step instead of four
// (the complex FLOP count of the algorithm stays 8 d^3 by convention; the FP64 pipe
// executes 6 d^3).  8 warps per CTA (2 x 4), warp tile 32 x 16 (4 x 2 DMMA tiles),
// so the three accumulator sets fit in registers.
constexpr int G3THREADS = 256;

// Main loop of one CTA tile for a warp whose valid output is MC x NC DMMA sub-tiles (8 x 8):
// sub-tiles wholly outside C issue neither fragment loads nor DMMAs.  The shape is a template
// parameter (dispatched once per warp) because a predicated-off DMMA still occupies the pipe;
// every instantiation runs the same cp.async / barrier sequence, so warps of one CTA may take
// different instantiations.  The all-zero k = 4 half-step of a segment's last K tile is skipped.
template <int TA, int TB, int MC, int NC>
__device__ __forceinline__ void g3_mainloop(double (&acc)[4][2][3][2], const GemmItem& it, double2* sAbase,
                                            double2* sBbase, int m0, int n0, int wm, int wn, int lr, int lc) {
  const int kt_per_seg = (it.k + GBK - 1) / GBK;
  const int kt_total = kt_per_seg * it.nseg;
  auto issue = [&](int kt) {
    if (kt < kt_total) {
      const int seg = kt / kt_per_seg;
      const int k0 = (kt - seg * kt_per_seg) * GBK;
      const int st = kt % GSTAGES;
      gemm_load_stage<TA, TB, G3THREADS>(sAbase + st * G_A_ELEMS, sBbase + st * G_A_ELEMS, seg ? it.A1 : it.A0,
                                         seg ? it.B1 : it.B0, it, m0, n0, k0);
    }
    cp_async_commit();
  };
#pragma unroll
  for (int s = 0; s < GSTAGES - 1; ++s) issue(s);
  constexpr int KS = GBK / 4;                                      // k-steps per stage
  const int last_steps = (it.k % GBK) ? ((it.k % GBK) + 3) / 4 : KS;  // a segment's last K tile
  int kin = 0;
  for (int kt = 0; kt < kt_total; ++kt) {
    cp_async_wait<GSTAGES - 2>();
    __syncthreads();
    issue(kt + GSTAGES - 1);
    const int st = kt % GSTAGES;
    const double2* sA = sAbase + st * G_A_ELEMS;
    const double2* sB = sBbase + st * G_A_ELEMS;
    const int ksteps = (kin == kt_per_seg - 1) ? last_steps : KS;
    if (++kin == kt_per_seg) kin = 0;
    if constexpr (MC > 0 && NC > 0) {
    // both k-steps of a stage unrolled (loads of the second overlap the first's DMMAs); only the
    // segment's last stage may skip its all-zero second half
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      if (ks >= ksteps) break;
      const int kk = ks * 4;
      double ar[MC], ai[MC], as[MC], br[NC], bi[NC], bs[NC];
#pragma unroll
      for (int mi = 0; mi < MC; ++mi) {
        const int m = wm + mi * 8 + lr, k = kk + lc;
        double2 a;
        if (TA == OP_N) a = sA[m * LD_KMAJ + k];
        else { a = sA[k * LD_NMAJ + m]; a.y = -a.y; }
        ar[mi] = a.x; ai[mi] = a.y; as[mi] = a.x + a.y;
      }
#pragma unroll
      for (int ni = 0; ni < NC; ++ni) {
        const int n = wn + ni * 8 + lr, k = kk + lc;
        double2 b;
        if (TB == OP_N) b = sB[k * LD_NMAJ + n];
        else { b = sB[n * LD_KMAJ + k]; b.y = -b.y; }
        br[ni] = b.x; bi[ni] = b.y; bs[ni] = b.x + b.y;
      }
#pragma unroll
      for (int mi = 0; mi < MC; ++mi)
#pragma unroll
        for (int ni = 0; ni < NC; ++ni) {
          dmma(acc[mi][ni][0][0], acc[mi][ni][0][1], ar[mi], br[ni]);
          dmma(acc[mi][ni][1][0], acc[mi][ni][1][1], ai[mi], bi[ni]);
          dmma(acc[mi][ni][2][0], acc[mi][ni][2][1], as[mi], bs[ni]);
        }
    }
    }
  }
}

template <int TA, int TB, int EPI>
__global__ void __launch_bounds__(G3THREADS, 2) zgemm3m_kernel(const GemmItem* __restrict__ items, int nitems,
                                                               GemmArgs args) {
  extern __shared__ double2 gsm[];
  int lo = 0, hi = nitems - 1;
  const int tile = blockIdx.x;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (items[mid].tile_start <= tile) lo = mid;
    else hi = mid - 1;
  }
  const GemmItem it = items[lo];
  const int local = tile - it.tile_start;
  const int m0 = (local / it.tiles_n) * GBM;
  const int n0 = (local % it.tiles_n) * GBN;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = (warp >> 2) * 32, wn = (warp & 3) * 16;
  const int lr = lane >> 2, lc = lane & 3;

  double acc[4][2][3][2];  // [mi][ni][T1,T2,T3][c0,c1]
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int c = 0; c < 3; ++c) acc[a][b][c][0] = acc[a][b][c][1] = 0.0;

  double2* sAbase = gsm;
  double2* sBbase = gsm + GSTAGES * G_A_ELEMS;
  const int mc = max(0, min(4, (it.m - m0 - wm + 7) / 8));
  const int nc = max(0, min(2, (it.n - n0 - wn + 7) / 8));
  switch ((mc == 0 || nc == 0) ? -1 : (mc - 1) * 2 + (nc - 1)) {
    case 7: g3_mainloop<TA, TB, 4, 2>(acc, it, sAbase, sBbase, m0, n0, wm, wn, lr, lc); break;
    case 6: g3_mainloop<TA, TB, 4, 1>(acc, it, sAbase, sBbase, m0, n0, wm, wn, lr, lc); break;
    case 5: g3_mainloop<TA, TB, 3, 2>(acc, it, sAbase, sBbase, m0, n0, wm, wn, lr, lc); break;
    case 4: g3_mainloop<TA, TB, 3, 1>(acc, it, sAbase, sBbase, m0, n0, wm, wn, lr, lc); break;
    case 3: g3_mainloop<TA, TB, 2, 2>(acc, it, sAbase, sBbase, m0, n0, wm, wn, lr, lc); break;
    case 2: g3_mainloop<TA, TB, 2, 1>(acc, it, sAbase, sBbase, m0, n0, wm, wn, lr, lc); break;
    case 1: g3_mainloop<TA, TB, 1, 2>(acc, it, sAbase, sBbase, m0, n0, wm, wn, lr, lc); break;
    case 0: g3_mainloop<TA, TB, 1, 1>(acc, it, sAbase, sBbase, m0, n0, wm, wn, lr, lc); break;
    default: g3_mainloop<TA, TB, 0, 0>(acc, it, sAbase, sBbase, m0, n0, wm, wn, lr, lc); break;
  }
  cp_async_wait<0>();

  const bool trace = EPI == EPI_TRACE || (EPI == EPI_MIXED && it.nF > 0);  // uniform per CTA
  if (!trace) {
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 2; ++ni)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int m = m0 + wm + mi * 8 + lr;
          const int n = n0 + wn + ni * 8 + 2 * lc + v;
          if (m < it.m && n < it.n) {
            const double t1 = acc[mi][ni][0][v], t2 = acc[mi][ni][1][v], t3 = acc[mi][ni][2][v];
            epi_store(it, args, m, n, t1 - t2, t3 - t1 - t2);
          }
        }
  } else {
    __shared__ double2 red[G3THREADS / 32][4];
    for (int f = 0; f < it.nF; ++f) {
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
            if (p < it.m && q < it.n) {
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
    __syncthreads();
    if (threadIdx.x < it.nF) {
      double2 s = make_double2(0.0, 0.0);
      for (int w = 0; w < G3THREADS / 32; ++w) { s.x += red[w][threadIdx.x].x; s.y += red[w][threadIdx.x].y; }
      it.tr_out[(size_t)local * it.nF + threadIdx.x] = s;
    }
  }
}

}  // namespace sqoc
