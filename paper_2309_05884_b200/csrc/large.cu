// Large-block GRAPE path: host orchestration + elementwise / reduction kernels.
// See large.cuh for the per-slice algebra and zgemm.cuh for the DMMA GEMM.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>

#include "../../include/symqoc_b200.h"
#include "large.cuh"

namespace sqoc {

static double inv_fact(int k) {
  double f = 1.0;
  for (int i = 2; i <= k; ++i) f *= i;
  return 1.0 / f;
}

// Same plan rule as the tiny kernel's choose_taylor (tiny.cuh).
static void choose_taylor_host(double nrm, int& nb, int& s) {
  const double theta[4] = {0.33, 0.67, 1.10, 1.65};
  int best = 1 << 30;
  nb = 4;
  s = 0;
  for (int i = 0; i < 4; ++i) {
    int si = 0;
    double x = nrm;
    while (x > theta[i] && si < 60) { x *= 0.5; ++si; }
    const int cost = (4 + i) + 1 + si;
    if (cost < best || (cost == best && si < s)) { best = cost; nb = 4 + i; s = si; }
  }
}

// ------------------------------------------------------------------ kernels
__global__ void bound_kernel(const double* __restrict__ u, int K, int N, int nblk, const double* __restrict__ gnorm,
                             unsigned long long* out) {
  double best = 0.0;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < N; j += gridDim.x * blockDim.x) {
    for (int b = 0; b < nblk; ++b) {
      double v = gnorm[b * (K + 1)];
      for (int k = 0; k < K; ++k) v += fabs(u[k * N + j]) * gnorm[b * (K + 1) + k + 1];
      best = fmax(best, v);
    }
  }
  for (int o = 16; o > 0; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(best));
}

__global__ void build_a_kernel(int j, int K, int N, const double* __restrict__ u, const int* __restrict__ dims,
                               const size_t* __restrict__ off, const double2* const* __restrict__ gen, double scale,
                               double2* __restrict__ A) {
  const int b = blockIdx.y;
  const int d = dims[b];
  const size_t dd = (size_t)d * d;
  const double2* g = gen[b];
  double uk[4];
  for (int k = 0; k < 4; ++k) uk[k] = k < K ? u[k * N + j] : 0.0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < dd; i += (size_t)gridDim.x * blockDim.x) {
    double2 a = g[i];
    for (int k = 0; k < K; ++k) {
      const double2 e = g[(k + 1) * dd + i];
      a.x = fma(uk[k], e.x, a.x);
      a.y = fma(uk[k], e.y, a.y);
    }
    A[off[b] + i] = make_double2(a.x * scale, a.y * scale);
  }
}

// T = cm A3 + c0 I + c1 A + c2 A2 ;  dT = cm dA3 + c1 Ad + c2 dA2 (when pair)
__global__ void horner_init_kernel(int pair, const int* __restrict__ dims, const size_t* __restrict__ off, double cm,
                                   double c0, double c1, double c2, const double2* __restrict__ A,
                                   const double2* __restrict__ A2, const double2* __restrict__ A3,
                                   const double2* __restrict__ Ad, const double2* __restrict__ dA2,
                                   const double2* __restrict__ dA3, double2* __restrict__ T, double2* __restrict__ dT) {
  const int b = blockIdx.y;
  const int d = dims[b];
  const size_t dd = (size_t)d * d;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < dd; i += (size_t)gridDim.x * blockDim.x) {
    const size_t o = off[b] + i;
    double2 t = make_double2(cm * A3[o].x + c1 * A[o].x + c2 * A2[o].x, cm * A3[o].y + c1 * A[o].y + c2 * A2[o].y);
    if (i / d == i % d) t.x += c0;
    T[o] = t;
    if (pair)
      dT[o] = make_double2(cm * dA3[o].x + c1 * Ad[o].x + c2 * dA2[o].x, cm * dA3[o].y + c1 * Ad[o].y + c2 * dA2[o].y);
  }
}

// X = I (gate) or psi_0 (state);  L = V or psi_f
__global__ void init_xl_kernel(int gate, int R, const int* __restrict__ dims, const size_t* __restrict__ offr,
                               const double2* const* __restrict__ x0, const double2* const* __restrict__ tgt,
                               double2* __restrict__ X, double2* __restrict__ L) {
  const int b = blockIdx.y;
  const int d = dims[b];
  const int r = gate ? d : R;
  const size_t n = (size_t)d * r;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const size_t o = offr[b] + i;
    if (gate) X[o] = make_double2((i / r == i % r) ? 1.0 : 0.0, 0.0);
    else X[o] = x0[b][i];
    L[o] = tgt[b][i];
  }
}

// tau_b = sum conj(V) * X over the block (one CTA per block, fixed tree)
__global__ void tau_kernel(int gate, int R, const int* __restrict__ dims, const size_t* __restrict__ offr,
                           const double2* __restrict__ X, const double2* const* __restrict__ tgt,
                           double2* __restrict__ tau_local, double2* __restrict__ tau_out, const int* __restrict__ gidx) {
  __shared__ double2 red[256];
  const int b = blockIdx.x;
  const int d = dims[b];
  const size_t n = (size_t)d * (gate ? d : R);
  double sx = 0.0, sy = 0.0;
  for (size_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double2 v = tgt[b][i], x = X[offr[b] + i];
    sx += v.x * x.x + v.y * x.y;
    sy += v.x * x.y - v.y * x.x;
  }
  red[threadIdx.x] = make_double2(sx, sy);
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      red[threadIdx.x].x += red[threadIdx.x + s].x;
      red[threadIdx.x].y += red[threadIdx.x + s].y;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    tau_local[b] = red[0];
    tau_out[gidx[b]] = red[0];
  }
}

// grad_bkj = 2 w_b Re(conj(tau_b) sum_tiles partial)   (one CTA per block, fixed order)
__global__ void trace_reduce_kernel(int j, int K, int N, const int* __restrict__ tile_off, const double2* __restrict__ part,
                                    const double2* __restrict__ tau, const double* __restrict__ w,
                                    const int* __restrict__ gidx, double* __restrict__ gradb, size_t block_stride) {
  __shared__ double2 red[256];
  const int b = blockIdx.x;
  const int t0 = tile_off[b], t1 = tile_off[b + 1];
  for (int k = 0; k < K; ++k) {
    double sx = 0.0, sy = 0.0;
    for (int t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
      sx += part[(size_t)t * K + k].x;
      sy += part[(size_t)t * K + k].y;
    }
    red[threadIdx.x] = make_double2(sx, sy);
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
      if (threadIdx.x < s) {
        red[threadIdx.x].x += red[threadIdx.x + s].x;
        red[threadIdx.x].y += red[threadIdx.x + s].y;
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      const double2 g = red[0], t = tau[b];
      gradb[gidx[b] * block_stride + (size_t)k * N + j] = 2.0 * w[b] * (t.x * g.x + t.y * g.y);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ host side
template <int TA, int TB, int EPI>
static cudaError_t launch_gemm(const GemmItem* items, int n, int tiles, GemmArgs a, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(zgemm_kernel<TA, TB, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)G_SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  zgemm_kernel<TA, TB, EPI><<<tiles, GTHREADS, G_SMEM, st>>>(items, n, a);
  return cudaGetLastError();
}

enum Op { F_A2, F_A3, F_H, F_S, F_X, B_C, B_P2, B_P3, B_H, B_S, B_D, B_XL };

static int tiles_of(int m, int n) { return ((m + GBM - 1) / GBM) * ((n + GBN - 1) / GBN); }

static GemmItem mk(const double2* A0, const double2* B0, const double2* A1, const double2* B1, double2* C,
                   const double2* E0, const double2* E1, int m, int n, int k, int nseg, int lda, int ldb, int ldc,
                   int diag) {
  GemmItem it{};
  it.A0 = A0; it.B0 = B0; it.A1 = A1; it.B1 = B1; it.C = C; it.E0 = E0; it.E1 = E1;
  it.m = m; it.n = n; it.k = k; it.nseg = nseg; it.lda = lda; it.ldb = ldb; it.ldc = ldc; it.diag = diag;
  it.tiles_n = (n + GBN - 1) / GBN;
  return it;
}

static std::pair<GemmItem*, int> get_list(LargeGroup& g, int op, int p, int q, int r, int* tiles_out) {
  auto key = std::make_tuple(op, p, q, r);
  auto found = g.lists.find(key);
  std::vector<GemmItem> v;
  if (found == g.lists.end()) {
    for (int b = 0; b < g.nblk; ++b) {
      const int d = g.blocks[b].d, R = g.gate ? d : 1;
      const size_t o = g.off[b], orr = g.offr[b];
      double2 *A = g.A + o, *Ad = g.Ad + o, *A2 = g.A2 + o, *dA2 = g.dA2 + o, *A3 = g.A3 + o, *dA3 = g.dA3 + o;
      double2 *Tp = g.T[p] + o, *Tn = g.T[1 - p] + o, *dTp = g.dT[p] + o, *dTn = g.dT[1 - p] + o;
      double2 *Xq = g.X[q] + orr, *Xn = g.X[1 - q] + orr, *Lr = g.L[r] + orr, *Ln = g.L[1 - r] + orr;
      switch (op) {
        case F_A2: v.push_back(mk(A, A, 0, 0, A2, 0, 0, d, d, d, 1, d, d, d, 0)); break;
        case F_A3: v.push_back(mk(A2, A, 0, 0, A3, 0, 0, d, d, d, 1, d, d, d, 0)); break;
        case F_H: v.push_back(mk(Tp, A3, 0, 0, Tn, A, A2, d, d, d, 1, d, d, d, 1)); break;
        case F_S: v.push_back(mk(Tp, Tp, 0, 0, Tn, 0, 0, d, d, d, 1, d, d, d, 0)); break;
        case F_X: v.push_back(mk(Tp, Xq, 0, 0, Xn, 0, 0, d, R, d, 1, d, R, R, 0)); break;
        case B_C: v.push_back(mk(Xq, Lr, 0, 0, Ad, 0, 0, d, d, R, 1, R, R, d, 0)); break;
        case B_P2:
          v.push_back(mk(A, A, 0, 0, A2, 0, 0, d, d, d, 1, d, d, d, 0));
          v.push_back(mk(A, Ad, Ad, A, dA2, 0, 0, d, d, d, 2, d, d, d, 0));
          break;
        case B_P3:
          v.push_back(mk(A2, A, 0, 0, A3, 0, 0, d, d, d, 1, d, d, d, 0));
          v.push_back(mk(A2, Ad, dA2, A, dA3, 0, 0, d, d, d, 2, d, d, d, 0));
          break;
        case B_H:
          v.push_back(mk(Tp, A3, 0, 0, Tn, A, A2, d, d, d, 1, d, d, d, 1));
          v.push_back(mk(Tp, dA3, dTp, A3, dTn, Ad, dA2, d, d, d, 2, d, d, d, 0));
          break;
        case B_S:
          v.push_back(mk(Tp, Tp, 0, 0, Tn, 0, 0, d, d, d, 1, d, d, d, 0));
          v.push_back(mk(Tp, dTp, dTp, Tp, dTn, 0, 0, d, d, d, 2, d, d, d, 0));
          break;
        case B_D: {
          GemmItem it = mk(Tp, dTp, 0, 0, nullptr, 0, 0, d, d, d, 1, d, d, d, 0);
          it.F = g.blocks[b].gen + (size_t)d * d;
          it.fstride = (long)d * d;
          it.nF = g.K;
          it.tr_out = g.trace_part + (size_t)g.trace_tile_off[b] * g.K;
          v.push_back(it);
          break;
        }
        case B_XL:
          v.push_back(mk(Tp, Xq, 0, 0, Xn, 0, 0, d, R, d, 1, d, R, R, 0));
          v.push_back(mk(Tp, Lr, 0, 0, Ln, 0, 0, d, R, d, 1, d, R, R, 0));
          break;
      }
    }
    int t = 0;
    for (auto& it : v) {
      it.tile_start = t;
      t += tiles_of(it.m, it.n);
    }
    GemmItem* dev = nullptr;
    if (cudaMalloc(&dev, v.size() * sizeof(GemmItem)) != cudaSuccess) return {nullptr, 0};
    cudaMemcpy(dev, v.data(), v.size() * sizeof(GemmItem), cudaMemcpyHostToDevice);
    g.list_mem.push_back(dev);
    found = g.lists.emplace(key, std::make_pair(dev, (int)v.size())).first;
    g.list_tiles[key] = t;
  }
  *tiles_out = g.list_tiles[key];
  return found->second;
}

#define LCHK(x)                                                  \
  do {                                                           \
    cudaError_t e_ = (x);                                        \
    if (e_ != cudaSuccess) {                                     \
      g.err = std::string(#x) + ": " + cudaGetErrorString(e_);   \
      return SQOC_ERR_CUDA;                                      \
    }                                                            \
  } while (0)

static int gemm(LargeGroup& g, int op, int p, int q, int r, GemmArgs a, cudaStream_t st) {
  int tiles = 0;
  auto lst = get_list(g, op, p, q, r, &tiles);
  if (!lst.first) {
    g.err = "work list allocation failed";
    return SQOC_ERR_CUDA;
  }
  cudaError_t e;
  switch (op) {
    case B_C: e = launch_gemm<OP_N, OP_C, EPI_STORE>(lst.first, lst.second, tiles, a, st); break;
    case B_D: e = launch_gemm<OP_C, OP_N, EPI_TRACE>(lst.first, lst.second, tiles, a, st); break;
    case B_XL: e = launch_gemm<OP_C, OP_N, EPI_STORE>(lst.first, lst.second, tiles, a, st); break;
    default: e = launch_gemm<OP_N, OP_N, EPI_STORE>(lst.first, lst.second, tiles, a, st); break;
  }
  if (e != cudaSuccess) {
    g.err = std::string("zgemm launch: ") + cudaGetErrorString(e);
    return SQOC_ERR_CUDA;
  }
  g.launches++;
  return SQOC_OK;
}

int large_init(LargeGroup& g, const std::vector<LargeBlockSpec>& blocks, int K, int N, bool gate) {
  g.blocks = blocks;
  g.nblk = (int)blocks.size();
  g.K = K;
  g.N = N;
  g.gate = gate;
  g.off.resize(g.nblk);
  g.offr.resize(g.nblk);
  g.total = g.totalr = 0;
  g.trace_tile_off.assign(g.nblk + 1, 0);
  for (int b = 0; b < g.nblk; ++b) {
    const int d = blocks[b].d;
    g.off[b] = g.total;
    g.total += (size_t)d * d;
    g.offr[b] = g.totalr;
    g.totalr += (size_t)d * (gate ? d : 1);
    g.trace_tile_off[b + 1] = g.trace_tile_off[b] + tiles_of(d, d);
  }
  g.trace_tiles = g.trace_tile_off[g.nblk];
  const size_t bytes = g.total * sizeof(double2);
  double2** sq[] = {&g.A, &g.Ad, &g.A2, &g.dA2, &g.A3, &g.dA3, &g.T[0], &g.T[1], &g.dT[0], &g.dT[1]};
  for (auto pp : sq) LCHK(cudaMalloc(pp, bytes));
  double2** rect[] = {&g.X[0], &g.X[1], &g.L[0], &g.L[1]};
  for (auto pp : rect) LCHK(cudaMalloc(pp, g.totalr * sizeof(double2)));
  LCHK(cudaMalloc(&g.trace_part, (size_t)g.trace_tiles * K * sizeof(double2)));
  LCHK(cudaMalloc(&g.tau_dev, g.nblk * sizeof(double2)));
  LCHK(cudaMalloc(&g.norm_dev, sizeof(double)));
  std::vector<double> gn, w;
  std::vector<int> dims, gidx;
  std::vector<const double2*> gen, tgt, x0;
  for (auto& b : blocks) {
    for (int k = 0; k <= K; ++k) gn.push_back(b.gen_norm[k]);
    dims.push_back(b.d);
    gidx.push_back(b.global_index);
    gen.push_back(b.gen);
    tgt.push_back(b.target);
    x0.push_back(b.x0);
    w.push_back(b.weight);
  }
  LCHK(cudaMalloc(&g.gnorm_dev, gn.size() * sizeof(double)));
  LCHK(cudaMemcpy(g.gnorm_dev, gn.data(), gn.size() * sizeof(double), cudaMemcpyHostToDevice));
  LCHK(cudaMalloc(&g.d_dev, (g.nblk + 1) * sizeof(int)));
  LCHK(cudaMemcpy(g.d_dev, dims.data(), g.nblk * sizeof(int), cudaMemcpyHostToDevice));
  LCHK(cudaMalloc(&g.off_dev, g.nblk * sizeof(size_t)));
  LCHK(cudaMemcpy(g.off_dev, g.off.data(), g.nblk * sizeof(size_t), cudaMemcpyHostToDevice));
  LCHK(cudaMalloc(&g.offr_dev, g.nblk * sizeof(size_t)));
  LCHK(cudaMemcpy(g.offr_dev, g.offr.data(), g.nblk * sizeof(size_t), cudaMemcpyHostToDevice));
  LCHK(cudaMalloc(&g.gen_dev, g.nblk * sizeof(double2*)));
  LCHK(cudaMemcpy(g.gen_dev, gen.data(), g.nblk * sizeof(double2*), cudaMemcpyHostToDevice));
  LCHK(cudaMalloc(&g.tgt_dev, g.nblk * sizeof(double2*)));
  LCHK(cudaMemcpy(g.tgt_dev, tgt.data(), g.nblk * sizeof(double2*), cudaMemcpyHostToDevice));
  LCHK(cudaMalloc(&g.x0_dev, g.nblk * sizeof(double2*)));
  LCHK(cudaMemcpy(g.x0_dev, x0.data(), g.nblk * sizeof(double2*), cudaMemcpyHostToDevice));
  LCHK(cudaMalloc(&g.w_dev, g.nblk * sizeof(double)));
  LCHK(cudaMemcpy(g.w_dev, w.data(), g.nblk * sizeof(double), cudaMemcpyHostToDevice));
  LCHK(cudaMalloc(&g.gidx_dev, g.nblk * sizeof(int)));
  LCHK(cudaMemcpy(g.gidx_dev, gidx.data(), g.nblk * sizeof(int), cudaMemcpyHostToDevice));
  LCHK(cudaMalloc(&g.tile_off_dev, (g.nblk + 1) * sizeof(int)));
  LCHK(cudaMemcpy(g.tile_off_dev, g.trace_tile_off.data(), (g.nblk + 1) * sizeof(int), cudaMemcpyHostToDevice));
  return SQOC_OK;
}

void large_free(LargeGroup& g) {
  double2* bufs[] = {g.A, g.Ad, g.A2, g.dA2, g.A3, g.dA3, g.T[0], g.T[1], g.dT[0], g.dT[1],
                     g.X[0], g.X[1], g.L[0], g.L[1], g.trace_part, g.tau_dev};
  for (auto b : bufs) cudaFree(b);
  cudaFree(g.norm_dev);
  cudaFree(g.gnorm_dev);
  cudaFree(g.d_dev);
  cudaFree(g.off_dev);
  cudaFree(g.offr_dev);
  cudaFree(g.gen_dev);
  cudaFree(g.tgt_dev);
  cudaFree(g.x0_dev);
  cudaFree(g.w_dev);
  cudaFree(g.gidx_dev);
  cudaFree(g.tile_off_dev);
  for (auto m : g.list_mem) cudaFree(m);
  g.list_mem.clear();
  g.lists.clear();
  g.list_tiles.clear();
}

int large_eval(LargeGroup& g, const LargeArgs& a, cudaStream_t st) {
  const int K = g.K, N = g.N, nblk = g.nblk;
  int maxd = 0;
  for (auto& b : g.blocks) maxd = std::max(maxd, b.d);
  const dim3 ew_grid((unsigned)std::min<size_t>(((size_t)maxd * maxd + 255) / 256, 4096), nblk);
  const int* toff = g.tile_off_dev;
  g.launches = 0;
  for (int s = 0; s < a.batch; ++s) {
    const double* u = a.u + (size_t)s * K * N;
    // ---- plan (nb, s) from the norm bound over all slices and blocks ----
    LCHK(cudaMemsetAsync(g.norm_dev, 0, sizeof(double), st));
    bound_kernel<<<std::max(1, std::min((N + 255) / 256, 148)), 256, 0, st>>>(
        u, K, N, nblk, g.gnorm_dev, reinterpret_cast<unsigned long long*>(g.norm_dev));
    LCHK(cudaGetLastError());
    double bound = 0.0;
    LCHK(cudaMemcpyAsync(&bound, g.norm_dev, sizeof(double), cudaMemcpyDeviceToHost, st));
    LCHK(cudaStreamSynchronize(st));
    g.launches++;
    int nb, sq;
    choose_taylor_host(bound, nb, sq);
    const double scale = std::ldexp(1.0, -sq);
    const double cm = inv_fact(3 * nb);
    // ---- forward sweep ----
    init_xl_kernel<<<ew_grid, 256, 0, st>>>(g.gate, 1, g.d_dev, g.offr_dev, g.x0_dev, g.tgt_dev, g.X[0], g.L[0]);
    LCHK(cudaGetLastError());
    g.launches++;
    int q = 0, r = 0;
    GemmArgs one{1.0, 0.0, 0.0, 0.0};
    for (int j = 0; j < N; ++j) {
      build_a_kernel<<<ew_grid, 256, 0, st>>>(j, K, N, u, g.d_dev, g.off_dev, g.gen_dev, scale, g.A);
      LCHK(cudaGetLastError());
      g.launches++;
      int rc;
      if ((rc = gemm(g, F_A2, 0, 0, 0, one, st))) return rc;
      if ((rc = gemm(g, F_A3, 0, 0, 0, one, st))) return rc;
      const int t0 = nb - 1;
      horner_init_kernel<<<ew_grid, 256, 0, st>>>(0, g.d_dev, g.off_dev, cm, inv_fact(3 * t0), inv_fact(3 * t0 + 1),
                                                  inv_fact(3 * t0 + 2), g.A, g.A2, g.A3, g.Ad, g.dA2, g.dA3, g.T[0],
                                                  g.dT[0]);
      LCHK(cudaGetLastError());
      g.launches++;
      int p = 0;
      for (int t = nb - 2; t >= 0; --t) {
        GemmArgs h{1.0, inv_fact(3 * t + 1), inv_fact(3 * t + 2), inv_fact(3 * t)};
        if ((rc = gemm(g, F_H, p, 0, 0, h, st))) return rc;
        p ^= 1;
      }
      for (int i = 0; i < sq; ++i) {
        if ((rc = gemm(g, F_S, p, 0, 0, one, st))) return rc;
        p ^= 1;
      }
      if ((rc = gemm(g, F_X, p, q, 0, one, st))) return rc;
      q ^= 1;
    }
    tau_kernel<<<nblk, 256, 0, st>>>(g.gate, 1, g.d_dev, g.offr_dev, g.X[q], g.tgt_dev, g.tau_dev,
                                     a.tau_out + (size_t)s * a.tau_stride, g.gidx_dev);
    LCHK(cudaGetLastError());
    g.launches++;
    // ---- backward sweep ----
    for (int j = N - 1; j >= 0; --j) {
      build_a_kernel<<<ew_grid, 256, 0, st>>>(j, K, N, u, g.d_dev, g.off_dev, g.gen_dev, scale, g.A);
      LCHK(cudaGetLastError());
      g.launches++;
      int rc;
      if ((rc = gemm(g, B_C, 0, q, r, GemmArgs{scale, 0.0, 0.0, 0.0}, st))) return rc;
      if ((rc = gemm(g, B_P2, 0, 0, 0, one, st))) return rc;
      if ((rc = gemm(g, B_P3, 0, 0, 0, one, st))) return rc;
      const int t0 = nb - 1;
      horner_init_kernel<<<ew_grid, 256, 0, st>>>(1, g.d_dev, g.off_dev, cm, inv_fact(3 * t0), inv_fact(3 * t0 + 1),
                                                  inv_fact(3 * t0 + 2), g.A, g.A2, g.A3, g.Ad, g.dA2, g.dA3, g.T[0],
                                                  g.dT[0]);
      LCHK(cudaGetLastError());
      g.launches++;
      int p = 0;
      for (int t = nb - 2; t >= 0; --t) {
        GemmArgs h{1.0, inv_fact(3 * t + 1), inv_fact(3 * t + 2), inv_fact(3 * t)};
        if ((rc = gemm(g, B_H, p, 0, 0, h, st))) return rc;
        p ^= 1;
      }
      for (int i = 0; i < sq; ++i) {
        if ((rc = gemm(g, B_S, p, 0, 0, one, st))) return rc;
        p ^= 1;
      }
      if ((rc = gemm(g, B_D, p, 0, 0, one, st))) return rc;
      trace_reduce_kernel<<<nblk, 256, 0, st>>>(j, K, N, toff, g.trace_part, g.tau_dev, g.w_dev, g.gidx_dev,
                                                a.gradb + (size_t)s * K * N, a.gradb_block_stride);
      LCHK(cudaGetLastError());
      g.launches++;
      if ((rc = gemm(g, B_XL, p, q, r, one, st))) return rc;
      q ^= 1;
      r ^= 1;
    }
  }
  return SQOC_OK;
}

}  // namespace sqoc
