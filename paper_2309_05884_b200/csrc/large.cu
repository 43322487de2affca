// Large-block GRAPE path: host orchestration + elementwise / reduction kernels.
// See large.cuh for the per-slice algebra and zgemm.cuh for the DMMA GEMM.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../../include/symqoc_b200.h"
#include "devonce.h"
#include "large.cuh"
#include "schemes.h"

namespace sqoc {

// ------------------------------------------------------------------ propagator schemes
// R(A) = y(A / 2^s)^(2^s) with y an exact Taylor polynomial evaluated by an optimized product
// scheme (coefficients derived in tools/derive_expm_schemes.py; same s4 as tiny.cuh):
//   s4: degree 12 in 4 products (theta 0.33),  s5: degree 18 in 5 products (theta 1.10)
// versus 5 and 7 products for Paterson-Stockmeyer at the same degrees.  Every step is one
// GEMM C = L R whose epilogue writes up to two linear combinations alpha acc + sum_t beta_t
// E_t + gamma I over the basis slots E = (A, A2, A3, A6) -- so the schemes need no separate
// elementwise passes.  Slots: 0 A, 1 A2, 2 A3, 3 A6, 4 P, 5 Q, 6 W1, 7 W2, 8 Y (unsquared R).
struct PolyOut {
  int slot;
  double alpha, beta[4], gamma;
};
struct PolyStep {
  int L, R, nout;
  PolyOut out[2];
};
struct PolyScheme {
  int degree, nsteps;
  double theta;
  PolyStep step[5];
};
constexpr int kSlots = 9, kSlotY = 8;

// s4: A2 = A A; A3 = A2 A, P = x6 A3 + x4 A + x5 A2; Z = P A3 + z(A) -> Q, W = Z + b(A) -> W1;
//     Y = W1 Q + c(A)
static const PolyScheme kS4 = {
    12, 4, 0.33,
    {{0, 0, 1, {{1, 1.0, {0, 0, 0, 0}, 0.0}}},
     {1, 0, 2, {{2, 1.0, {0, 0, 0, 0}, 0.0}, {4, SQOC_S4_X6, {SQOC_S4_X4, SQOC_S4_X5, 0, 0}, 0.0}}},
     {4, 2, 2,
      {{5, 1.0, {SQOC_S4_Z1, SQOC_S4_Z2, SQOC_S4_Z3, 0}, SQOC_S4_Z0},
       {6, 1.0, {SQOC_S4_Z1 + SQOC_S4_B1, SQOC_S4_Z2 + SQOC_S4_B2, SQOC_S4_Z3 + SQOC_S4_B3, 0},
        SQOC_S4_Z0 + SQOC_S4_B0}}},
     {6, 5, 1, {{8, 1.0, {SQOC_S4_C1, SQOC_S4_C2, SQOC_S4_C3, 0}, SQOC_S4_C0}}}}};

// s5: A2 = A A; A3 = A2 A, P = A + be2 A2 + be3 A3; A6 = A3 A3, Q = ga2 A2 + ga3 A3 + ga6 A6;
//     Z = P Q -> W1 = Z + b(A), W2 = Z + e(A);  Y = W1 W2 + c(A)
static const PolyScheme kS5 = {
    18, 5, 1.10,
    {{0, 0, 1, {{1, 1.0, {0, 0, 0, 0}, 0.0}}},
     {1, 0, 2, {{2, 1.0, {0, 0, 0, 0}, 0.0}, {4, SQOC_S5_BE3, {1.0, SQOC_S5_BE2, 0, 0}, 0.0}}},
     {2, 2, 2, {{3, 1.0, {0, 0, 0, 0}, 0.0}, {5, SQOC_S5_GA6, {0, SQOC_S5_GA2, SQOC_S5_GA3, 0}, 0.0}}},
     {4, 5, 2,
      {{6, 1.0, {SQOC_S5_B1, SQOC_S5_B2, SQOC_S5_B3, SQOC_S5_B6}, SQOC_S5_B0},
       {7, 1.0, {SQOC_S5_E1, SQOC_S5_E2, SQOC_S5_E3, SQOC_S5_E6}, SQOC_S5_E0}}},
     {6, 7, 1, {{8, 1.0, {SQOC_S5_C1, SQOC_S5_C2, SQOC_S5_C3, SQOC_S5_C6}, SQOC_S5_C0}}}}};

static int squarings_for(double nrm, double theta) {
  int s = 0;
  while (nrm > theta && s < 60) { nrm *= 0.5; ++s; }
  return s;
}
// Cheapest scheme for the norm bound: products + squarings (ties -> fewer squarings).
static const PolyScheme* choose_scheme(double nrm, int& s) {
  const int s4 = squarings_for(nrm, kS4.theta), s5 = squarings_for(nrm, kS5.theta);
  if (4 + s4 < 5 + s5) {
    s = s4;
    return &kS4;
  }
  s = s5;
  return &kS5;
}
static const PolyScheme& scheme_of(int degree) { return degree == 12 ? kS4 : kS5; }

static GemmArgs step_args(const PolyStep& st) {
  GemmArgs a{};
  const PolyOut& o = st.out[0];
  a.alpha = o.alpha;
  a.beta0 = o.beta[0];
  a.beta1 = o.beta[1];
  a.beta2 = o.beta[2];
  a.beta3 = o.beta[3];
  a.gamma = o.gamma;
  if (st.nout > 1) {
    const PolyOut& q = st.out[1];
    a.alpha2 = q.alpha;
    a.beta2_0 = q.beta[0];
    a.beta2_1 = q.beta[1];
    a.beta2_2 = q.beta[2];
    a.beta2_3 = q.beta[3];
    a.gamma2 = q.gamma;
  }
  return a;
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

// A[z][b] = (a_0 + sum_k u_k,(j0+z) a_k) * scale  for slice z of a slice batch (blockIdx.z)
__global__ void build_a_kernel(int j0, int K, int N, const double* __restrict__ u, const int* __restrict__ dims,
                               const size_t* __restrict__ off, const double2* const* __restrict__ gen, double scale,
                               double2* __restrict__ A, size_t slice_stride) {
  const int b = blockIdx.y;
  const int j = j0 + blockIdx.z;
  const int d = dims[b];
  const size_t dd = (size_t)d * d;
  const double2* g = gen[b];
  double uk[4];
  for (int k = 0; k < 4; ++k) uk[k] = k < K ? u[k * N + j] : 0.0;
  double2* out = A + blockIdx.z * slice_stride + off[b];
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < dd; i += (size_t)gridDim.x * blockDim.x) {
    double2 a = g[i];
    for (int k = 0; k < K; ++k) {
      const double2 e = g[(k + 1) * dd + i];
      a.x = fma(uk[k], e.x, a.x);
      a.y = fma(uk[k], e.y, a.y);
    }
    out[i] = make_double2(a.x * scale, a.y * scale);
  }
}

// g[z][b][k] = sum_pq M[z][b][p][q] * a_k[q][p]   (one CTA per (block, slice); fixed tree)
__global__ void slice_trace_kernel(int K, const int* __restrict__ dims, const size_t* __restrict__ off,
                                   const double2* const* __restrict__ gent, const double2* __restrict__ M,
                                   size_t slice_stride, double2* __restrict__ out, int nblk) {
  __shared__ double2 red[4][256];
  const int b = blockIdx.x, z = blockIdx.y;
  const int d = dims[b];
  const size_t dd = (size_t)d * d;
  const double2* m = M + z * slice_stride + off[b];
  double sx[4] = {0, 0, 0, 0}, sy[4] = {0, 0, 0, 0};
  for (size_t i = threadIdx.x; i < dd; i += blockDim.x) {
    const double2 v = m[i];
    for (int k = 0; k < K; ++k) {
      const double2 e = gent[b][(size_t)k * dd + i];  // a_k^T stored row-major
      sx[k] += v.x * e.x - v.y * e.y;
      sy[k] += v.x * e.y + v.y * e.x;
    }
  }
  for (int k = 0; k < K; ++k) red[k][threadIdx.x] = make_double2(sx[k], sy[k]);
  __syncthreads();
  for (int st = blockDim.x / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st)
      for (int k = 0; k < K; ++k) {
        red[k][threadIdx.x].x += red[k][threadIdx.x + st].x;
        red[k][threadIdx.x].y += red[k][threadIdx.x + st].y;
      }
    __syncthreads();
  }
  if (threadIdx.x < K) out[((size_t)z * nblk + b) * K + threadIdx.x] = red[threadIdx.x][0];
}

// gradb[gidx_b][k][j] = 2 w_b Re(conj(tau_b) g[j][b][k])
__global__ void hist_grad_kernel(int K, int N, int nblk, const double2* __restrict__ g, const double2* __restrict__ tau,
                                 const double* __restrict__ w, const int* __restrict__ gidx, double* __restrict__ gradb,
                                 size_t block_stride) {
  const size_t total = (size_t)N * nblk * K;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int k = i % K;
    const int b = (i / K) % nblk;
    const int j = i / ((size_t)K * nblk);
    const double2 v = g[i], t = tau[b];
    gradb[gidx[b] * block_stride + (size_t)k * N + j] = 2.0 * w[b] * (t.x * v.x + t.y * v.y);
  }
}

// X = I (gate without X_start) or xsrc[b] (state psi_0, or a sharding boundary);  L = lsrc[b]
__global__ void init_xl_kernel(int gate, int x_from_ptr, const int* __restrict__ dims, const size_t* __restrict__ offr,
                               const double2* const* __restrict__ xsrc, const double2* const* __restrict__ lsrc,
                               double2* __restrict__ X, double2* __restrict__ L) {
  const int b = blockIdx.y;
  const int d = dims[b];
  const int r = gate ? d : 1;
  const size_t n = (size_t)d * r;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const size_t o = offr[b] + i;
    if (x_from_ptr) X[o] = xsrc[b][i];
    else X[o] = make_double2((i / r == i % r) ? 1.0 : 0.0, 0.0);
    L[o] = lsrc[b][i];
  }
}

__global__ void set_tau_kernel(int nblk, const double2* __restrict__ given, double2* __restrict__ tau_local,
                               double2* __restrict__ tau_out, const int* __restrict__ gidx) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < nblk) {
    tau_local[b] = given[b];
    tau_out[gidx[b]] = given[b];
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

// out[k][c][r] = in[k][r][c]  (K stacked d x d matrices)
__global__ void transpose_kernel(const double2* __restrict__ in, double2* __restrict__ out, int d) {
  __shared__ double2 tile[32][33];
  const size_t base = (size_t)blockIdx.z * d * d;
  const int x = blockIdx.x * 32 + threadIdx.x;
  for (int yy = threadIdx.y; yy < 32; yy += 8) {
    const int y = blockIdx.y * 32 + yy;
    if (x < d && y < d) tile[yy][threadIdx.x] = in[base + (size_t)y * d + x];
  }
  __syncthreads();
  const int ox = blockIdx.y * 32 + threadIdx.x;
  for (int yy = threadIdx.y; yy < 32; yy += 8) {
    const int oy = blockIdx.x * 32 + yy;
    if (ox < d && oy < d) out[base + (size_t)oy * d + ox] = tile[threadIdx.x][yy];
  }
}

// Augmented Taylor action, one term for every (block, slice): rows of V are y_i, x_1,i, .., x_K,i.
// W_k = V a_k^T (row r of W_k = a_k v_r).  New terms:
//   y_i   <- (W_0[y_i] + sum_k u_k,i W_k[y_i]) / l
//   x_k,i <- (W_0[x_k,i] + sum_k' u_k',i W_k'[x_k,i] + W_k[y_i]) / l ;  acc_k,i += x_k,i
__global__ void sv_combine_kernel(int l, int K, int N, const double* __restrict__ u, const int* __restrict__ dims,
                                  const size_t* __restrict__ offr, double2* __restrict__ V,
                                  const double2* __restrict__ W, size_t wstride, double2* __restrict__ acc) {
  const int b = blockIdx.y;
  const int d = dims[b];
  const size_t vb = (size_t)(K + 1) * N * offr[b];
  const size_t ab = (size_t)K * N * offr[b];
  const size_t n = (size_t)N * d;
  const double inv_l = 1.0 / l;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
    const int i = e / d;
    const size_t c = e % d;
    double uk[4];
    for (int k = 0; k < 4; ++k) uk[k] = k < K ? u[k * N + i] : 0.0;
    const size_t ry = vb + (size_t)i * d + c;  // y row
    double2 wy[5];
    for (int k = 0; k <= K; ++k) wy[k] = W[k * wstride + ry];
    double2 ny = wy[0];
    for (int k = 0; k < K; ++k) { ny.x += uk[k] * wy[k + 1].x; ny.y += uk[k] * wy[k + 1].y; }
    for (int k = 0; k < K; ++k) {
      const size_t rx = vb + ((size_t)(k + 1) * N + i) * d + c;
      double2 nx = W[rx];
      for (int q = 0; q < K; ++q) {
        const double2 w = W[(q + 1) * wstride + rx];
        nx.x += uk[q] * w.x;
        nx.y += uk[q] * w.y;
      }
      nx.x = (nx.x + wy[k + 1].x) * inv_l;
      nx.y = (nx.y + wy[k + 1].y) * inv_l;
      V[rx] = nx;
      double2* ac = acc + ab + ((size_t)k * N + i) * d + c;
      ac->x += nx.x;
      ac->y += nx.y;
    }
    V[ry] = make_double2(ny.x * inv_l, ny.y * inv_l);
  }
}

// V: y_i = psi_i, x_k,i = 0;  acc = 0
__global__ void sv_init_kernel(int K, int N, const int* __restrict__ dims, const size_t* __restrict__ offr,
                               size_t totalr, const double2* __restrict__ psi, double2* __restrict__ V,
                               double2* __restrict__ acc) {
  const int b = blockIdx.y;
  const int d = dims[b];
  const size_t vb = (size_t)(K + 1) * N * offr[b];
  const size_t ab = (size_t)K * N * offr[b];
  const size_t n = (size_t)N * d;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
    const int i = e / d;
    const size_t c = e % d;
    V[vb + e] = psi[(size_t)i * totalr + offr[b] + c];
    for (int k = 0; k < K; ++k) {
      V[vb + ((size_t)(k + 1) * N) * d + e] = make_double2(0.0, 0.0);
      acc[ab + (size_t)k * N * d + e] = make_double2(0.0, 0.0);
    }
  }
}

// g[i][b][k] = <chi_{i+1}, acc_k,i>   (one CTA per (block, slice))
__global__ void sv_dot_kernel(int K, int N, int nblk, const int* __restrict__ dims, const size_t* __restrict__ offr,
                              size_t totalr, const double2* __restrict__ chi, const double2* __restrict__ acc,
                              double2* __restrict__ g) {
  __shared__ double2 red[4][256];
  const int b = blockIdx.x, i = blockIdx.y;
  const int d = dims[b];
  const size_t ab = (size_t)K * N * offr[b];
  const double2* c = chi + (size_t)(i + 1) * totalr + offr[b];
  double sx[4] = {0, 0, 0, 0}, sy[4] = {0, 0, 0, 0};
  for (int e = threadIdx.x; e < d; e += blockDim.x) {
    const double2 cv = c[e];
    for (int k = 0; k < K; ++k) {
      const double2 a = acc[ab + ((size_t)k * N + i) * d + e];
      sx[k] += cv.x * a.x + cv.y * a.y;
      sy[k] += cv.x * a.y - cv.y * a.x;
    }
  }
  for (int k = 0; k < K; ++k) red[k][threadIdx.x] = make_double2(sx[k], sy[k]);
  __syncthreads();
  for (int st = blockDim.x / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st)
      for (int k = 0; k < K; ++k) {
        red[k][threadIdx.x].x += red[k][threadIdx.x + st].x;
        red[k][threadIdx.x].y += red[k][threadIdx.x + st].y;
      }
    __syncthreads();
  }
  if (threadIdx.x < K) g[((size_t)i * nblk + b) * K + threadIdx.x] = red[threadIdx.x][0];
}

#define LCHK(x)                                                  \
  do {                                                           \
    cudaError_t e_ = (x);                                        \
    if (e_ != cudaSuccess) {                                     \
      g.err = std::string(#x) + ": " + cudaGetErrorString(e_);   \
      return SQOC_ERR_CUDA;                                      \
    }                                                            \
  } while (0)

// ------------------------------------------------------------------ host side
// Complex product algorithm for the large path: 3M (Gauss, 3 DMMAs per complex k-step) by
// default, 4M with SQOC_GEMM_4M=1 in the environment (checked once per process).
static int g_gemm_mode = -1;  // -1 unset, 3 or 4
static bool use_3m() {
  if (g_gemm_mode < 0) {
    const char* e = getenv("SQOC_GEMM_4M");
    g_gemm_mode = (e && e[0] == '1') ? 4 : 3;
  }
  return g_gemm_mode == 3;
}

int large_complex_mults() { return use_3m() ? 3 : 4; }

int large_set_complex_gemm(int mults) {
  if (mults != 3 && mults != 4) return SQOC_ERR_ARG;
  g_gemm_mode = mults;
  return SQOC_OK;
}

// Large-path 3M GEMM: the persistent warp-specialised TMA kernel (zgemm_tma.cuh, default) or the
// per-tile cp.async kernel (zgemm3m_kernel); SQOC_GEMM_TMA=0/1 in the environment or
// sqoc_set_gemm_staging selects it.
static int g_staging = -1;  // -1 unset, 0 cp.async, 1 persistent TMA
static int staging() {
  if (g_staging < 0) {
    const char* e = getenv("SQOC_GEMM_TMA");
    g_staging = (e && e[0] == '0') ? 0 : 1;
  }
  return g_staging;
}
int large_set_staging(int mode) {
  if (mode < 0 || mode > 1) return SQOC_ERR_ARG;
  g_staging = mode;
  return SQOC_OK;
}
int large_staging() { return staging(); }

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
    else
      (void)cudaGetLastError();
  });
  return fn;
}

// rows x cols complex matrix (row stride ld complex) as FP64 pairs; boxes of box_rows x 8 complex, 128B swizzle
static bool make_map(CUtensorMap* out, const double2* base, int rows, int cols, int ld, int box_rows) {
  EncodeTiledFn enc = encode_tiled();
  if (!enc || !base) return false;
  cuuint64_t dims[2] = {(cuuint64_t)2 * cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(double2)};
  cuuint32_t box[2] = {16, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  return enc(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double2*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// k-major view [k][cols] (row stride ld complex) as a 3-D map: 16 doubles (8 columns) x rows x
// floor(cols / 8) column blocks, box 16 x 8 x 8, 128B swizzle (see ItemMaps)
static bool make_map3(CUtensorMap* out, const double2* base, int rows, int cols, int ld) {
  EncodeTiledFn enc = encode_tiled();
  if (!enc || !base || cols < 64) return false;  // cols < 64: no tile has eight full column blocks
  static const bool off = [] { const char* e = getenv("SQOC_TMA3D"); return e && e[0] == '0'; }();
  if (off) return false;  // A/B knob: 2-D boxes only
  cuuint64_t dims[3] = {16, (cuuint64_t)rows, (cuuint64_t)(cols / 8)};
  cuuint64_t strides[2] = {(cuuint64_t)ld * sizeof(double2), 128};
  cuuint32_t box[3] = {16, 8, 8};
  cuuint32_t es[3] = {1, 1, 1};
  const bool ok = enc(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double2*>(base), dims, strides, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  if (!ok) memset(out, 0, sizeof(*out));
  return ok;
}

// Tensor maps of every item in both staging orientations (host); false if the driver cannot encode.
static bool build_maps(const std::vector<GemmItem>& v, std::vector<ItemMaps>& maps) {
  maps.assign(v.size(), ItemMaps{});
  for (size_t i = 0; i < v.size(); ++i) {
    const GemmItem& it = v[i];
    for (int seg = 0; seg < it.nseg; ++seg) {
      const double2* A = seg ? it.A1 : it.A0;
      const double2* B = seg ? it.B1 : it.B0;
      CUtensorMap* m = maps[i].m + 6 * seg;
      if (!make_map(m + 0, A, it.m, it.k, it.lda, GBM) || !make_map(m + 1, A, it.k, it.m, it.lda, 8) ||
          !make_map(m + 2, B, it.k, it.n, it.ldb, 8) || !make_map(m + 3, B, it.n, it.k, it.ldb, GBN))
        return false;
      // optional single-box views of the k-major orientations (the 2-D boxes remain the fallback)
      if (make_map3(m + 4, A, it.k, it.m, it.lda)) maps[i].has3d |= 1u << (2 * seg);
      if (make_map3(m + 5, B, it.k, it.n, it.ldb)) maps[i].has3d |= 1u << (2 * seg + 1);
    }
  }
  static bool said = false;
  if (!said && getenv("SQOC_DEBUG") && !v.empty()) {
    said = true;
    fprintf(stderr, "[sqoc] 3-D tensor maps of the first GEMM list: has3d = 0x%x (m = %d, n = %d)\n", maps[0].has3d,
            v[0].m, v[0].n);
  }
  return true;
}

// The persistent kernel's tiles, most expensive first (K stages x the busiest warp's DMMA sub-tiles;
// dealt round-robin over the CTAs this balances full, edge and 2-segment tiles).
constexpr double kPersistentMinK = 256.0;  // mean K (x segments) from which a list uses the persistent kernel

static void build_tiles(const std::vector<GemmItem>& v, std::vector<TileRef>& out) {
  std::vector<std::pair<double, TileRef>> all;
  for (size_t i = 0; i < v.size(); ++i) {
    const GemmItem& it = v[i];
    const int tm = (it.m + GBM - 1) / GBM, tn = (it.n + GBN - 1) / GBN;
    const double kt = (double)((it.k + GBK - 1) / GBK) * it.nseg;
    for (int a = 0; a < tm; ++a)
      for (int b = (it.herm ? a : 0); b < tn; ++b) {  // Hermitian products: the mirror tiles are not computed
        const int rows = std::min(GBM, it.m - a * GBM), cols = std::min(GBN, it.n - b * GBN);
        int th, tw, wc;
        pt_layout((rows + 7) / 8, (cols + 7) / 8, th, tw, wc);
        all.push_back({kt * (th * tw + 1), TileRef{(int)i, a * GBM, b * GBN, a * tn + b}});
      }
  }
  std::stable_sort(all.begin(), all.end(), [](const auto& x, const auto& y) { return x.first > y.first; });
  out.clear();
  for (auto& x : all) out.push_back(x.second);
}

static int sm_count() {
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 148;
  if (!cache[dev]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = n > 0 ? n : 148;
  }
  return cache[dev];
}

template <int TA, int TB, int EPI>
static cudaError_t launch_gemm(const GemmItem* items, const ItemMaps* maps, const TileRef* tref, int* counter, int n,
                              int tiles, GemmArgs a, cudaStream_t st, int pt_tiles = -1) {
  static std::mutex mu;
  static uint64_t done = 0;
  cudaError_t e = once_per_device(mu, done, [] {
    cudaError_t r = cudaFuncSetAttribute(zgemm_kernel<TA, TB, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)G_SMEM);
    if (r == cudaSuccess)
      r = cudaFuncSetAttribute(zgemm3m_kernel<TA, TB, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G_SMEM);
    if (r == cudaSuccess)
      r = cudaFuncSetAttribute(zgemm3m_pt_kernel<TA, TB, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)PT_SMEM);
    return r;
  });
  if (e != cudaSuccess) return e;
  if (use_3m() && maps && tref && counter && staging() == 1) {
    e = cudaMemsetAsync(counter, 0, sizeof(int), st);
    if (e != cudaSuccess) return e;
    const int nt = pt_tiles >= 0 ? pt_tiles : tiles;  // the persistent list may skip mirror tiles
    zgemm3m_pt_kernel<TA, TB, EPI><<<std::min(nt, sm_count()), PT_THREADS, PT_SMEM, st>>>(items, maps, tref, nt,
                                                                                          counter, a);
  } else if (use_3m()) zgemm3m_kernel<TA, TB, EPI><<<tiles, G3THREADS, G_SMEM, st>>>(items, n, a);
  else zgemm_kernel<TA, TB, EPI><<<tiles, GTHREADS, G_SMEM, st>>>(items, n, a);
  return cudaGetLastError();
}

static int tiles_of(int m, int n) { return ((m + GBM - 1) / GBM) * ((n + GBN - 1) / GBN); }

// GEMM timing / accounting around every launch (event pairs only when g.timing is on)
static void gemm_begin(LargeGroup& g, const ListRef& l, cudaStream_t st) {
  g.gemm_macs += l.macs;
  g.gemm_launches++;
  if (!g.timing) return;
  while (g.tev.size() < g.tev_used + 2) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    g.tev.push_back(e);
  }
  cudaEventRecord(g.tev[g.tev_used], st);
}
static void gemm_end(LargeGroup& g, cudaStream_t st) {
  if (!g.timing || g.tev.size() < g.tev_used + 2) return;
  cudaEventRecord(g.tev[g.tev_used + 1], st);
  g.tev_used += 2;
}

int large_gemm_time(LargeGroup& g, double* ms) {
  double t = 0.0;
  for (size_t i = 0; i + 1 < g.tev_used; i += 2) {
    float x = 0.f;
    LCHK(cudaEventElapsedTime(&x, g.tev[i], g.tev[i + 1]));
    t += x;
  }
  *ms = t;
  return SQOC_OK;
}

static ListRef upload_list(std::vector<GemmItem>& v, std::vector<void*>& mem) {
  ListRef ref;
  int t = 0;
  for (auto& x : v) {
    x.tile_start = t;
    t += tiles_of(x.m, x.n);
  }
  if (v.empty()) return ref;
  std::vector<ItemMaps> maps;
  std::vector<TileRef> tref;
  build_tiles(v, tref);
  // short-K lists (cfg 2's ~100-dim blocks: ~13 K stages a tile) keep the per-tile kernel, whose two
  // CTAs per SM hide each other's epilogues (r02 same-box A/B: cfg 2 41.1 vs 48.6 ms)
  double kmean = 0.0;
  for (auto& x : v) kmean += (double)x.k * x.nseg / v.size();
  bool has_trace = false;
  for (auto& x : v) has_trace = has_trace || x.nF > 0;
  // Lists with fused-trace items (dense-generator and sequential state paths: B_UC, B_D) keep the cp.async
  // kernel: with the persistent kernel their per-slice gradient entries came out wrong intermittently
  // (isolated slices, 1e-12 .. 1e-4 relative, F and the other slices exact; r02, tools/race_ab.sh) -- the
  // cause is not found yet, SQOC_PT_TRACE=1 re-enables it for debugging.  The default gate path takes its
  // traces on the sparse generators (sp_trace_kernel) and is not affected.
  static const int pt_trace = [] { const char* e = getenv("SQOC_PT_TRACE"); return e ? atoi(e) : 0; }();
  const bool persistent = kmean >= kPersistentMinK && use_3m() && staging() == 1 && (pt_trace || !has_trace) &&
                          build_maps(v, maps);
  if (!persistent)  // the per-tile kernels map every tile of every item: no mirror-tile skipping
    for (auto& x : v) x.herm = 0;
  for (auto& x : v) {  // executed complex MACs (a Hermitian item runs its upper tile triangle only)
    const int tm = (x.m + GBM - 1) / GBM;
    const double frac = x.herm ? (double)(tm + 1) / (2.0 * tm) : 1.0;
    ref.macs += (double)x.m * x.n * x.k * x.nseg * frac;
  }
  if (cudaMalloc(&ref.dev, v.size() * sizeof(GemmItem)) != cudaSuccess) return ListRef{};
  cudaMemcpy(ref.dev, v.data(), v.size() * sizeof(GemmItem), cudaMemcpyHostToDevice);
  mem.push_back(ref.dev);
  if (persistent && cudaMalloc(&ref.maps, maps.size() * sizeof(ItemMaps)) == cudaSuccess &&
      cudaMalloc(&ref.tref, tref.size() * sizeof(TileRef)) == cudaSuccess) {
    cudaMemcpy(ref.maps, maps.data(), maps.size() * sizeof(ItemMaps), cudaMemcpyHostToDevice);
    cudaMemcpy(ref.tref, tref.data(), tref.size() * sizeof(TileRef), cudaMemcpyHostToDevice);
    mem.push_back(ref.maps);
    mem.push_back(ref.tref);
    ref.pt_tiles = (int)tref.size();
  } else {
    (void)cudaGetLastError();
    cudaFree(ref.maps);
    ref.maps = nullptr;  // cp.async kernel for this list
    ref.tref = nullptr;
    if (persistent) {  // allocation failure after the mirror tiles were dropped: recompute everything
      for (auto& x : v) x.herm = 0;
      cudaMemcpy(ref.dev, v.data(), v.size() * sizeof(GemmItem), cudaMemcpyHostToDevice);
    }
  }
  // The copies above come from pageable host memory: cudaMemcpy returns once the data is staged, the DMA
  // of anything larger than the inline limit (the ~75 KB tile list of cfg 3) may still be in flight, and
  // the evaluation streams are non-blocking -- they do not wait for the legacy stream the DMA runs on.
  // Without this the first launch of a freshly built list could read a partly written tile list or
  // tensor maps (r02: rare rounding-to-1e-8 gradient deviations in the first evaluation of an engine,
  // tools/repeat_check.py; the cp.async kernel only reads the 2 KB item array, which is copied inline).
  cudaDeviceSynchronize();
  ref.n = (int)v.size();
  ref.tiles = t;
  return ref;
}

// Sequential schedule ops.  Gate objective: B_UC = [M = U^dag Ad | trace Tr(U^dag dT E_k)] in one
// launch, B_CU: Ad = M U.  State objective: B_C, B_D, B_XL (vector X / Lam).
enum Op { F_STEP, F_S, F_X, B_C, B_STEP, B_S, B_D, B_XL, B_UC, B_CU, B_STEP1D, B_M, B_STEPD, B_SD };

static GemmItem mk(const double2* A0, const double2* B0, const double2* A1, const double2* B1, double2* C,
                   const double2* E0, const double2* E1, int m, int n, int k, int nseg, int lda, int ldb, int ldc,
                   int diag) {
  GemmItem it{};
  it.A0 = A0; it.B0 = B0; it.A1 = A1; it.B1 = B1; it.C = C; it.E0 = E0; it.E1 = E1;
  it.m = m; it.n = n; it.k = k; it.nseg = nseg; it.lda = lda; it.ldb = ldb; it.ldc = ldc; it.diag = diag;
  it.tiles_n = (n + GBN - 1) / GBN;
  return it;
}

static bool herm_enabled() {  // SQOC_HERM=0: compute the mirror tiles of Hermitian products too (A/B)
  const char* e = getenv("SQOC_HERM");
  return !(e && e[0] == '0');
}

// Work-list item(s) of scheme step k for one d x d block.  slot(c) / dslot(c) give the block's
// matrix for scheme slot c and its derivative.  fwd: C = L R (+ epilogue combinations over the
// basis slots); deriv: dC = L dR + dL R (+ the same combinations over the derivative basis,
// no identity term).
template <class SF, class DF>
static void push_step(std::vector<GemmItem>& v, const PolyScheme& sc, int k, int d, SF slot, DF dslot, bool fwd,
                      bool deriv) {
  const PolyStep& st = sc.step[k];
  bool used[4] = {false, false, false, false};
  for (int o = 0; o < st.nout; ++o)
    for (int t = 0; t < 4; ++t) used[t] = used[t] || st.out[o].beta[t] != 0.0;
  auto epi = [&](GemmItem& it, auto S) {
    const double2** E[4] = {&it.E0, &it.E1, &it.E2, &it.E3};
    for (int t = 0; t < 4; ++t) *E[t] = used[t] ? S(t) : nullptr;
    it.C2 = st.nout > 1 ? S(st.out[1].slot) : nullptr;
  };
  if (fwd) {
    GemmItem it = mk(slot(st.L), slot(st.R), 0, 0, slot(st.out[0].slot), 0, 0, d, d, d, 1, d, d, d, 1);
    epi(it, slot);
    // A and A3 are anti-Hermitian (A = -i dt H), so A A and A3 A3 are Hermitian: half the tiles
    it.herm = (st.L == st.R && (st.L == 0 || st.L == 2) && herm_enabled()) ? 1 : 0;
    v.push_back(it);
  }
  if (deriv) {
    GemmItem it = mk(slot(st.L), dslot(st.R), dslot(st.L), slot(st.R), dslot(st.out[0].slot), 0, 0, d, d, d, 2, d, d,
                     d, 0);
    epi(it, dslot);
    v.push_back(it);
  }
}

// Sequential schedule lists.  F_STEP / B_STEP: p = step index, q = scheme degree.
static ListRef get_list(LargeGroup& g, int op, int p, int q, int r) {
  auto key = std::make_tuple(op, p, q, r);
  auto found = g.lists.find(key);
  if (found != g.lists.end()) return found->second;
  std::vector<GemmItem> v;
  for (int b = 0; b < g.nblk; ++b) {
    const int d = g.blocks[b].d, R = g.gate ? d : 1;
    const size_t o = g.off[b], orr = g.offr[b];
    double2* Ad = g.Ad + o;
    double2 *Tp = g.T[p] + o, *Tn = g.T[1 - p] + o, *dTp = g.dT[p] + o, *dTn = g.dT[1 - p] + o;
    double2 *Xq = g.X[q] + orr, *Xn = g.X[1 - q] + orr, *Lr = g.L[r] + orr, *Ln = g.L[1 - r] + orr;
    auto slot = [&](int c) -> double2* {
      switch (c) {
        case 0: return g.A + o;
        case 1: return g.A2 + o;
        case 2: return g.A3 + o;
        case kSlotY: return g.T[0] + o;
        default: return g.xs[c - 3] + o;
      }
    };
    auto dslot = [&](int c) -> double2* {
      switch (c) {
        case 0: return g.Ad + o;
        case 1: return g.dA2 + o;
        case 2: return g.dA3 + o;
        case kSlotY: return g.dT[0] + o;
        default: return g.dxs[c - 3] + o;
      }
    };
    auto trace_item = [&]() {
      GemmItem it = mk(Tp, dTp, 0, 0, nullptr, 0, 0, d, d, d, 1, d, d, d, 0);
      it.F = g.blocks[b].gen + (size_t)d * d;
      it.fstride = (long)d * d;
      it.nF = g.K;
      it.tr_out = g.trace_part + (size_t)g.trace_tile_off[b] * g.K;
      return it;
    };
    switch (op) {
      case F_STEP: push_step(v, scheme_of(q), p, d, slot, dslot, true, false); break;
      case B_STEP: push_step(v, scheme_of(q), p, d, slot, dslot, true, true); break;
      case B_STEPD: push_step(v, scheme_of(q), p, d, slot, dslot, false, true); break;  // value from uh
      case F_S: v.push_back(mk(Tp, Tp, 0, 0, Tn, 0, 0, d, d, d, 1, d, d, d, 0)); break;
      case F_X: v.push_back(mk(Tp, Xq, 0, 0, Xn, 0, 0, d, R, d, 1, d, R, R, 0)); break;
      case B_C: v.push_back(mk(Xq, Lr, 0, 0, Ad, 0, 0, d, d, R, 1, R, R, d, 0)); break;
      case B_S:
        v.push_back(mk(Tp, Tp, 0, 0, Tn, 0, 0, d, d, d, 1, d, d, d, 0));
        v.push_back(mk(Tp, dTp, dTp, Tp, dTn, 0, 0, d, d, d, 2, d, d, d, 0));
        break;
      case B_SD: v.push_back(mk(Tp, dTp, dTp, Tp, dTn, 0, 0, d, d, d, 2, d, d, d, 0)); break;  // value from uh
      case B_D: v.push_back(trace_item()); break;
      case B_XL:
        v.push_back(mk(Tp, Xq, 0, 0, Xn, 0, 0, d, R, d, 1, d, R, R, 0));
        v.push_back(mk(Tp, Lr, 0, 0, Ln, 0, 0, d, R, d, 1, d, R, R, 0));
        break;
      case B_UC:  // gate: M (in X[0]) = U^dag Ad, and the trace item
        v.push_back(mk(Tp, Ad, 0, 0, g.X[0] + orr, 0, 0, d, d, d, 1, d, d, d, 0));
        v.push_back(trace_item());
        break;
      case B_CU:  // gate: Ad = M U
        v.push_back(mk(g.X[0] + orr, Tp, 0, 0, Ad, 0, 0, d, d, d, 1, d, d, d, 0));
        break;
      case B_M:  // gate, sparse trace: M (in X[0]) = U^dag Ad only (the trace runs in sp_trace_kernel)
        v.push_back(mk(Tp, Ad, 0, 0, g.X[0] + orr, 0, 0, d, d, d, 1, d, d, d, 0));
        break;
      case B_STEP1D: {  // sparse step 1's dense derivative term: dslot(out) = slot(L) dslot(R)
        const PolyStep& st1 = scheme_of(q).step[1];
        v.push_back(mk(slot(st1.L), dslot(st1.R), 0, 0, dslot(st1.out[0].slot), 0, 0, d, d, d, 1, d, d, d, 0));
        break;
      }
    }
  }
  ListRef ref = upload_list(v, g.list_mem);
  if (ref.dev) g.lists.emplace(key, ref);
  return ref;
}

static int gemm(LargeGroup& g, int op, int p, int q, int r, GemmArgs a, cudaStream_t st) {
  ListRef l = get_list(g, op, p, q, r);
  if (!l.dev) {
    g.err = "work list allocation failed";
    return SQOC_ERR_CUDA;
  }
  if (g.dry) return SQOC_OK;
  gemm_begin(g, l, st);
  cudaError_t e;
  switch (op) {
    case B_C: e = launch_gemm<OP_N, OP_C, EPI_STORE>(l.dev, l.maps, l.tref, g.pt_counter, l.n, l.tiles, a, st, l.pt_tiles); break;
    case B_D: e = launch_gemm<OP_C, OP_N, EPI_TRACE>(l.dev, l.maps, l.tref, g.pt_counter, l.n, l.tiles, a, st, l.pt_tiles); break;
    case B_XL: e = launch_gemm<OP_C, OP_N, EPI_STORE>(l.dev, l.maps, l.tref, g.pt_counter, l.n, l.tiles, a, st, l.pt_tiles); break;
    case B_UC: e = launch_gemm<OP_C, OP_N, EPI_MIXED>(l.dev, l.maps, l.tref, g.pt_counter, l.n, l.tiles, a, st, l.pt_tiles); break;
    case B_M: e = launch_gemm<OP_C, OP_N, EPI_STORE>(l.dev, l.maps, l.tref, g.pt_counter, l.n, l.tiles, a, st, l.pt_tiles); break;
    default: e = launch_gemm<OP_N, OP_N, EPI_STORE>(l.dev, l.maps, l.tref, g.pt_counter, l.n, l.tiles, a, st, l.pt_tiles); break;
  }
  gemm_end(g, st);
  if (e != cudaSuccess) {
    g.err = std::string("zgemm launch: ") + cudaGetErrorString(e);
    return SQOC_ERR_CUDA;
  }
  g.launches++;
  return SQOC_OK;
}

// ------------------------------------------------------------------ sparse-generator products
// Scheme steps 0 (A2 = A A) and 1 (A3 = A2 A, + P) of both schemes have A as a factor: with the
// sparse A_j they run in spmm_cols_kernel (S D) / spmm_rows_kernel (D S) (sparse.cuh), same epilogues
// as push_step.  Work lists:
//   SP_F0  forward step 0:  A2 = S A                                      (cols)
//   SP_F1  forward step 1:  A3, P = A2 S                                  (rows)
//   SP_B0R backward step 0, first half of the derivative: dA2 = dA S      (rows, raw store)
//   SP_B0C backward step 0: A2 = S A; dA2 = S dA + dA2 (+ epilogue)       (cols)
//   SP_B1  backward step 1: A3, P = A2 S; dA3, dP = dA2 S + dA3           (rows; dA3 holds the term
//          A2 dA: the dense B_STEP1D GEMM, or S (S dA) from SP_B1D)
// All-sparse derivative chain (r02): A2 dA = A (A dA), so with T = S dA kept in a free derivative slot
// (dslot 3, written only by step 2) the dense term becomes one more sparse product:
//   SP_B0T backward step 0: A2 = S A (+ epilogue); T = S dA (raw)           (cols)
//   SP_B0S backward step 0: dA2 = dA S + T (raw)                            (rows)
//   SP_B1D backward step 1: dA3 = S T (raw)                                 (cols)
enum SpOp { SP_F0, SP_F1, SP_B0R, SP_B0C, SP_B1, SP_B0T, SP_B0S, SP_B1D, SP_B0T1 };

static SpListRef sp_list(LargeGroup& g, int op, int degree) {
  auto key = std::make_tuple(op, degree, 0, 0);
  auto found = g.splists.find(key);
  if (found != g.splists.end()) return found->second;
  const int k = (op == SP_F1 || op == SP_B1 || op == SP_B1D) ? 1 : 0;
  const PolyStep& st = scheme_of(degree).step[k];
  bool used[4] = {false, false, false, false};
  for (int o = 0; o < st.nout; ++o)
    for (int t = 0; t < 4; ++t) used[t] = used[t] || st.out[o].beta[t] != 0.0;
  std::vector<SpItem> v;
  int tiles = 0;
  for (int b = 0; b < g.nblk; ++b) {
    const int d = g.blocks[b].d;
    const size_t o = g.off[b];
    auto slot = [&](int c) -> double2* {
      switch (c) {
        case 0: return g.A + o;
        case 1: return g.A2 + o;
        case 2: return g.A3 + o;
        case kSlotY: return g.T[0] + o;
        default: return g.xs[c - 3] + o;
      }
    };
    auto dslot = [&](int c) -> double2* {
      switch (c) {
        case 0: return g.Ad + o;
        case 1: return g.dA2 + o;
        case 2: return g.dA3 + o;
        case kSlotY: return g.dT[0] + o;
        default: return g.dxs[c - 3] + o;
      }
    };
    auto item = [&](bool der, const double2* D, bool raw, bool add_x, double2* C = nullptr,
                    const double2* X = nullptr) {
      SpItem it{};
      it.blk = b;
      it.D = D;
      it.C = C ? C : der ? dslot(st.out[0].slot) : slot(st.out[0].slot);
      it.add_x = add_x ? 1 : 0;
      it.X = add_x ? (X ? X : it.C) : nullptr;
      if (!raw) {
        it.diag = der ? 0 : 1;
        it.C2 = st.nout > 1 ? (der ? dslot(st.out[1].slot) : slot(st.out[1].slot)) : nullptr;
        for (int t = 0; t < 4; ++t) it.E[t] = used[t] ? (der ? dslot(t) : slot(t)) : nullptr;
      }
      it.tile_start = tiles;
      tiles += (d + g.sp_w - 1) / g.sp_w;
      v.push_back(it);
    };
    switch (op) {
      case SP_F0: item(false, slot(st.R), false, false); break;
      case SP_F1: item(false, slot(st.L), false, false); break;
      case SP_B0R: item(true, dslot(st.L), true, false); break;
      case SP_B0C:
        item(false, slot(st.R), false, false);
        item(true, dslot(st.R), false, true);
        break;
      case SP_B1:
        item(false, slot(st.L), false, false);
        item(true, dslot(st.L), false, true);
        break;
      case SP_B0T:
        item(false, slot(st.R), false, false);
        item(true, dslot(st.R), true, false, dslot(3));
        break;
      case SP_B0T1: item(true, dslot(st.R), true, false, dslot(3)); break;  // T = S dA only (A2 by spgemm_a2)
      case SP_B0S: item(true, dslot(st.L), true, true, nullptr, dslot(3)); break;
      case SP_B1D: item(true, dslot(3), true, false, dslot(2)); break;
    }
  }
  SpListRef ref;
  if (cudaMalloc(&ref.dev, v.size() * sizeof(SpItem)) != cudaSuccess) return SpListRef{};
  cudaMemcpy(ref.dev, v.data(), v.size() * sizeof(SpItem), cudaMemcpyHostToDevice);
  g.splist_mem.push_back(ref.dev);
  cudaDeviceSynchronize();  // pageable H2D copy: see upload_list
  ref.n = (int)v.size();
  ref.rows = tiles;
  g.splists.emplace(key, ref);
  return ref;
}

constexpr int kSpMaxSmem = 200 * 1024;  // one dense row of double2 in shared memory: d <= 12800

static int sp_smem_attr(LargeGroup& g) {
  static std::mutex mu;
  static uint64_t done = 0;
  cudaError_t e = once_per_device(mu, done, [] {
    const auto a = cudaFuncAttributeMaxDynamicSharedMemorySize;
    cudaError_t r = cudaFuncSetAttribute(spmm_cols_kernel<0>, a, kSpMaxSmem);
    if (r == cudaSuccess) r = cudaFuncSetAttribute(spmm_rows_kernel<0>, a, kSpMaxSmem);
    if (r == cudaSuccess) r = cudaFuncSetAttribute(sp_trace_kernel<0>, a, kSpMaxSmem);
    if (r == cudaSuccess) r = cudaFuncSetAttribute(spmm_cols_kernel<kSpMaxW>, a, kSpMaxSmem);
    if (r == cudaSuccess) r = cudaFuncSetAttribute(spmm_rows_kernel<kSpMaxW>, a, kSpMaxSmem);
    if (r == cudaSuccess) r = cudaFuncSetAttribute(sp_trace_kernel<kSpMaxW>, a, kSpMaxSmem);
    return r;
  });
  if (e != cudaSuccess) {
    g.err = std::string("sparse kernel attributes: ") + cudaGetErrorString(e);
    return SQOC_ERR_CUDA;
  }
  return SQOC_OK;
}

static int sp_launch(LargeGroup& g, int op, int degree, GemmArgs a, cudaStream_t st) {
  SpListRef l = sp_list(g, op, degree);
  if (!l.dev) {
    g.err = "sparse work list allocation failed";
    return SQOC_ERR_CUDA;
  }
  int rc = sp_smem_attr(g);
  if (rc) return rc;
  if (g.dry) return SQOC_OK;
  const bool cols = op == SP_F0 || op == SP_B0C || op == SP_B0T || op == SP_B1D || op == SP_B0T1;
  const size_t smem = g.sp_smem * g.sp_w;
  const bool full_w = g.sp_w == kSpMaxW;  // compile-time panel width
  if (cols && full_w) spmm_cols_kernel<kSpMaxW><<<l.rows, kSpThreads, smem, st>>>(l.dev, l.n, g.sp_dev, g.sp_w, a);
  else if (cols) spmm_cols_kernel<0><<<l.rows, kSpThreads, smem, st>>>(l.dev, l.n, g.sp_dev, g.sp_w, a);
  else if (full_w) spmm_rows_kernel<kSpMaxW><<<l.rows, kSpThreads, smem, st>>>(l.dev, l.n, g.sp_dev, g.sp_w, a);
  else spmm_rows_kernel<0><<<l.rows, kSpThreads, smem, st>>>(l.dev, l.n, g.sp_dev, g.sp_w, a);
  LCHK(cudaGetLastError());
  g.launches++;
  return SQOC_OK;
}

// forward scheme step k (< 2) on the sparse A
// A2 = A A on the squared pattern (step 0 of both schemes is a plain store of the product)
static int sp_a2(LargeGroup& g, cudaStream_t st) {
  if (g.dry) return SQOC_OK;
  spgemm_a2_kernel<<<dim3(128, g.nblk), 256, 0, st>>>(g.sp_dev, g.off_dev, g.A2);
  LCHK(cudaGetLastError());
  g.launches++;
  return SQOC_OK;
}

static int sp_fwd_step(LargeGroup& g, int k, int degree, GemmArgs a, cudaStream_t st) {
  if (k == 0 && g.sp_a2) return sp_a2(g, st);
  return sp_launch(g, k == 0 ? SP_F0 : SP_F1, degree, a, st);
}

// backward pair step k (< 2): value and derivative halves
static bool sp_chain() {  // all-sparse derivative chain (SQOC_SPCHAIN=0: the dense A2 dA GEMM instead)
  const char* e = getenv("SQOC_SPCHAIN");
  return !(e && e[0] == '0');
}

static int sp_pair_step(LargeGroup& g, int k, int degree, GemmArgs a, cudaStream_t st) {
  int rc;
  const GemmArgs raw{1.0, 0.0, 0.0, 0.0};
  if (k == 0) {
    if (sp_chain()) {  // step 0's epilogue is a plain store (both schemes), so raw items may share it
      if (g.sp_a2) {  // value A2 on its own pattern; only T = S dA remains an S x dense product
        if ((rc = sp_a2(g, st))) return rc;
        if ((rc = sp_launch(g, SP_B0T1, degree, raw, st))) return rc;
      } else if ((rc = sp_launch(g, SP_B0T, degree, a, st))) return rc;
      return sp_launch(g, SP_B0S, degree, raw, st);
    }
    if ((rc = sp_launch(g, SP_B0R, degree, raw, st))) return rc;
    return sp_launch(g, SP_B0C, degree, a, st);
  }
  if (sp_chain() && (rc = sp_launch(g, SP_B1D, degree, raw, st))) return rc;
  return sp_launch(g, SP_B1, degree, a, st);
}

static int sp_values(LargeGroup& g, int j, const double* u, double scale, cudaStream_t st) {
  if (g.dry) return SQOC_OK;
  sp_values_kernel<<<dim3(64, g.nblk), 256, 0, st>>>(j, g.K, g.N, u, scale, g.sp_dev);
  LCHK(cudaGetLastError());
  g.launches++;
  return SQOC_OK;
}

// Tr(U^dag N a_k) by rows (U = T[p], N = dT[p]) into sp_part, then the per-slice gradient entries
static int sp_trace(LargeGroup& g, int j, int p, const LargeArgs& a, int s_idx, cudaStream_t st) {
  int rc = sp_smem_attr(g);
  if (rc) return rc;
  if (g.dry) return SQOC_OK;
  if (g.sp_w == kSpMaxW)
    sp_trace_kernel<kSpMaxW><<<g.sp_trace_tiles, kSpThreads, g.sp_smem * g.sp_w, st>>>(
        g.sp_trace_dev + (size_t)p * g.nblk, g.nblk, g.sp_dev, g.K, g.sp_w);
  else
    sp_trace_kernel<0><<<g.sp_trace_tiles, kSpThreads, g.sp_smem * g.sp_w, st>>>(g.sp_trace_dev + (size_t)p * g.nblk,
                                                                         g.nblk, g.sp_dev, g.K, g.sp_w);
  LCHK(cudaGetLastError());
  trace_reduce_kernel<<<g.nblk, 256, 0, st>>>(j, g.K, g.N, g.sp_rowoff_dev, g.sp_part, g.tau_dev, g.w_dev, g.gidx_dev,
                                              a.gradb + (size_t)s_idx * g.K * g.N, a.gradb_block_stride);
  LCHK(cudaGetLastError());
  g.launches += 2;
  return SQOC_OK;
}

// Upload the patterns (CSR from the host spec, CSC derived here) when every block is sparse enough.
static int sp_init(LargeGroup& g, const std::vector<LargeBlockSpec>& blocks) {
  const char* env = getenv("SQOC_SPARSE");
  if (env && env[0] == '0') return SQOC_OK;
  for (auto& b : blocks)
    if (b.sp_rp.size() != (size_t)b.d + 1 || (double)b.sp_ci.size() > (double)b.d * b.d / 8.0) return SQOC_OK;
  std::vector<SpBlockDev> host(g.nblk);
  std::vector<int> rowoff(g.nblk + 1, 0);
  bool a2_all = true;  // every block's A2 = A A pattern is small enough for the sparse x sparse kernel
  int maxd = 0;
  const int K1 = g.K + 1;
  for (int b = 0; b < g.nblk; ++b) {
    const LargeBlockSpec& bs = blocks[b];
    const int d = bs.d, nnz = (int)bs.sp_ci.size();
    maxd = std::max(maxd, d);
    // row and column ELL layouts of the union pattern, rows / columns sorted by entry count (longest
    // first; entry e of the row at sorted position t at e * d + t) with per-32-chunk loop bounds
    std::vector<int> rcount(d, 0), ccount(d, 0);
    for (int i = 0; i < d; ++i) {
      rcount[i] = bs.sp_rp[i + 1] - bs.sp_rp[i];
      for (int e = bs.sp_rp[i]; e < bs.sp_rp[i + 1]; ++e) ccount[bs.sp_ci[e]]++;
    }
    auto up4 = [](int x) { return (std::max(1, x) + 3) & ~3; };  // the kernels read entry groups of 4
    const int wr = up4(*std::max_element(rcount.begin(), rcount.end()));
    const int wc = up4(*std::max_element(ccount.begin(), ccount.end()));
    // pairs: sort neighbours (2p, 2p + 1) together by their larger count, so that two adjacent lanes of
    // the rows kernel (thread per column) still store the two halves of one 32-byte sector
    auto sorted_by = [&](const std::vector<int>& cnt, std::vector<int>& perm, std::vector<int>& pos,
                         std::vector<int>& chunk, bool pairs) {
      perm.resize(d);
      for (int i = 0; i < d; ++i) perm[i] = i;
      if (pairs) {
        std::vector<int> pp((d + 1) / 2);
        for (size_t p = 0; p < pp.size(); ++p) pp[p] = (int)p;
        auto key = [&](int p) { return std::max(cnt[2 * p], 2 * p + 1 < d ? cnt[2 * p + 1] : 0); };
        std::stable_sort(pp.begin(), pp.end(), [&](int x, int y) { return key(x) > key(y); });
        int t = 0;
        for (int p : pp) {
          perm[t++] = 2 * p;
          if (2 * p + 1 < d) perm[t++] = 2 * p + 1;
        }
      } else
        std::stable_sort(perm.begin(), perm.end(), [&](int x, int y) { return cnt[x] > cnt[y]; });
      pos.resize(d);
      for (int t = 0; t < d; ++t) pos[perm[t]] = t;
      chunk.assign((d + 31) / 32, 0);
      for (int t = 0; t < d; ++t) chunk[t / 32] = std::max(chunk[t / 32], cnt[perm[t]]);
    };
    std::vector<int> r_perm, r_pos, r_cnt, c_perm, c_pos, c_cnt;
    // measured (r02, cfg 3, 6 slices): 376.98 ms with the pairs against 376.26 ms with the plain sort -- off
    static const bool pair_cols = [] { const char* e = getenv("SQOC_SPPAIRS"); return e && e[0] == '1'; }();
    sorted_by(rcount, r_perm, r_pos, r_cnt, false);
    sorted_by(ccount, c_perm, c_pos, c_cnt, pair_cols);
    std::vector<int> r_idx((size_t)wr * d, 0), c_idx((size_t)wc * d, 0);
    std::vector<double2> r_gv((size_t)K1 * wr * d, make_double2(0.0, 0.0)), c_gv((size_t)K1 * wc * d, make_double2(0.0, 0.0));
    std::vector<int> cfill(d, 0);
    for (int i = 0; i < d; ++i)  // rows ascending: each column's entries in row order
      for (int e = bs.sp_rp[i]; e < bs.sp_rp[i + 1]; ++e) {
        const int er = e - bs.sp_rp[i], c = bs.sp_ci[e], ec = cfill[c]++;
        const size_t ri = (size_t)er * d + r_pos[i], cj = (size_t)ec * d + c_pos[c];
        r_idx[ri] = c;
        c_idx[cj] = i;
        for (int k = 0; k < K1; ++k) {
          const double2 v = bs.sp_gv[(size_t)k * nnz + e];
          r_gv[(size_t)k * wr * d + ri] = v;
          c_gv[(size_t)k * wc * d + cj] = v;
        }
      }
    auto up = [&](const void* src, size_t bytes) -> void* {
      void* dst = nullptr;
      if (cudaMalloc(&dst, std::max<size_t>(bytes, 16)) != cudaSuccess) return nullptr;
      g.sp_mem.push_back(dst);
      if (bytes && src) cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice);
      return dst;
    };
    SpBlockDev& h = host[b];
    h.d = d;
    h.wr = wr;
    h.wc = wc;
    h.r_perm = static_cast<const int*>(up(r_perm.data(), r_perm.size() * sizeof(int)));
    h.c_perm = static_cast<const int*>(up(c_perm.data(), c_perm.size() * sizeof(int)));
    h.r_cnt = static_cast<const int*>(up(r_cnt.data(), r_cnt.size() * sizeof(int)));
    h.c_cnt = static_cast<const int*>(up(c_cnt.data(), c_cnt.size() * sizeof(int)));
    h.r_idx = static_cast<const int*>(up(r_idx.data(), r_idx.size() * sizeof(int)));
    h.c_idx = static_cast<const int*>(up(c_idx.data(), c_idx.size() * sizeof(int)));
    h.r_gv = static_cast<const double2*>(up(r_gv.data(), r_gv.size() * sizeof(double2)));
    h.c_gv = static_cast<const double2*>(up(c_gv.data(), c_gv.size() * sizeof(double2)));
    h.r_sv = static_cast<double2*>(up(nullptr, (size_t)wr * d * sizeof(double2)));
    h.c_sv = static_cast<double2*>(up(nullptr, (size_t)wc * d * sizeof(double2)));
    {  // symbolic A2 = A A: per nonzero (i, k) of the squared pattern the (A_ij, A_jk) pairs, j ascending
      auto sv_off = [&](int i, int e) { return (e - bs.sp_rp[i]) * d + r_pos[i]; };  // CSR entry e of row i in r_sv
      double est = 0.0;  // pair count; dense-ish patterns keep the S x dense product
      for (int i = 0; i < d; ++i)
        for (int e = bs.sp_rp[i]; e < bs.sp_rp[i + 1]; ++e) est += rcount[bs.sp_ci[e]];
      a2_all = a2_all && est <= 4.0 * (double)d * d;
      std::vector<int> a2_ptr(1, 0), a2_out;
      std::vector<int2> a2_pairs;
      std::vector<std::vector<int2>> acc(d);
      std::vector<int> touched;
      for (int i = 0; i < d && a2_all; ++i) {
        touched.clear();
        for (int e = bs.sp_rp[i]; e < bs.sp_rp[i + 1]; ++e) {
          const int j = bs.sp_ci[e];
          for (int f = bs.sp_rp[j]; f < bs.sp_rp[j + 1]; ++f) {
            const int k = bs.sp_ci[f];
            if (acc[k].empty()) touched.push_back(k);
            acc[k].push_back(make_int2(sv_off(i, e), sv_off(j, f)));
          }
        }
        std::sort(touched.begin(), touched.end());
        for (int k : touched) {
          a2_out.push_back(i * d + k);
          a2_pairs.insert(a2_pairs.end(), acc[k].begin(), acc[k].end());
          a2_ptr.push_back((int)a2_pairs.size());
          acc[k].clear();
        }
      }
      h.a2_nnz = (int)a2_out.size();
      h.a2_ptr = static_cast<const int*>(up(a2_ptr.data(), a2_ptr.size() * sizeof(int)));
      h.a2_out = static_cast<const int*>(up(a2_out.data(), a2_out.size() * sizeof(int)));
      h.a2_pairs = static_cast<const int2*>(up(a2_pairs.data(), a2_pairs.size() * sizeof(int2)));
      if (!h.a2_ptr || !h.a2_out || !h.a2_pairs) {
        g.err = "sparse A2 pattern allocation failed";
        return SQOC_ERR_CUDA;
      }
    }
    if (!h.r_perm || !h.c_perm || !h.r_cnt || !h.c_cnt || !h.r_idx || !h.c_idx || !h.r_gv || !h.c_gv || !h.r_sv ||
        !h.c_sv) {
      g.err = "sparse pattern allocation failed";
      return SQOC_ERR_CUDA;
    }
    rowoff[b + 1] = rowoff[b] + d;
  }
  LCHK(cudaMalloc(&g.sp_dev, g.nblk * sizeof(SpBlockDev)));
  LCHK(cudaMemcpy(g.sp_dev, host.data(), g.nblk * sizeof(SpBlockDev), cudaMemcpyHostToDevice));
  LCHK(cudaMalloc(&g.sp_rowoff_dev, (g.nblk + 1) * sizeof(int)));
  LCHK(cudaMemcpy(g.sp_rowoff_dev, rowoff.data(), (g.nblk + 1) * sizeof(int), cudaMemcpyHostToDevice));
  LCHK(cudaMalloc(&g.sp_part, (size_t)rowoff[g.nblk] * std::max(g.K, 1) * sizeof(double2)));
  g.sp_smem = (size_t)maxd * sizeof(double2);  // one dense row or column panel of width 1
  g.sp_w = (int)std::max<size_t>(1, std::min<size_t>(kSpMaxW, kSpMaxSmem / g.sp_smem));
  std::vector<SpTraceItem> tr;
  for (int p = 0; p < 2; ++p) {
    int tiles = 0;
    for (int b = 0; b < g.nblk; ++b) {
      SpTraceItem it{};
      it.blk = b;
      it.tile_start = tiles;
      tiles += (g.blocks[b].d + g.sp_w - 1) / g.sp_w;
      it.U = g.T[p] + g.off[b];
      it.N = g.dT[p] + g.off[b];
      it.part = g.sp_part + (size_t)rowoff[b] * g.K;
      tr.push_back(it);
    }
    g.sp_trace_tiles = tiles;
  }
  LCHK(cudaMalloc(&g.sp_trace_dev, tr.size() * sizeof(SpTraceItem)));
  LCHK(cudaMemcpy(g.sp_trace_dev, tr.data(), tr.size() * sizeof(SpTraceItem), cudaMemcpyHostToDevice));
  g.sp_on = g.sp_smem <= (size_t)kSpMaxSmem;
  const char* a2env = getenv("SQOC_SPGEMM");
  g.sp_a2 = g.sp_on && a2_all && !(a2env && a2env[0] == '0');
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
  LCHK(cudaMemset(g.A2, 0, bytes));  // spgemm_a2_kernel writes the pattern of A A only: the rest stays zero
  for (int i = 0; i < 5; ++i) {
    LCHK(cudaMalloc(&g.xs[i], bytes));
    LCHK(cudaMalloc(&g.dxs[i], bytes));
  }
  double2** rect[] = {&g.X[0], &g.X[1], &g.L[0], &g.L[1]};
  for (auto pp : rect) LCHK(cudaMalloc(pp, g.totalr * sizeof(double2)));
  LCHK(cudaMalloc(&g.trace_part, (size_t)g.trace_tiles * K * sizeof(double2)));
  LCHK(cudaMalloc(&g.tau_dev, g.nblk * sizeof(double2)));
  LCHK(cudaMalloc(&g.norm_dev, sizeof(double)));
  LCHK(cudaMalloc(&g.pt_counter, sizeof(int)));
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
  {  // a_k^T for k = 0..K per block (state-vector schedule: W_k = V a_k^T)
    std::vector<const double2*> gt;
    for (int b = 0; b < g.nblk; ++b) {
      const int d = blocks[b].d;
      double2* t = nullptr;
      LCHK(cudaMalloc(&t, (size_t)(K + 1) * d * d * sizeof(double2)));
      transpose_kernel<<<dim3((d + 31) / 32, (d + 31) / 32, K + 1), dim3(32, 8)>>>(blocks[b].gen, t, d);
      LCHK(cudaGetLastError());
      g.gentall_mem.push_back(t);
      gt.push_back(t);
    }
    LCHK(cudaMalloc(&g.gentall_dev, g.nblk * sizeof(double2*)));
    LCHK(cudaMemcpy(g.gentall_dev, gt.data(), g.nblk * sizeof(double2*), cudaMemcpyHostToDevice));
  }
  {  // a_k^T per block for the history-mode slice traces
    std::vector<const double2*> gt;
    for (int b = 0; b < g.nblk; ++b) {
      const int d = blocks[b].d;
      double2* t = nullptr;
      LCHK(cudaMalloc(&t, (size_t)K * d * d * sizeof(double2)));
      transpose_kernel<<<dim3((d + 31) / 32, (d + 31) / 32, K), dim3(32, 8)>>>(blocks[b].gen + (size_t)d * d, t, d);
      LCHK(cudaGetLastError());
      g.gent_mem.push_back(t);
      gt.push_back(t);
    }
    LCHK(cudaMalloc(&g.gent_dev, g.nblk * sizeof(double2*)));
    LCHK(cudaMemcpy(g.gent_dev, gt.data(), g.nblk * sizeof(double2*), cudaMemcpyHostToDevice));
  }
  LCHK(cudaMalloc(&g.tile_off_dev, (g.nblk + 1) * sizeof(int)));
  LCHK(cudaMemcpy(g.tile_off_dev, g.trace_tile_off.data(), (g.nblk + 1) * sizeof(int), cudaMemcpyHostToDevice));
  const int rc_sp = sp_init(g, blocks);
  // the setup above used the legacy default stream (memset of A2, generator transposes); evaluations run on
  // non-blocking streams that do not wait for it
  LCHK(cudaDeviceSynchronize());
  return rc_sp;
}

int large_set_norms(LargeGroup& g, const std::vector<double>& gn) {
  if (gn.size() != (size_t)g.nblk * (g.K + 1)) {
    g.err = "norm bound array has the wrong size";
    return SQOC_ERR_ARG;
  }
  for (int b = 0; b < g.nblk; ++b)
    for (int k = 0; k <= g.K; ++k) g.blocks[b].gen_norm[k] = gn[(size_t)b * (g.K + 1) + k];
  LCHK(cudaMemcpy(g.gnorm_dev, gn.data(), gn.size() * sizeof(double), cudaMemcpyHostToDevice));
  return SQOC_OK;
}

void large_free(LargeGroup& g) {
  double2* bufs[] = {g.A, g.Ad, g.A2, g.dA2, g.A3, g.dA3, g.T[0], g.T[1], g.dT[0], g.dT[1],
                     g.X[0], g.X[1], g.L[0], g.L[1], g.trace_part, g.tau_dev};
  for (auto b : bufs) cudaFree(b);
  for (int i = 0; i < 5; ++i) {
    cudaFree(g.xs[i]);
    cudaFree(g.dxs[i]);
  }
  cudaFree(g.norm_dev);
  cudaFree(g.pt_counter);
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
  double2* hb[] = {g.h_chain, g.h_X, g.h_L, g.h_dH[0], g.h_dH[1], g.h_g, g.h_I};
  for (auto x : hb) cudaFree(x);
  for (auto x : g.h_d) cudaFree(x);
  for (auto m : g.gent_mem) cudaFree(m);
  g.gent_mem.clear();
  for (auto m : g.gentall_mem) cudaFree(m);
  g.gentall_mem.clear();
  cudaFree(g.gentall_dev);
  cudaFree(g.uh);
  g.uh = nullptr;
  double2* sv[] = {g.sv_U, g.sv_chunk, g.sv_psi, g.sv_chi, g.sv_V, g.sv_W, g.sv_acc, g.sv_g, g.mf_t};
  for (auto x : sv) cudaFree(x);
  for (auto m : g.sp_mem) cudaFree(m);
  g.sp_mem.clear();
  for (auto m : g.splist_mem) cudaFree(m);
  g.splist_mem.clear();
  g.splists.clear();
  cudaFree(g.sp_dev);
  cudaFree(g.sp_rowoff_dev);
  cudaFree(g.sp_part);
  cudaFree(g.sp_trace_dev);
  cudaFree(g.chunk_vec);
  cudaFree(g.chunk_tau);
  cudaFree(g.chunk_ptrs);
  for (auto e : g.carry_ev)
    if (e) cudaEventDestroy(e);
  cudaFree(g.gent_dev);
  for (auto m : g.hlist_mem) cudaFree(m);
  g.hlist_mem.clear();
  g.hlists.clear();
  for (auto m : g.list_mem) cudaFree(m);
  g.list_mem.clear();
  g.lists.clear();
  for (auto e : g.tev) cudaEventDestroy(e);
  g.tev.clear();
}

// ------------------------------------------------------------------ boundary conditions
static int bc_init(LargeGroup& g, double2* X, double2* L, dim3 grid, cudaStream_t st) {
  const bool xp = g.bc_x_dev != nullptr || !g.gate;
  init_xl_kernel<<<grid, 256, 0, st>>>(g.gate, xp ? 1 : 0, g.d_dev, g.offr_dev,
                                       g.bc_x_dev ? g.bc_x_dev : g.x0_dev, g.bc_l_dev ? g.bc_l_dev : g.tgt_dev, X, L);
  LCHK(cudaGetLastError());
  g.launches++;
  return SQOC_OK;
}

// tau from X_N (or the full-grid tau a chunk's phase 2 formed from the gathered products)
static int bc_tau(LargeGroup& g, const double2* XN, const LargeArgs& a, int s_idx, cudaStream_t st) {
  if (g.bc_tau) {
    set_tau_kernel<<<(g.nblk + 127) / 128, 128, 0, st>>>(g.nblk, g.bc_tau, g.tau_dev,
                                                          a.tau_out + (size_t)s_idx * a.tau_stride, g.gidx_dev);
  } else {
    tau_kernel<<<g.nblk, 256, 0, st>>>(g.gate, 1, g.d_dev, g.offr_dev, XN, g.tgt_dev, g.tau_dev,
                                       a.tau_out + (size_t)s_idx * a.tau_stride, g.gidx_dev);
  }
  LCHK(cudaGetLastError());
  g.launches++;
  return SQOC_OK;
}

// ------------------------------------------------------------------ history schedule
enum HOp { H_STEP, H_S, H_X, H_L, H_B, H_DSTEP, H_DS, H_XP1, H_XP2, H_XP3, H_LP1, H_LP2, H_LP3 };

// h_chain slots 0..8 (scheme), then S_1..S_s; derivative arrays h_d[0..7] + h_dH[2].
static size_t history_bytes(const LargeGroup& g, int C) {
  const size_t N = g.N;
  return sizeof(double2) * ((size_t)(C + 10) * N * g.total + 2 * (N + 1) * g.totalr + N * g.nblk * g.K);
}

static void hist_free(LargeGroup& g) {
  double2* hb[] = {g.h_chain, g.h_X, g.h_L, g.h_dH[0], g.h_dH[1], g.h_g, g.h_I};
  for (auto x : hb) cudaFree(x);
  for (auto& x : g.h_d) {
    cudaFree(x);
    x = nullptr;
  }
  g.h_chain = g.h_X = g.h_L = g.h_dH[0] = g.h_dH[1] = g.h_g = g.h_I = nullptr;
  for (auto m : g.hlist_mem) cudaFree(m);
  g.hlist_mem.clear();
  g.hlists.clear();
  g.h_C = 0;
}

static int hist_alloc(LargeGroup& g, int degree, int sq) {
  const int C = kSlots + sq;
  g.h_deg = degree;
  g.h_s = sq;
  if (C <= g.h_C) return SQOC_OK;  // buffers large enough; lists depend on (degree, s) via keys
  hist_free(g);
  const size_t N = g.N, sq_bytes = N * g.total * sizeof(double2);
  LCHK(cudaMalloc(&g.h_chain, (size_t)C * sq_bytes));
  LCHK(cudaMalloc(&g.h_X, (N + 1) * g.totalr * sizeof(double2)));
  LCHK(cudaMalloc(&g.h_L, (N + 1) * g.totalr * sizeof(double2)));
  for (auto& x : g.h_d) LCHK(cudaMalloc(&x, sq_bytes));
  for (auto& x : g.h_dH) LCHK(cudaMalloc(&x, sq_bytes));
  LCHK(cudaMalloc(&g.h_g, N * g.nblk * g.K * sizeof(double2)));
  if (g.gate) {  // identity blocks for the chunked prefix / suffix scans
    std::vector<double2> eye(g.totalr, make_double2(0.0, 0.0));
    for (int b = 0; b < g.nblk; ++b)
      for (int r = 0; r < g.blocks[b].d; ++r) eye[g.offr[b] + (size_t)r * g.blocks[b].d + r] = make_double2(1.0, 0.0);
    LCHK(cudaMalloc(&g.h_I, g.totalr * sizeof(double2)));
    LCHK(cudaMemcpy(g.h_I, eye.data(), g.totalr * sizeof(double2), cudaMemcpyHostToDevice));
    LCHK(cudaDeviceSynchronize());  // pageable H2D copy vs the non-blocking evaluation stream: see upload_list
  }
  g.h_C = C;
  return SQOC_OK;
}

// Work list for history op `op` (index idx, parity p), over slices [i0, i1) x blocks.
static ListRef hist_list(LargeGroup& g, int op, int idx, int p, int i0, int i1) {
  auto key = std::make_tuple(op * 1000000 + idx * 4 + p, g.h_deg * 100 + g.h_s, i0, i1);
  auto it = g.hlists.find(key);
  if (it != g.hlists.end()) return it->second;
  std::vector<GemmItem> v;
  const PolyScheme& sc = scheme_of(g.h_deg);
  for (int i = i0; i < i1; ++i)
    for (int b = 0; b < g.nblk; ++b) {
      const int d = g.blocks[b].d, R = g.gate ? d : 1;
      const size_t o = (size_t)i * g.total + g.off[b];
      auto ch = [&](int c) { return g.h_chain + (size_t)c * g.N * g.total + o; };
      double2* U = ch(kSlotY + g.h_s);
      double2* dA = g.h_d[0] + o;
      double2 *dHp = g.h_dH[p] + o, *dHn = g.h_dH[1 - p] + o;
      double2* Xi = g.h_X + (size_t)i * g.totalr + g.offr[b];
      double2* Xn = g.h_X + (size_t)(i + 1) * g.totalr + g.offr[b];
      double2* Li = g.h_L + (size_t)i * g.totalr + g.offr[b];
      double2* Ln = g.h_L + (size_t)(i + 1) * g.totalr + g.offr[b];
      auto dslot = [&](int c) -> double2* { return c == kSlotY ? g.h_dH[0] + o : g.h_d[c] + o; };
      switch (op) {
        case H_STEP: push_step(v, sc, idx, d, ch, dslot, true, false); break;
        case H_DSTEP: push_step(v, sc, idx, d, ch, dslot, false, true); break;
        case H_S: v.push_back(mk(ch(kSlotY + idx - 1), ch(kSlotY + idx - 1), 0, 0, ch(kSlotY + idx), 0, 0,
                                 d, d, d, 1, d, d, d, 0)); break;
        case H_X: v.push_back(mk(U, Xi, 0, 0, Xn, 0, 0, d, R, d, 1, d, R, R, 0)); break;
        case H_L: v.push_back(mk(U, Ln, 0, 0, Li, 0, 0, d, R, d, 1, d, R, R, 0)); break;
        case H_B: v.push_back(mk(Xi, Ln, 0, 0, dA, 0, 0, d, d, R, 1, R, R, d, 0)); break;
        case H_DS: {
          double2* S = ch(kSlotY + idx - 1);
          v.push_back(mk(S, dHp, dHp, S, dHn, 0, 0, d, d, d, 2, d, d, d, 0));
          break;
        }
      }
    }
  ListRef ref = upload_list(v, g.hlist_mem);
  if (ref.dev) g.hlists[key] = ref;
  return ref;
}

static int hgemm(LargeGroup& g, int op, int idx, int p, int i0, int i1, GemmArgs a, cudaStream_t st) {
  ListRef l = hist_list(g, op, idx, p, i0, i1);
  if (!l.dev) {
    g.err = "history work list allocation failed";
    return SQOC_ERR_CUDA;
  }
  cudaError_t e;
  gemm_begin(g, l, st);
  if (op == H_L) e = launch_gemm<OP_C, OP_N, EPI_STORE>(l.dev, l.maps, l.tref, g.pt_counter, l.n, l.tiles, a, st, l.pt_tiles);
  else if (op == H_B) e = launch_gemm<OP_N, OP_C, EPI_STORE>(l.dev, l.maps, l.tref, g.pt_counter, l.n, l.tiles, a, st, l.pt_tiles);
  else e = launch_gemm<OP_N, OP_N, EPI_STORE>(l.dev, l.maps, l.tref, g.pt_counter, l.n, l.tiles, a, st, l.pt_tiles);
  gemm_end(g, st);
  if (e != cudaSuccess) {
    g.err = std::string("zgemm launch: ") + cudaGetErrorString(e);
    return SQOC_ERR_CUDA;
  }
  g.launches++;
  return SQOC_OK;
}

// Chunked prefix / suffix scans of the X / Lam recurrences (gate): depth ~2 sqrt(N)
// launches instead of N, each batched over chunks x blocks.  Lc = chunk length.
//   X: chunk 0 runs exactly from X_0; chunks c >= 1 form local prefixes P_i = U_i ... U_{cLc}
//      (into h_d[1]), the chunk starts X[cLc] = P_{cLc-1} X[(c-1)Lc] are carried sequentially,
//      and X[i+1] = P_i X[cLc] fixes every slice up in one launch.
//   Lam: the mirror image with local suffixes Q_i = U_i^dag ... U_{(c+1)Lc-1}^dag (into h_d[2]).
static ListRef scan_list(LargeGroup& g, int op, int idx, int Lc, int C) {
  auto key = std::make_tuple(op * 1000000 + idx * 4, g.h_deg * 100 + g.h_s, Lc, C);
  auto it = g.hlists.find(key);
  if (it != g.hlists.end()) return it->second;
  const int N = g.N;
  std::vector<GemmItem> v;
  auto U = [&](int i, int b) { return g.h_chain + ((size_t)(kSlotY + g.h_s) * N + i) * g.total + g.off[b]; };
  auto X = [&](int i, int b) { return g.h_X + (size_t)i * g.totalr + g.offr[b]; };
  auto L = [&](int i, int b) { return g.h_L + (size_t)i * g.totalr + g.offr[b]; };
  auto P = [&](int i, int b) { return g.h_d[1] + (size_t)i * g.total + g.off[b]; };  // scratch before the
  auto Q = [&](int i, int b) { return g.h_d[2] + (size_t)i * g.total + g.off[b]; };  // derivative chain
  auto I = [&](int b) { return g.h_I + g.offr[b]; };
  for (int b = 0; b < g.nblk; ++b) {
    const int d = g.blocks[b].d;
    auto add = [&](const double2* A, const double2* B, double2* Cm) {
      v.push_back(mk(A, B, 0, 0, Cm, 0, 0, d, d, d, 1, d, d, d, 0));
    };
    switch (op) {
      case H_XP1:  // step t = idx of every chunk
        for (int c = 0; c < C; ++c) {
          const int i = c * Lc + idx;
          if (i >= N || idx >= Lc) continue;
          if (c == 0) add(U(i, b), X(i, b), X(i + 1, b));
          else add(U(i, b), idx == 0 ? I(b) : P(i - 1, b), P(i, b));
        }
        break;
      case H_XP2:  // carry into chunk idx (>= 2)
        add(P(idx * Lc - 1, b), X((idx - 1) * Lc, b), X(idx * Lc, b));
        break;
      case H_XP3:  // fix-up of chunks >= 1
        for (int c = 1; c < C; ++c)
          for (int i = c * Lc; i < std::min((c + 1) * Lc, N); ++i) add(P(i, b), X(c * Lc, b), X(i + 1, b));
        break;
      case H_LP1:  // step t = idx from each chunk's end
        for (int c = 0; c < C; ++c) {
          const int end = std::min((c + 1) * Lc, N);
          const int i = end - 1 - idx;
          if (i < c * Lc) continue;
          if (c == C - 1) v.push_back(mk(U(i, b), L(i + 1, b), 0, 0, L(i, b), 0, 0, d, d, d, 1, d, d, d, 0));
          else v.push_back(mk(U(i, b), idx == 0 ? I(b) : Q(i + 1, b), 0, 0, Q(i, b), 0, 0, d, d, d, 1, d, d, d, 0));
        }
        break;
      case H_LP2:  // carry: Lam at the start of chunk idx (<= C-2)
        add(Q(idx * Lc, b), L((idx + 1) * Lc, b), L(idx * Lc, b));
        break;
      case H_LP3:  // fix-up of chunks <= C-2
        for (int c = 0; c < C - 1; ++c)
          for (int i = c * Lc + 1; i < (c + 1) * Lc; ++i) add(Q(i, b), L((c + 1) * Lc, b), L(i, b));
        break;
    }
  }
  ListRef ref = upload_list(v, g.hlist_mem);
  if (ref.dev || v.empty()) g.hlists[key] = ref;
  return ref;
}

static int scan_gemm(LargeGroup& g, int op, int idx, int Lc, int C, cudaStream_t st) {
  ListRef l = scan_list(g, op, idx, Lc, C);
  if (!l.n) return SQOC_OK;
  const GemmArgs one{1.0, 0.0, 0.0, 0.0};
  gemm_begin(g, l, st);
  cudaError_t e = (op == H_LP1) ? launch_gemm<OP_C, OP_N, EPI_STORE>(l.dev, l.maps, l.tref, g.pt_counter, l.n, l.tiles, one, st, l.pt_tiles)
                                : launch_gemm<OP_N, OP_N, EPI_STORE>(l.dev, l.maps, l.tref, g.pt_counter, l.n, l.tiles, one, st, l.pt_tiles);
  gemm_end(g, st);
  if (e != cudaSuccess) {
    g.err = std::string("zgemm launch: ") + cudaGetErrorString(e);
    return SQOC_ERR_CUDA;
  }
  g.launches++;
  return SQOC_OK;
}

static int history_scans(LargeGroup& g, bool do_x, bool do_l, cudaStream_t st) {
  const int N = g.N;
  const int Lc = std::max(1, (int)std::ceil(std::sqrt((double)N)));
  const int C = (N + Lc - 1) / Lc;
  int rc;
  if (do_x) {
    for (int t = 0; t < Lc; ++t)
      if ((rc = scan_gemm(g, H_XP1, t, Lc, C, st))) return rc;
    for (int c = 2; c < C; ++c)
      if ((rc = scan_gemm(g, H_XP2, c, Lc, C, st))) return rc;
    if ((rc = scan_gemm(g, H_XP3, 0, Lc, C, st))) return rc;
  }
  if (do_l) {
    for (int t = 0; t < Lc; ++t)
      if ((rc = scan_gemm(g, H_LP1, t, Lc, C, st))) return rc;
    for (int c = C - 2; c >= 0; --c)
      if ((rc = scan_gemm(g, H_LP2, c, Lc, C, st))) return rc;
    if ((rc = scan_gemm(g, H_LP3, 0, Lc, C, st))) return rc;
  }
  return SQOC_OK;
}

static int large_eval_history(LargeGroup& g, const LargeArgs& a, int s_idx, const double* u, int sq,
                              cudaStream_t st) {
  const int K = g.K, N = g.N, nblk = g.nblk;
  const PolyScheme& sc = scheme_of(g.h_deg);
  int maxd = 0;
  for (auto& b : g.blocks) maxd = std::max(maxd, b.d);
  const unsigned ew_x = (unsigned)std::max<size_t>(1, std::min<size_t>(((size_t)maxd * maxd + 255) / 256, 64));
  const dim3 grid_all(ew_x, nblk, N);
  const double scale = std::ldexp(1.0, -sq);
  const size_t stride = g.total;
  GemmArgs one{1.0, 0.0, 0.0, 0.0};
  int rc;
  // ---- forward: all propagators, every intermediate kept ----
  build_a_kernel<<<grid_all, 256, 0, st>>>(0, K, N, u, g.d_dev, g.off_dev, g.gen_dev, scale, g.h_chain, stride);
  LCHK(cudaGetLastError());
  g.launches++;
  for (int k = 0; k < sc.nsteps; ++k)
    if ((rc = hgemm(g, H_STEP, k, 0, 0, N, step_args(sc.step[k]), st))) return rc;
  for (int i = 1; i <= sq; ++i)
    if ((rc = hgemm(g, H_S, i, 0, 0, N, one, st))) return rc;
  // ---- forward / backward recurrences (sequential over slices, batched over blocks) ----
  const dim3 ew_grid(ew_x, nblk);
  if ((rc = bc_init(g, g.h_X, g.h_L + (size_t)N * g.totalr, ew_grid, st))) return rc;
  const bool chunked = g.gate && N >= 64 && g.h_I != nullptr;  // chunked scans (gate: d x d recurrences)
  if (chunked) {
    if ((rc = history_scans(g, true, false, st))) return rc;
  } else {
    for (int i = 0; i < N; ++i)
      if ((rc = hgemm(g, H_X, 0, 0, i, i + 1, one, st))) return rc;
  }
  if ((rc = bc_tau(g, g.h_X + (size_t)N * g.totalr, a, s_idx, st))) return rc;
  if (chunked) {
    if ((rc = history_scans(g, false, true, st))) return rc;
  } else {
    for (int i = N - 1; i >= 0; --i)
      if ((rc = hgemm(g, H_L, 0, 0, i, i + 1, one, st))) return rc;
  }
  // ---- Frechet derivatives of every slice: L_R(A_i, X_i Lam_{i+1}^dag), derivative-only chain ----
  if ((rc = hgemm(g, H_B, 0, 0, 0, N, GemmArgs{scale, 0.0, 0.0, 0.0}, st))) return rc;
  for (int k = 0; k < sc.nsteps; ++k)
    if ((rc = hgemm(g, H_DSTEP, k, 0, 0, N, step_args(sc.step[k]), st))) return rc;
  int p = 0;
  for (int i = 1; i <= sq; ++i) {
    if ((rc = hgemm(g, H_DS, i, p, 0, N, one, st))) return rc;
    p ^= 1;
  }
  slice_trace_kernel<<<dim3(nblk, N), 256, 0, st>>>(K, g.d_dev, g.off_dev, g.gent_dev, g.h_dH[p], stride, g.h_g, nblk);
  LCHK(cudaGetLastError());
  hist_grad_kernel<<<256, 256, 0, st>>>(K, N, nblk, g.h_g, g.tau_dev, g.w_dev, g.gidx_dev,
                                        a.gradb + (size_t)s_idx * K * N, a.gradb_block_stride);
  LCHK(cudaGetLastError());
  g.launches += 2;
  return SQOC_OK;
}

// ------------------------------------------------------------------ state-vector schedule
enum SOp { SV_STEP, SV_S, SV_PSI, SV_CHI, SV_W };
constexpr int kSvSlots = kSlots + 1;  // scheme slots + squaring partner

static size_t sv_fixed_bytes(const LargeGroup& g) {
  const size_t N = g.N, K = g.K;
  return sizeof(double2) * (N * g.total + 2 * (N + 1) * g.totalr + (K + 1) * N * g.totalr * (K + 2) +
                            K * N * g.totalr + N * g.nblk * K);
}

static int sv_alloc(LargeGroup& g, bool with_u) {
  const size_t N = g.N, K = g.K;
  if (!g.sv_psi) {  // vector histories + augmented-action buffers (shared by modes 2 and 3)
    LCHK(cudaMalloc(&g.sv_psi, (N + 1) * g.totalr * sizeof(double2)));
    LCHK(cudaMalloc(&g.sv_chi, (N + 1) * g.totalr * sizeof(double2)));
    LCHK(cudaMalloc(&g.sv_V, (K + 1) * N * g.totalr * sizeof(double2)));
    LCHK(cudaMalloc(&g.sv_W, (K + 1) * (K + 1) * N * g.totalr * sizeof(double2)));
    LCHK(cudaMalloc(&g.sv_acc, K * N * g.totalr * sizeof(double2)));
    LCHK(cudaMalloc(&g.sv_g, N * g.nblk * K * sizeof(double2)));
    LCHK(cudaMalloc(&g.mf_t, 3 * g.totalr * sizeof(double2)));
  }
  if (!with_u || g.sv_U) return SQOC_OK;
  LCHK(cudaMalloc(&g.sv_U, N * g.total * sizeof(double2)));
  size_t free_b = 0, total_b = 0;
  LCHK(cudaMemGetInfo(&free_b, &total_b));
  const size_t per_slice = kSvSlots * g.total * sizeof(double2);
  g.sv_S = (int)std::max<size_t>(1, std::min<size_t>(N, (size_t)(0.5 * (double)free_b) / per_slice));
  g.sv_S = std::min(g.sv_S, 64);
  LCHK(cudaMalloc(&g.sv_chunk, (size_t)g.sv_S * per_slice));
  return SQOC_OK;
}

static ListRef sv_list(LargeGroup& g, int op, int idx, int p, int i0, int i1) {
  auto key = std::make_tuple(2000000000 + op * 1000000 + idx * 4 + p, g.last_degree * 100 + g.last_s, i0, i1);
  auto it = g.hlists.find(key);
  if (it != g.hlists.end()) return it->second;
  std::vector<GemmItem> v;
  const size_t S = g.sv_S, sl = g.total;
  auto cb = [&](int c, int z, int b) { return g.sv_chunk + ((size_t)c * S + z) * sl + g.off[b]; };
  if (op == SV_W) {
    for (int b = 0; b < g.nblk; ++b) {
      const int d = g.blocks[b].d;
      const size_t rows = (size_t)(g.K + 1) * g.N;
      const double2* Vb = g.sv_V + rows * g.offr[b];
      double2* Wb = g.sv_W + (size_t)idx * rows * g.totalr + rows * g.offr[b];
      const double2* Bt = static_cast<const double2*>(g.gentall_mem[b]);
      v.push_back(mk(Vb, Bt + (size_t)idx * d * d, 0, 0, Wb, 0, 0, (int)rows, d, d, 1, d, d, d, 0));
    }
  } else {
    const PolyScheme& sc = scheme_of(g.last_degree);
    for (int z = i0; z < i1; ++z)
      for (int b = 0; b < g.nblk; ++b) {
        const int d = g.blocks[b].d;
        double2 *Tp = cb(kSlotY + p, z, b), *Tn = cb(kSlotY + 1 - p, z, b);
        double2* U = g.sv_U + (size_t)z * sl + g.off[b];
        double2* Pi = g.sv_psi + (size_t)z * g.totalr + g.offr[b];
        double2* Pn = g.sv_psi + (size_t)(z + 1) * g.totalr + g.offr[b];
        double2* Ci = g.sv_chi + (size_t)z * g.totalr + g.offr[b];
        double2* Cn = g.sv_chi + (size_t)(z + 1) * g.totalr + g.offr[b];
        auto slot = [&](int c) { return cb(c, z, b); };
        switch (op) {
          case SV_STEP: push_step(v, sc, idx, d, slot, slot, true, false); break;
          case SV_S: v.push_back(mk(Tp, Tp, 0, 0, Tn, 0, 0, d, d, d, 1, d, d, d, 0)); break;
          case SV_PSI: v.push_back(mk(U, Pi, 0, 0, Pn, 0, 0, d, 1, d, 1, d, 1, 1, 0)); break;
          case SV_CHI: v.push_back(mk(U, Cn, 0, 0, Ci, 0, 0, d, 1, d, 1, d, 1, 1, 0)); break;
        }
      }
  }
  ListRef ref = upload_list(v, g.hlist_mem);
  if (ref.dev) g.hlists[key] = ref;
  return ref;
}

static int svgemm(LargeGroup& g, int op, int idx, int p, int i0, int i1, GemmArgs a, cudaStream_t st) {
  ListRef l = sv_list(g, op, idx, p, i0, i1);
  if (!l.dev) {
    g.err = "state-vector work list allocation failed";
    return SQOC_ERR_CUDA;
  }
  gemm_begin(g, l, st);
  cudaError_t e = (op == SV_CHI) ? launch_gemm<OP_C, OP_N, EPI_STORE>(l.dev, l.maps, l.tref, g.pt_counter, l.n, l.tiles, a, st, l.pt_tiles)
                                 : launch_gemm<OP_N, OP_N, EPI_STORE>(l.dev, l.maps, l.tref, g.pt_counter, l.n, l.tiles, a, st, l.pt_tiles);
  gemm_end(g, st);
  if (e != cudaSuccess) {
    g.err = std::string("zgemm launch: ") + cudaGetErrorString(e);
    return SQOC_ERR_CUDA;
  }
  g.launches++;
  return SQOC_OK;
}

// Number of Taylor terms m with beta^(m+1)/(m+1)! / (1 - beta/(m+2)) <= 1e-17.
static int taylor_terms(double beta) {
  double term = 1.0;
  for (int m = 1; m < 200; ++m) {
    term *= beta / m;  // beta^m / m!
    const double next = term * beta / (m + 1);
    if (beta < m + 2 && next / (1.0 - beta / (m + 2)) <= 1e-17) return m;
  }
  return 200;
}

static int sv_gradient(LargeGroup& g, const LargeArgs& a, int s_idx, const double* u, double bound, cudaStream_t st);

static unsigned sv_ew_x(const LargeGroup& g) {
  int maxd = 0;
  for (auto& b : g.blocks) maxd = std::max(maxd, b.d);
  return (unsigned)std::max<size_t>(1, std::min<size_t>(((size_t)maxd * maxd + 255) / 256, 256));
}

// propagators U_i of every slice, S slices per launch, kept in sv_U for both vector sweeps
static int sv_propagators(LargeGroup& g, const double* u, int sq, cudaStream_t st) {
  const int K = g.K, N = g.N, nblk = g.nblk;
  const PolyScheme& sc = scheme_of(g.last_degree);
  const unsigned ew_x = sv_ew_x(g);
  const double scale = std::ldexp(1.0, -sq);
  const size_t S = g.sv_S, sl = g.total;
  GemmArgs one{1.0, 0.0, 0.0, 0.0};
  int rc;
  for (int i0 = 0; i0 < N; i0 += (int)S) {
    const int n_here = std::min<int>((int)S, N - i0);
    const dim3 grid(ew_x, nblk, n_here);
    build_a_kernel<<<grid, 256, 0, st>>>(i0, K, N, u, g.d_dev, g.off_dev, g.gen_dev, scale, g.sv_chunk, sl);
    LCHK(cudaGetLastError());
    g.launches++;
    for (int k = 0; k < sc.nsteps; ++k)
      if ((rc = svgemm(g, SV_STEP, k, 0, 0, n_here, step_args(sc.step[k]), st))) return rc;
    int p = 0;
    for (int i = 0; i < sq; ++i) {
      if ((rc = svgemm(g, SV_S, 0, p, 0, n_here, one, st))) return rc;
      p ^= 1;
    }
    LCHK(cudaMemcpyAsync(g.sv_U + (size_t)i0 * sl, g.sv_chunk + (size_t)(kSlotY + p) * S * sl,
                         (size_t)n_here * sl * sizeof(double2), cudaMemcpyDeviceToDevice, st));
  }
  return SQOC_OK;
}

// psi / chi sweeps over the U_i in sv_U (sequential over slices, batched over blocks) + gradient
static int sv_sweeps(LargeGroup& g, const LargeArgs& a, int s_idx, const double* u, double bound, cudaStream_t st) {
  const int N = g.N;
  GemmArgs one{1.0, 0.0, 0.0, 0.0};
  int rc;
  const dim3 ew_grid(sv_ew_x(g), g.nblk);
  if ((rc = bc_init(g, g.sv_psi, g.sv_chi + (size_t)N * g.totalr, ew_grid, st))) return rc;
  for (int i = 0; i < N; ++i)
    if ((rc = svgemm(g, SV_PSI, 0, 0, i, i + 1, one, st))) return rc;
  if ((rc = bc_tau(g, g.sv_psi + (size_t)N * g.totalr, a, s_idx, st))) return rc;
  for (int i = N - 1; i >= 0; --i)
    if ((rc = svgemm(g, SV_CHI, 0, 0, i, i + 1, one, st))) return rc;
  return sv_gradient(g, a, s_idx, u, bound, st);
}

// dtau/du_k,i = <chi_{i+1}| L(A_i, a_k) |psi_i> for every slice by the augmented Taylor action
// exp([[A, a_k],[0, A]]) [0; psi] (top block = L(A, a_k) psi), batched over slices as GEMMs
// W_k = V a_k^T; needs the psi / chi histories in sv_psi / sv_chi.
static int sv_gradient(LargeGroup& g, const LargeArgs& a, int s_idx, const double* u, double bound, cudaStream_t st) {
  const int K = g.K, N = g.N, nblk = g.nblk;
  int maxd = 0;
  for (auto& b : g.blocks) maxd = std::max(maxd, b.d);
  int rc;
  GemmArgs one{1.0, 0.0, 0.0, 0.0};
  double emax = 0.0;
  for (auto& b : g.blocks)
    for (int k = 1; k <= K; ++k) emax = std::max(emax, b.gen_norm[k]);
  const int m = taylor_terms(bound + emax);
  g.last_taylor_terms = m;
  const dim3 vgrid((unsigned)std::min<size_t>(((size_t)N * maxd + 255) / 256, 4096), nblk);
  sv_init_kernel<<<vgrid, 256, 0, st>>>(K, N, g.d_dev, g.offr_dev, g.totalr, g.sv_psi, g.sv_V, g.sv_acc);
  LCHK(cudaGetLastError());
  g.launches++;
  const size_t wstride = (size_t)(K + 1) * N * g.totalr;
  for (int l = 1; l <= m; ++l) {
    for (int k = 0; k <= K; ++k)
      if ((rc = svgemm(g, SV_W, k, 0, 0, 0, one, st))) return rc;
    sv_combine_kernel<<<vgrid, 256, 0, st>>>(l, K, N, u, g.d_dev, g.offr_dev, g.sv_V, g.sv_W, wstride, g.sv_acc);
    LCHK(cudaGetLastError());
    g.launches++;
  }
  sv_dot_kernel<<<dim3(nblk, N), 256, 0, st>>>(K, N, nblk, g.d_dev, g.offr_dev, g.totalr, g.sv_chi, g.sv_acc, g.sv_g);
  LCHK(cudaGetLastError());
  hist_grad_kernel<<<256, 256, 0, st>>>(K, N, nblk, g.sv_g, g.tau_dev, g.w_dev, g.gidx_dev,
                                        a.gradb + (size_t)s_idx * K * N, a.gradb_block_stride);
  LCHK(cudaGetLastError());
  g.launches += 2;
  return SQOC_OK;
}

// ------------------------------------------------------------------ matrix-free state schedule
// y = sgn A t for every block (one warp per row, coalesced rows of the dense A); t_out = y * scale;
// acc += t_out.  HBM-bound: one read of A per Taylor term.
__global__ void mv_taylor_kernel(int nblk, const int* __restrict__ dims, const size_t* __restrict__ off,
                                 const size_t* __restrict__ offr, const double2* __restrict__ A,
                                 const double2* __restrict__ tin, double2* __restrict__ tout,
                                 double2* __restrict__ acc, double scale) {
  const int warps = blockDim.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.y;
  const int d = dims[b];
  const double2* Ab = A + off[b];
  const double2* t = tin + offr[b];
  for (int row = blockIdx.x * warps + (threadIdx.x >> 5); row < d; row += gridDim.x * warps) {
    const double2* ar = Ab + (size_t)row * d;
    double sx = 0.0, sy = 0.0;
    for (int c = lane; c < d; c += 32) {
      const double2 x = __ldg(ar + c), v = __ldg(t + c);
      sx = fma(x.x, v.x, sx);
      sx = fma(-x.y, v.y, sx);
      sy = fma(x.x, v.y, sy);
      sy = fma(x.y, v.x, sy);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sx += __shfl_xor_sync(0xffffffffu, sx, o);
      sy += __shfl_xor_sync(0xffffffffu, sy, o);
    }
    if (lane == 0) {
      const double2 y = make_double2(sx * scale, sy * scale);
      tout[offr[b] + row] = y;
      double2 z = acc[offr[b] + row];
      acc[offr[b] + row] = make_double2(z.x + y.x, z.y + y.y);
    }
  }
}

__global__ void vcopy_kernel(size_t n, const double2* __restrict__ a, double2* __restrict__ b, double2* __restrict__ c) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    b[i] = a[i];
    if (c) c[i] = a[i];
  }
}

// exp(sgn A) applied to `in` -> `out` by sigma substeps of a degree-m Taylor action (A in g.A)
static int mf_action(LargeGroup& g, double sgn, int m, int sigma, const double2* in, double2* out, cudaStream_t st) {
  int maxd = 0;
  for (auto& b : g.blocks) maxd = std::max(maxd, b.d);
  double2 *t0 = g.mf_t, *t1 = g.mf_t + g.totalr;
  const unsigned vg = (unsigned)std::min<size_t>((g.totalr + 255) / 256, 1024);
  vcopy_kernel<<<vg, 256, 0, st>>>(g.totalr, in, out, t0);  // acc = t = in
  LCHK(cudaGetLastError());
  g.launches++;
  const dim3 grid((unsigned)std::max(1, std::min((maxd + 7) / 8, 1184)), g.nblk);
  for (int sub = 0; sub < sigma; ++sub) {
    if (sub > 0) {
      vcopy_kernel<<<vg, 256, 0, st>>>(g.totalr, out, t0, nullptr);
      LCHK(cudaGetLastError());
      g.launches++;
    }
    for (int l = 1; l <= m; ++l) {
      mv_taylor_kernel<<<grid, 256, 0, st>>>(g.nblk, g.d_dev, g.off_dev, g.offr_dev, g.A, t0, t1, out,
                                             sgn / (sigma * (double)l));
      LCHK(cudaGetLastError());
      g.launches++;
      std::swap(t0, t1);
    }
  }
  return SQOC_OK;
}

static int large_eval_matrix_free(LargeGroup& g, const LargeArgs& a, int s_idx, const double* u, double bound,
                                  cudaStream_t st) {
  const int K = g.K, N = g.N, nblk = g.nblk;
  int maxd = 0;
  for (auto& b : g.blocks) maxd = std::max(maxd, b.d);
  const dim3 ew_grid((unsigned)std::min<size_t>(((size_t)maxd * maxd + 255) / 256, 4096), nblk);
  int sigma = std::max(1, (int)std::ceil(bound / 3.0));
  const int m = taylor_terms(bound / sigma);
  g.last_taylor_terms = m;
  int rc;
  if ((rc = bc_init(g, g.sv_psi, g.sv_chi + (size_t)N * g.totalr, dim3(ew_grid.x, nblk), st))) return rc;
  for (int j = 0; j < N; ++j) {  // psi_{j+1} = exp(A_j) psi_j
    build_a_kernel<<<ew_grid, 256, 0, st>>>(j, K, N, u, g.d_dev, g.off_dev, g.gen_dev, 1.0, g.A, 0);
    LCHK(cudaGetLastError());
    g.launches++;
    if ((rc = mf_action(g, 1.0, m, sigma, g.sv_psi + (size_t)j * g.totalr, g.sv_psi + (size_t)(j + 1) * g.totalr, st)))
      return rc;
  }
  if ((rc = bc_tau(g, g.sv_psi + (size_t)N * g.totalr, a, s_idx, st))) return rc;
  for (int j = N - 1; j >= 0; --j) {  // chi_j = exp(A_j)^dag chi_{j+1} = exp(-A_j) chi_{j+1} (A anti-Hermitian)
    build_a_kernel<<<ew_grid, 256, 0, st>>>(j, K, N, u, g.d_dev, g.off_dev, g.gen_dev, 1.0, g.A, 0);
    LCHK(cudaGetLastError());
    g.launches++;
    if ((rc = mf_action(g, -1.0, m, sigma, g.sv_chi + (size_t)(j + 1) * g.totalr, g.sv_chi + (size_t)j * g.totalr, st)))
      return rc;
  }
  return sv_gradient(g, a, s_idx, u, bound, st);
}


// ------------------------------------------------------------------ slice-sequential schedule
// Propagator history for the sequential sweeps: allocated on first use when N sum d^2 complex values fit
// in 90% of the free device memory (cfg 3 on one B200: 500 x 285 MB = 142.5 GB of ~170 GB free).  The
// backward sweep then reads U_j instead of forming it (one GEMM-unit per slice fewer).
static bool uh_ensure(LargeGroup& g) {
  const char* env = getenv("SQOC_UHIST");
  if ((env && env[0] == '0') || g.N <= 0) return false;
  if (g.uh) return true;
  const size_t bytes = (size_t)g.N * g.total * sizeof(double2);
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) return false;
  if (bytes > (size_t)(0.9 * (double)free_b)) return false;
  if (cudaMalloc(&g.uh, bytes) != cudaSuccess) {
    cudaGetLastError();  // clear the failed allocation; run without the history
    g.uh = nullptr;
    return false;
  }
  return true;
}

// forward sweep from the boundary X_0 (I / psi_0 / a chunk's X_start); returns the parity q of X_N
static int seq_forward(LargeGroup& g, const double* u, const PolyScheme& sc, int sq, dim3 ew_grid, cudaStream_t st,
                       int* q_out, bool keep_u = false) {
  const int K = g.K, N = g.N;
  const double scale = std::ldexp(1.0, -sq);
  int rc;
  if (!g.dry && (rc = bc_init(g, g.X[0], g.L[0], ew_grid, st))) return rc;
  int q = 0;
  GemmArgs one{1.0, 0.0, 0.0, 0.0};
  for (int j = 0; j < N; ++j) {
    if (!g.dry) {
      build_a_kernel<<<ew_grid, 256, 0, st>>>(j, K, N, u, g.d_dev, g.off_dev, g.gen_dev, scale, g.A, 0);
      LCHK(cudaGetLastError());
      g.launches++;
    }
    if (g.sp_on && (rc = sp_values(g, j, u, scale, st))) return rc;
    for (int k = 0; k < sc.nsteps; ++k) {
      if (g.sp_on && k < 2) rc = sp_fwd_step(g, k, sc.degree, step_args(sc.step[k]), st);
      else rc = gemm(g, F_STEP, k, sc.degree, 0, step_args(sc.step[k]), st);
      if (rc) return rc;
    }
    int p = 0;
    for (int i = 0; i < sq; ++i) {
      if ((rc = gemm(g, F_S, p, 0, 0, one, st))) return rc;
      p ^= 1;
    }
    if (keep_u && !g.dry)
      LCHK(cudaMemcpyAsync(g.uh + (size_t)j * g.total, g.T[p], g.total * sizeof(double2), cudaMemcpyDeviceToDevice,
                           st));
    if ((rc = gemm(g, F_X, p, q, 0, one, st))) return rc;
    q ^= 1;
  }
  if (!g.dry) g.uh_valid = keep_u;
  *q_out = q;
  return SQOC_OK;
}

// backward sweep from X_N (X[q]) and Lam_N (L[0]); tau must already be set
static int seq_backward(LargeGroup& g, const LargeArgs& a, int s_idx, const double* u, const PolyScheme& sc, int sq,
                        int q, dim3 ew_grid, cudaStream_t st, bool have_u = false) {
  const int K = g.K, N = g.N, nblk = g.nblk;
  const double scale = std::ldexp(1.0, -sq);
  GemmArgs one{1.0, 0.0, 0.0, 0.0};
  int rc, r = 0;
  if (g.gate) {  // one carry: Ad = 2^-s C_N, C_N = X_N Lam_N^dag
    if ((rc = gemm(g, B_C, 0, q, 0, GemmArgs{scale, 0.0, 0.0, 0.0}, st))) return rc;
  }
  for (int j = N - 1; j >= 0; --j) {
    if (!g.dry) {
      build_a_kernel<<<ew_grid, 256, 0, st>>>(j, K, N, u, g.d_dev, g.off_dev, g.gen_dev, scale, g.A, 0);
      LCHK(cudaGetLastError());
      g.launches++;
    }
    if (!g.gate && (rc = gemm(g, B_C, 0, q, r, GemmArgs{scale, 0.0, 0.0, 0.0}, st))) return rc;
    if (g.sp_on && (rc = sp_values(g, j, u, scale, st))) return rc;
    for (int k = 0; k < sc.nsteps; ++k) {
      if (g.sp_on && k == 0) {
        rc = sp_pair_step(g, 0, sc.degree, step_args(sc.step[0]), st);
      } else if (g.sp_on && k == 1) {
        rc = sp_chain() ? SQOC_OK : gemm(g, B_STEP1D, 0, sc.degree, 0, one, st);
        if (rc == SQOC_OK) rc = sp_pair_step(g, 1, sc.degree, step_args(sc.step[1]), st);
      } else if (have_u && sq == 0 && k == sc.nsteps - 1) {  // U_j = Y from the forward's history
        rc = gemm(g, B_STEPD, k, sc.degree, 0, step_args(sc.step[k]), st);
      } else {
        rc = gemm(g, B_STEP, k, sc.degree, 0, step_args(sc.step[k]), st);
      }
      if (rc) return rc;
    }
    int p = 0;
    for (int i = 0; i < sq; ++i) {
      if ((rc = gemm(g, have_u && i == sq - 1 ? B_SD : B_S, p, 0, 0, one, st))) return rc;
      p ^= 1;
    }
    if (have_u && !g.dry)  // U_j into the slot the value product would have written (Y = T[0] at s = 0, else T[p])
      LCHK(cudaMemcpyAsync(g.T[p], g.uh + (size_t)j * g.total, g.total * sizeof(double2), cudaMemcpyDeviceToDevice,
                           st));
    if (g.gate && g.sp_on) {  // M = U^dag Ad on the tensor cores, the trace on the sparse a_k
      if ((rc = gemm(g, B_M, p, 0, 0, one, st))) return rc;
      if ((rc = sp_trace(g, j, p, a, s_idx, st))) return rc;
    } else {
      if ((rc = gemm(g, g.gate ? B_UC : B_D, p, 0, 0, one, st))) return rc;
      if (!g.dry) {
        trace_reduce_kernel<<<nblk, 256, 0, st>>>(j, K, N, g.tile_off_dev, g.trace_part, g.tau_dev, g.w_dev,
                                                  g.gidx_dev, a.gradb + (size_t)s_idx * K * N, a.gradb_block_stride);
        LCHK(cudaGetLastError());
        g.launches++;
      }
    }
    if (g.gate) {  // C_{j-1} = U^dag C_j U
      if (j > 0 && (rc = gemm(g, B_CU, p, 0, 0, one, st))) return rc;
    } else {
      if ((rc = gemm(g, B_XL, p, q, r, one, st))) return rc;
      q ^= 1;
      r ^= 1;
    }
  }
  return SQOC_OK;
}

// ------------------------------------------------------------------ slice-chunk sharding
__global__ void eye_kernel(const int* __restrict__ dims, const size_t* __restrict__ off, double2* __restrict__ out) {
  const int b = blockIdx.y;
  const int d = dims[b];
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < (size_t)d * d; i += (size_t)gridDim.x * blockDim.x)
    out[off[b] + i] = make_double2((i / d == i % d) ? 1.0 : 0.0, 0.0);
}

// One launch per carry step, each batched over the blocks; all lists uploaded in one stream-ordered
// allocation (freed in stream order after the last launch).
struct CarryStep {
  int ta;          // OP_N or OP_C on the chunk product
  size_t first, n; // items
};

static int run_carry_steps(LargeGroup& g, std::vector<GemmItem>& items, const std::vector<CarryStep>& steps,
                           cudaStream_t st) {
  if (items.empty()) return SQOC_OK;
  for (auto& s : steps) {  // tile offsets restart per launch
    int t = 0;
    for (size_t i = s.first; i < s.first + s.n; ++i) {
      items[i].tile_start = t;
      t += tiles_of(items[i].m, items[i].n);
    }
  }
  GemmItem* dev = nullptr;
  ItemMaps* maps = nullptr;
  LCHK(cudaMallocAsync(reinterpret_cast<void**>(&dev), items.size() * sizeof(GemmItem), st));
  LCHK(cudaMemcpyAsync(dev, items.data(), items.size() * sizeof(GemmItem), cudaMemcpyHostToDevice, st));
  std::vector<ItemMaps> hmaps;
  TileRef* trefs = nullptr;
  std::vector<std::vector<TileRef>> step_tiles(steps.size());
  size_t ntref = 0;
  for (size_t q = 0; q < steps.size(); ++q) {  // tile lists per launch (items relative to the launch's first)
    std::vector<GemmItem> sub(items.begin() + steps[q].first, items.begin() + steps[q].first + steps[q].n);
    build_tiles(sub, step_tiles[q]);
    ntref += step_tiles[q].size();
  }
  if (build_maps(items, hmaps)) {
    LCHK(cudaMallocAsync(reinterpret_cast<void**>(&maps), hmaps.size() * sizeof(ItemMaps), st));
    LCHK(cudaMemcpyAsync(maps, hmaps.data(), hmaps.size() * sizeof(ItemMaps), cudaMemcpyHostToDevice, st));
    std::vector<TileRef> flat;
    for (auto& t : step_tiles) flat.insert(flat.end(), t.begin(), t.end());
    LCHK(cudaMallocAsync(reinterpret_cast<void**>(&trefs), ntref * sizeof(TileRef), st));
    LCHK(cudaMemcpyAsync(trefs, flat.data(), ntref * sizeof(TileRef), cudaMemcpyHostToDevice, st));
  }
  size_t tref_off = 0;
  GemmArgs one{1.0, 0.0, 0.0, 0.0};
  for (auto& s : steps) {
    int tiles = 0;
    ListRef l;
    for (size_t i = s.first; i < s.first + s.n; ++i) {
      tiles += tiles_of(items[i].m, items[i].n);
      l.macs += (double)items[i].m * items[i].n * items[i].k;
    }
    gemm_begin(g, l, st);
    const ItemMaps* mp = maps ? maps + s.first : nullptr;
    const TileRef* tp = trefs ? trefs + tref_off : nullptr;
    tref_off += (size_t)tiles;
    cudaError_t e = s.ta == OP_C
                        ? launch_gemm<OP_C, OP_N, EPI_STORE>(dev + s.first, mp, tp, g.pt_counter, (int)s.n, tiles, one, st)
                        : launch_gemm<OP_N, OP_N, EPI_STORE>(dev + s.first, mp, tp, g.pt_counter, (int)s.n, tiles, one, st);
    gemm_end(g, st);
    if (e != cudaSuccess) {
      cudaFreeAsync(dev, st);
      if (maps) cudaFreeAsync(maps, st);
      if (trefs) cudaFreeAsync(trefs, st);
      g.err = std::string("carry zgemm launch: ") + cudaGetErrorString(e);
      return SQOC_ERR_CUDA;
    }
    g.launches++;
    g.carry_gemms++;
  }
  LCHK(cudaFreeAsync(dev, st));
  if (maps) LCHK(cudaFreeAsync(maps, st));
  if (trefs) LCHK(cudaFreeAsync(trefs, st));
  return SQOC_OK;
}

// Boundary values of chunk c from the gathered products (chunk_in).  Gate: X_end -> X[0],
// Lam_end -> L[0]; state: psi_start / chi_end in chunk_vec; tau of every block -> chunk_tau.
static int chunk_carries(LargeGroup& g, cudaStream_t st) {
  const int P = g.chunk_P, c = g.chunk_c, nb = g.nblk;
  const size_t tot = g.total;
  auto Cp = [&](int i, int b) { return g.chunk_in + (size_t)i * tot + g.off[b]; };
  std::vector<GemmItem> items;
  std::vector<CarryStep> steps;
  std::vector<const double2*> xs(nb), ls(nb);
  if (!g.chunk_vec) {
    LCHK(cudaMalloc(&g.chunk_vec, 5 * g.totalr * sizeof(double2)));
    LCHK(cudaMalloc(&g.chunk_tau, nb * sizeof(double2)));
    LCHK(cudaMalloc(reinterpret_cast<void**>(&g.chunk_ptrs), 2 * nb * sizeof(double2*)));
  }
  auto add_step = [&](int ta, auto item_of) {
    CarryStep s{ta, items.size(), (size_t)nb};
    for (int b = 0; b < nb; ++b) items.push_back(item_of(b, g.blocks[b].d));
    steps.push_back(s);
  };
  const double2* X_tau = nullptr;  // the matrix / vector tau is read against Lam_end / chi_end
  if (g.gate) {
    // left: M_1 = C_1 C_0, M_i = C_i M_{i-1}, X_end = M_c (T[0] / T[1] ping-pong, last into X[0])
    for (int i = 1; i <= c; ++i)
      add_step(OP_N, [&](int b, int d) {
        const double2* B = i == 1 ? Cp(0, b) : g.T[(i - 2) & 1] + g.off[b];
        double2* C = i == c ? g.X[0] + g.off[b] : g.T[(i - 1) & 1] + g.off[b];
        return mk(Cp(i, b), B, 0, 0, C, 0, 0, d, d, d, 1, d, d, d, 0);
      });
    if (c == 0) LCHK(cudaMemcpyAsync(g.X[0], Cp(0, 0), tot * sizeof(double2), cudaMemcpyDeviceToDevice, st));
    // right: R_1 = C_{P-1}^dag V, R_i = C_{P-i}^dag R_{i-1}, Lam_end = R_{P-1-c} (dT ping-pong, last into L[0])
    const int nr = P - 1 - c;
    for (int i = 1; i <= nr; ++i)
      add_step(OP_C, [&](int b, int d) {
        const double2* B = i == 1 ? g.blocks[b].target : g.dT[(i - 2) & 1] + g.off[b];
        double2* C = i == nr ? g.L[0] + g.off[b] : g.dT[(i - 1) & 1] + g.off[b];
        return mk(Cp(P - i, b), B, 0, 0, C, 0, 0, d, d, d, 1, d, d, d, 0);
      });
    if (nr == 0)
      for (int b = 0; b < nb; ++b)
        LCHK(cudaMemcpyAsync(g.L[0] + g.off[b], g.blocks[b].target, (size_t)g.blocks[b].d * g.blocks[b].d *
                             sizeof(double2), cudaMemcpyDeviceToDevice, st));
    for (int b = 0; b < nb; ++b) {
      xs[b] = g.X[0] + g.off[b];
      ls[b] = g.L[0] + g.off[b];
    }
    X_tau = g.X[0];
  } else {
    // vectors: chunk_vec slots 0/1 left ping-pong, 2/3 right ping-pong, 4 = C_c psi_start
    auto V = [&](int slot, int b) { return g.chunk_vec + (size_t)slot * g.totalr + g.offr[b]; };
    for (int i = 1; i <= c; ++i)  // v_i = C_{i-1} v_{i-1}, v_0 = psi_0
      add_step(OP_N, [&](int b, int d) {
        const double2* x = i == 1 ? g.blocks[b].x0 : V((i - 2) & 1, b);
        return mk(Cp(i - 1, b), x, 0, 0, V((i - 1) & 1, b), 0, 0, d, 1, d, 1, d, 1, 1, 0);
      });
    for (int b = 0; b < nb; ++b) xs[b] = c == 0 ? g.blocks[b].x0 : V((c - 1) & 1, b);
    add_step(OP_N, [&](int b, int d) { return mk(Cp(c, b), xs[b], 0, 0, V(4, b), 0, 0, d, 1, d, 1, d, 1, 1, 0); });
    const int nr = P - 1 - c;
    for (int i = 1; i <= nr; ++i)  // w_i = C_{P-i}^dag w_{i-1}, w_0 = psi_f
      add_step(OP_C, [&](int b, int d) {
        const double2* x = i == 1 ? g.blocks[b].target : V(2 + ((i - 2) & 1), b);
        return mk(Cp(P - i, b), x, 0, 0, V(2 + ((i - 1) & 1), b), 0, 0, d, 1, d, 1, d, 1, 1, 0);
      });
    for (int b = 0; b < nb; ++b) ls[b] = nr == 0 ? g.blocks[b].target : V(2 + ((nr - 1) & 1), b);
    X_tau = g.chunk_vec + 4 * g.totalr;
  }
  int rc = run_carry_steps(g, items, steps, st);
  if (rc) return rc;
  std::vector<const double2*> ptrs(xs);
  ptrs.insert(ptrs.end(), ls.begin(), ls.end());
  LCHK(cudaMemcpyAsync(g.chunk_ptrs, ptrs.data(), 2 * nb * sizeof(double2*), cudaMemcpyHostToDevice, st));
  // tau_b = <Lam_end, X_end> (gate, = Tr(V^dag X_N)) or <chi_end, C_c psi_start> (state, = <psi_f|X_N|psi_0>)
  tau_kernel<<<nb, 256, 0, st>>>(g.gate, 1, g.d_dev, g.offr_dev, X_tau, g.chunk_ptrs + nb, g.chunk_tau, g.chunk_tau,
                                 g.gidx_dev);
  LCHK(cudaGetLastError());  // (chunk problems hold large blocks only: global index == local index)
  g.launches++;
  return SQOC_OK;
}

static int chunk_eval(LargeGroup& g, const LargeArgs& a, int s_idx, const double* u, const PolyScheme& sc, int sq,
                      double bound, dim3 ew_grid, cudaStream_t st) {
  int rc;
  if (g.chunk_phase == 1) {
    if (g.gate) {  // forward sweep from X = I; X_N is the chunk product
      g.mode = 0;
      int q = 0;
      if ((rc = seq_forward(g, u, sc, sq, ew_grid, st, &q, uh_ensure(g)))) return rc;
      LCHK(cudaMemcpyAsync(g.chunk_out, g.X[q], g.total * sizeof(double2), cudaMemcpyDeviceToDevice, st));
    } else {  // every U_j kept (the sweeps of phase 2 reuse them); product by one GEMM per slice
      g.mode = 2;
      if ((rc = sv_alloc(g, true))) return rc;
      if ((rc = sv_propagators(g, u, sq, st))) return rc;
      const int N = g.N;
      if (N == 0) {
        eye_kernel<<<ew_grid, 256, 0, st>>>(g.d_dev, g.off_dev, g.chunk_out);
        LCHK(cudaGetLastError());
      } else if (N == 1) {
        LCHK(cudaMemcpyAsync(g.chunk_out, g.sv_U, g.total * sizeof(double2), cudaMemcpyDeviceToDevice, st));
      }
      std::vector<GemmItem> items;
      std::vector<CarryStep> steps;
      for (int i = 1; i < N; ++i) {  // M_i = U_i M_{i-1}, M_0 = U_0 (T ping-pong, last into chunk_out)
        CarryStep s{OP_N, items.size(), (size_t)g.nblk};
        for (int b = 0; b < g.nblk; ++b) {
          const int d = g.blocks[b].d;
          const double2* B = i == 1 ? g.sv_U + g.off[b] : g.T[(i - 2) & 1] + g.off[b];
          double2* C = i == N - 1 ? g.chunk_out + g.off[b] : g.T[(i - 1) & 1] + g.off[b];
          items.push_back(mk(g.sv_U + (size_t)i * g.total + g.off[b], B, 0, 0, C, 0, 0, d, d, d, 1, d, d, d, 0));
        }
        steps.push_back(s);
      }
      g.carry_gemms = 0;
      if ((rc = run_carry_steps(g, items, steps, st))) return rc;
    }
    g.chunk_fwd_valid = true;
    return SQOC_OK;
  }
  // ---- phase 2 ----
  if (!g.gate && !g.chunk_fwd_valid) {
    g.err = "sqoc_chunk_backward needs sqoc_chunk_forward on the same problem and controls first";
    return SQOC_ERR_ARG;
  }
  g.carry_gemms = 0;
  if (g.timing) {
    for (auto& e : g.carry_ev)
      if (!e) LCHK(cudaEventCreate(&e));
    LCHK(cudaEventRecord(g.carry_ev[0], st));
  }
  if ((rc = chunk_carries(g, st))) return rc;
  if (g.timing) LCHK(cudaEventRecord(g.carry_ev[1], st));
  g.bc_tau = g.chunk_tau;
  if (g.gate) {
    g.mode = 0;
    rc = bc_tau(g, nullptr, a, s_idx, st);  // tau_dev and tau_out from the carries
    if (rc == SQOC_OK) rc = seq_backward(g, a, s_idx, u, sc, sq, 0, ew_grid, st, g.uh && g.uh_valid);
  } else {
    g.mode = 2;
    g.bc_x_dev = g.chunk_ptrs;
    g.bc_l_dev = g.chunk_ptrs + g.nblk;
    rc = sv_sweeps(g, a, s_idx, u, bound, st);
  }
  g.bc_tau = nullptr;
  g.bc_x_dev = g.bc_l_dev = nullptr;
  return rc;
}

int large_carry_time(LargeGroup& g, double* ms) {
  *ms = 0.0;
  if (!g.carry_ev[0] || !g.carry_ev[1]) return SQOC_OK;
  float x = 0.f;
  if (cudaEventElapsedTime(&x, g.carry_ev[0], g.carry_ev[1]) == cudaSuccess) *ms = x;
  else (void)cudaGetLastError();
  return SQOC_OK;
}

// ------------------------------------------------------------------ evaluation
int large_eval(LargeGroup& g, const LargeArgs& a, cudaStream_t st) {
  // First evaluation of a group on the persistent TMA kernel: run it once and discard the result.  r02
  // measured (tools/repeat_check.py, tools/stale_check.py): the first evaluation of a fresh engine
  // deviates intermittently by 1e-14 .. 1e-8 relative in the gradient, every later evaluation -- same or
  // different controls -- is bit-identical to the steady-state value (0 deviations in ~200), and the
  // cp.async kernel never deviates.  Not explained yet (not the lazy list setup, not staged host copies,
  // not tensor-map visibility: each was removed without effect; a timing window that only cold page
  // tables / TLBs open is the remaining suspect), so the cold pass is spent before the result counts.
  // SQOC_GEMM_TMA=0 selects the cp.async kernel and skips this.
  if (!g.warmed) {
    g.warmed = true;
    static const bool off = [] { const char* e = getenv("SQOC_WARM"); return e && e[0] == '0'; }();
    if (!off && use_3m() && staging() == 1) {
      const int rc0 = large_eval(g, a, st);
      if (rc0) return rc0;
    }
  }
  const int N = g.N, K = g.K, nblk = g.nblk;
  int maxd = 0;
  for (auto& b : g.blocks) maxd = std::max(maxd, b.d);
  const dim3 ew_grid((unsigned)std::min<size_t>(((size_t)maxd * maxd + 255) / 256, 4096), nblk);
  g.launches = 0;
  g.tev_used = 0;
  g.gemm_macs = 0.0;
  g.gemm_launches = 0;
  for (int s = 0; s < a.batch; ++s) {
    const double* u = a.u + (size_t)s * K * N;
    // ---- plan (scheme, s) from the norm bound over all slices and blocks ----
    LCHK(cudaMemsetAsync(g.norm_dev, 0, sizeof(double), st));
    bound_kernel<<<std::max(1, std::min((N + 255) / 256, 148)), 256, 0, st>>>(
        u, K, N, nblk, g.gnorm_dev, reinterpret_cast<unsigned long long*>(g.norm_dev));
    LCHK(cudaGetLastError());
    double bound = 0.0;
    LCHK(cudaMemcpyAsync(&bound, g.norm_dev, sizeof(double), cudaMemcpyDeviceToHost, st));
    LCHK(cudaStreamSynchronize(st));
    g.launches++;
    int sq;
    const PolyScheme& sc = *choose_scheme(bound, sq);
    g.last_degree = sc.degree;
    g.last_s = sq;
    int rc;
    if (g.chunk_phase) {
      if ((rc = chunk_eval(g, a, s, u, sc, sq, bound, ew_grid, st))) return rc;
      continue;
    }
    if (g.uh && g.force_mode != -1 && g.force_mode != 0) {  // another schedule forced: release the history
      cudaFree(g.uh);
      g.uh = nullptr;
      g.uh_valid = false;
    }
    if (!g.gate && N > 0 && g.force_mode == 3) {  // matrix-free state schedule (opt-in)
      if ((rc = sv_alloc(g, false))) return rc;
      g.mode = 3;
      if ((rc = large_eval_matrix_free(g, a, s, u, bound, st))) return rc;
      continue;
    }
    if (!g.gate && N > 0 && g.force_mode != 0 && g.force_mode != 1) {  // state-vector schedule
      bool use_sv = g.force_mode == 2;
      if (!use_sv) {
        size_t free_b = 0, total_b = 0;
        LCHK(cudaMemGetInfo(&free_b, &total_b));
        const size_t have = g.sv_U ? sv_fixed_bytes(g) : 0;
        use_sv = sv_fixed_bytes(g) + 5 * g.total * sizeof(double2) <= (size_t)(0.7 * (double)(free_b + have));
      }
      if (use_sv) {
        if ((rc = sv_alloc(g, true))) return rc;
        g.mode = 2;
        g.chunk_fwd_valid = false;  // sv_U now holds this evaluation's propagators
        if ((rc = sv_propagators(g, u, sq, st))) return rc;
        if ((rc = sv_sweeps(g, a, s, u, bound, st))) return rc;
        continue;
      }
    }
    {  // history schedule when every slice's chain fits comfortably in free memory
      bool use_hist = g.force_mode == 1;
      if (g.force_mode == -1 && N > 0) {
        size_t free_b = 0, total_b = 0;
        LCHK(cudaMemGetInfo(&free_b, &total_b));
        const size_t have = g.h_C ? history_bytes(g, g.h_C) : 0;
        use_hist = history_bytes(g, kSlots + sq) <= (size_t)(0.6 * (double)(free_b + have));
      }
      if (use_hist && N > 0) {
        if ((rc = hist_alloc(g, sc.degree, sq))) return rc;
        g.mode = 1;
        if ((rc = large_eval_history(g, a, s, u, sq, st))) return rc;
        continue;
      }
      g.mode = 0;
    }
    int q = 0;
    const bool keep = uh_ensure(g);
    if (g.seq_ready_key != sc.degree * 100 + sq) {  // build every list of this plan before anything runs
      const int n_save = g.N;
      g.dry = true;
      g.N = std::min(n_save, 2);  // two slices reach both parities of the ping-pong buffers
      int qd = 0;
      rc = seq_forward(g, u, sc, sq, ew_grid, st, &qd, keep);
      for (int qq = 0; qq < 2 && rc == SQOC_OK; ++qq) rc = seq_backward(g, a, s, u, sc, sq, qq, ew_grid, st, keep);
      g.dry = false;
      g.N = n_save;
      if (rc) return rc;
      LCHK(cudaDeviceSynchronize());
      g.seq_ready_key = sc.degree * 100 + sq;
    }
    if ((rc = seq_forward(g, u, sc, sq, ew_grid, st, &q, keep))) return rc;
    if ((rc = bc_tau(g, g.X[q], a, s, st))) return rc;
    if ((rc = seq_backward(g, a, s, u, sc, sq, q, ew_grid, st, keep))) return rc;
  }
  return SQOC_OK;
}

}  // namespace sqoc
