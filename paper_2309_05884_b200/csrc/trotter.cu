// Trotterised per-qubit propagator and its fidelity replay on the GPU.
//
// Reference: /root/reference/pkg/src/symqoc/trotter.py
//   PerQubitPlan.apply_step  :68-152  for i = n..1: coupling phases exp(-i tau/n H_cpl) on the rows,
//                                     then the 2 x 2 factor exp(-i tau h_i) on site i (the reference
//                                     swaps site i to the last slot and broadcasts over 2^(n-1)
//                                     blocks); Strang: i = 1..n with tau/2 factors and half phases,
//                                     then the mirror sweep
//   expm_2x2                 :48-65   closed form
//   fidelity_replay          :196-225 W <- U_trotter (W U_exact^dag), F_j = |Tr W|^2 / 4^n; the exact
//                                     step by a Taylor series of the sparse H (:183-193)
// Model (model.py:59-92, per-qubit controls): H = sum_i bz/2 Z_i + sum_k c_k/4 sum_i Z_i Z_{i+k}
//   + sum_i (bx_i X_i + by_i Y_i)/2, site 1 = most significant bit.
//
// Kernels (all HBM/L2- or shared-memory-bound integer-indexed complex work; no tensor cores):
//   tr_factor_kernel  one thread per (step, site): the 2 x 2 factors of every step up front
//   tr_cols_kernel<N> one CTA per column pair, the 2^N-row column pair resident in shared memory
//                     (32 B per row: one sector), every layer of the Trotter step -- and, for
//                     sqoc_trotter_apply, every step -- applied on chip; fused phase + gate passes;
//                     the replay's trace contributions (diagonal entries) as per-CTA partials
//   tr_rows_kernel<N> one CTA per row w of W: w <- w exp(+i tau H), i.e. the column vector w^T
//                     through the Taylor series of i tau H^T, every term on chip (two shared
//                     buffers, the output in registers); H^T acts as D(c) t[c] + sum_i
//                     (bx_i/2 + i by_i/2 (1 - 2 b_i(c))) t[c ^ m_i]; the term count is fixed per step
//                     from ||tau H|| <= tau (max|D| + sum_i (|bx_i| + |by_i|)/2) so the truncation is
//                     below 1e-17 (the reference stops at a 1e-13 term size)
//   tr_trace_reduce   fixed-order sum of the per-CTA partials (deterministic, no atomics)
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "../../include/symqoc_b200.h"
#include "devonce.h"

namespace sqoc {
int report_error(int code, const std::string& msg);  // engine.cu (sqoc_last_error)
}
using sqoc::report_error;

#define TR_CUDA(call)                                                                                \
  do {                                                                                               \
    cudaError_t e_ = (call);                                                                         \
    if (e_ != cudaSuccess) return report_error(SQOC_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

namespace {

constexpr int kMinQubits = 1, kMaxQubits = 12;

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c) {  // a b + c
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}

// exp(-i tau h), h = [[bz/2, (bx - i by)/2], [(bx + i by)/2, -bz/2]] (trotter.py:48-65, :132-136):
// c0 = 0, (vx, vy, vz) = (bx, by, bz)/2.  fac[4 * (step * n + site)] = u00, u01, u10, u11.
__global__ void tr_factor_kernel(const double* __restrict__ bx, const double* __restrict__ by, int steps, int n,
                                 double bz, double tau, double2* __restrict__ fac) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= steps * n) return;
  const double vx = 0.5 * bx[t], vy = 0.5 * by[t], vz = 0.5 * bz;
  const double r = sqrt(vx * vx + vy * vy + vz * vz);
  double2* u = fac + 4 * (size_t)t;
  if (r < 1e-300) {
    u[0] = make_double2(1.0, 0.0);
    u[1] = make_double2(0.0, 0.0);
    u[2] = make_double2(0.0, 0.0);
    u[3] = make_double2(1.0, 0.0);
    return;
  }
  const double nx = vx / r, ny = vy / r, nz = vz / r;
  double s, c;
  sincos(tau * r, &s, &c);
  // [[c - i s nz, -i s (nx - i ny)], [-i s (nx + i ny), c + i s nz]]
  u[0] = make_double2(c, -s * nz);
  u[1] = make_double2(-s * ny, -s * nx);
  u[2] = make_double2(s * ny, -s * nx);
  u[3] = make_double2(c, s * nz);
}

__global__ void tr_eye_kernel(double2* __restrict__ W, int dim) {
  const size_t total = (size_t)dim * dim;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x)
    W[i] = make_double2((i / dim == i % dim) ? 1.0 : 0.0, 0.0);
}

// One pass over a column pair in shared memory: optional phase before, the gate on bit `bit`,
// optional phase after (phases multiply the row index x: s[x] *= ph[x]).
template <int N>
__device__ __forceinline__ void col_pass(double2* s, int bit, const double2* __restrict__ g,
                                         const double2* __restrict__ pre, const double2* __restrict__ post) {
  constexpr int DIM = 1 << N;
  const double2 u00 = g[0], u01 = g[1], u10 = g[2], u11 = g[3];
  const int m = 1 << bit;
  for (int p = threadIdx.x; p < DIM; p += blockDim.x) {  // p = pair index * 2 + column
    const int pair = p >> 1, col = p & 1;
    const int lo = ((pair >> bit) << (bit + 1)) | (pair & (m - 1));
    const int hi = lo | m;
    double2 a = s[2 * lo + col], b = s[2 * hi + col];
    if (pre) {
      a = cmul(a, pre[lo]);
      b = cmul(b, pre[hi]);
    }
    double2 na = cfma(u00, a, cmul(u01, b));
    double2 nb = cfma(u10, a, cmul(u11, b));
    if (post) {
      na = cmul(na, post[lo]);
      nb = cmul(nb, post[hi]);
    }
    s[2 * lo + col] = na;
    s[2 * hi + col] = nb;
  }
  __syncthreads();
}

// n_steps Trotter steps on columns [2 blockIdx.x, 2 blockIdx.x + 1] of A (dim x cols, row-major).
// fac: [n_steps][n][4] (Strang: the tau/2 factors); phase: [dim] (Strang: the half phase), or null
// when uncoupled.  trace_out (replay, n_steps == 1): per-CTA partial sum of the diagonal entries.
template <int N>
__global__ void __launch_bounds__(256) tr_cols_kernel(double2* __restrict__ A, int cols, int n_steps,
                                                      const double2* __restrict__ fac,
                                                      const double2* __restrict__ phase, int strang,
                                                      double2* __restrict__ trace_out) {
  constexpr int DIM = 1 << N;
  extern __shared__ double2 s[];  // [DIM][2]
  const int c0 = 2 * blockIdx.x;
  const int nc = min(2, cols - c0);
  for (int p = threadIdx.x; p < 2 * DIM; p += blockDim.x) {
    const int x = p >> 1, col = p & 1;
    s[p] = col < nc ? A[(size_t)x * cols + c0 + col] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  for (int j = 0; j < n_steps; ++j) {
    const double2* f = fac + (size_t)j * N * 4;
    if (strang) {
      for (int i = 1; i <= N; ++i) col_pass<N>(s, N - i, f + 4 * (i - 1), nullptr, phase);
      for (int i = N; i >= 1; --i) col_pass<N>(s, N - i, f + 4 * (i - 1), phase, nullptr);
    } else {
      for (int i = N; i >= 1; --i) col_pass<N>(s, N - i, f + 4 * (i - 1), phase, nullptr);
    }
  }
  for (int p = threadIdx.x; p < 2 * DIM; p += blockDim.x) {
    const int x = p >> 1, col = p & 1;
    if (col < nc) A[(size_t)x * cols + c0 + col] = s[p];
  }
  if (trace_out && threadIdx.x == 0) {
    double2 t = s[2 * c0];
    if (nc > 1) {
      t.x += s[2 * (c0 + 1) + 1].x;
      t.y += s[2 * (c0 + 1) + 1].y;
    }
    trace_out[blockIdx.x] = t;
  }
}

// Taylor terms m with beta^(m+1)/(m+1)! / (1 - beta/(m+2)) <= 1e-17.
__device__ int tr_terms(double beta) {
  double term = 1.0;
  for (int m = 1; m < 120; ++m) {
    term *= beta / m;
    const double next = term * beta / (m + 1);
    if (beta < m + 2 && next / (1.0 - beta / (m + 2)) <= 1e-17) return m;
  }
  return 120;
}

// Row r of W <- W[r] exp(+i tau H): the column vector through sum_k (i tau H^T)^k / k!.
template <int N>
__global__ void __launch_bounds__(256) tr_rows_kernel(double2* __restrict__ W, const double* __restrict__ diag,
                                                      double dmax, const double* __restrict__ bx,
                                                      const double* __restrict__ by, double tau) {
  constexpr int DIM = 1 << N;
  constexpr int T = DIM < 32 ? 32 : (DIM < 256 ? DIM : 256);
  constexpr int Q = (DIM + T - 1) / T;
  extern __shared__ double2 sm[];  // t[2][DIM]
  double2* t0 = sm;
  double2* t1 = sm + DIM;
  double cx[N], cy[N];
  double beta = dmax;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    cx[i] = 0.5 * bx[i];
    cy[i] = 0.5 * by[i];
    beta += fabs(cx[i]) + fabs(cy[i]);
  }
  const int m_terms = tr_terms(tau * beta);
  double2* row = W + (size_t)blockIdx.x * DIM;
  double2 out[Q];
  double dloc[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int c = threadIdx.x + q * T;
    if (c < DIM) {
      out[q] = row[c];
      t0[c] = out[q];
      dloc[q] = diag[c];
    }
  }
  __syncthreads();
  for (int k = 1; k <= m_terms; ++k) {
    const double a = tau / k;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int c = threadIdx.x + q * T;
      if (c >= DIM) continue;
      double2 h = make_double2(dloc[q] * t0[c].x, dloc[q] * t0[c].y);
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const int bit = N - 1 - i;  // site i + 1
        const double sy = ((c >> bit) & 1) ? -cy[i] : cy[i];
        h = cfma(make_double2(cx[i], sy), t0[c ^ (1 << bit)], h);
      }
      const double2 nt = make_double2(-a * h.y, a * h.x);  // (i a) h
      t1[c] = nt;
      out[q].x += nt.x;
      out[q].y += nt.y;
    }
    __syncthreads();
    double2* tmp = t0;
    t0 = t1;
    t1 = tmp;
  }
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int c = threadIdx.x + q * T;
    if (c < DIM) row[c] = out[q];
  }
}

__global__ void tr_trace_reduce_kernel(const double2* __restrict__ part, int n_rec, int nct, double inv_dim2,
                                       double* __restrict__ fids) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rec) return;
  double sx = 0.0, sy = 0.0;
  for (int i = 0; i < nct; ++i) {
    sx += part[(size_t)r * nct + i].x;
    sy += part[(size_t)r * nct + i].y;
  }
  fids[r] = (sx * sx + sy * sy) * inv_dim2;
}

template <int N>
cudaError_t launch_cols(double2* A, int cols, int n_steps, const double2* fac, const double2* phase, int strang,
                        double2* trace_out, cudaStream_t st) {
  constexpr size_t smem = sizeof(double2) * 2 * (1 << N);
  static std::mutex mu;
  static uint64_t done = 0;
  cudaError_t e = sqoc::once_per_device(mu, done, [] {
    return cudaFuncSetAttribute(tr_cols_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  });
  if (e != cudaSuccess) return e;
  tr_cols_kernel<N><<<(cols + 1) / 2, 256, smem, st>>>(A, cols, n_steps, fac, phase, strang, trace_out);
  return cudaGetLastError();
}

template <int N>
cudaError_t launch_rows(double2* W, const double* diag, double dmax, const double* bx, const double* by, double tau,
                        cudaStream_t st) {
  constexpr int DIM = 1 << N;
  constexpr int T = DIM < 32 ? 32 : (DIM < 256 ? DIM : 256);
  constexpr size_t smem = sizeof(double2) * 2 * DIM;
  static std::mutex mu;
  static uint64_t done = 0;
  cudaError_t e = sqoc::once_per_device(mu, done, [] {
    return cudaFuncSetAttribute(tr_rows_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  });
  if (e != cudaSuccess) return e;
  tr_rows_kernel<N><<<DIM, T, smem, st>>>(W, diag, dmax, bx, by, tau);
  return cudaGetLastError();
}

#define TR_DISPATCH(n, CALL)                                                                     \
  switch (n) {                                                                                   \
    case 1: CALL(1); break;                                                                      \
    case 2: CALL(2); break;                                                                      \
    case 3: CALL(3); break;                                                                      \
    case 4: CALL(4); break;                                                                      \
    case 5: CALL(5); break;                                                                      \
    case 6: CALL(6); break;                                                                      \
    case 7: CALL(7); break;                                                                      \
    case 8: CALL(8); break;                                                                      \
    case 9: CALL(9); break;                                                                      \
    case 10: CALL(10); break;                                                                    \
    case 11: CALL(11); break;                                                                    \
    default: CALL(12); break;                                                                    \
  }

}  // namespace

struct sqoc_trotter {
  int device = 0, n = 0, dim = 0;
  double bz = 0.0, tau = 0.0;
  int strang = 0;
  bool coupled = false;
  double dmax = 0.0;
  double* diag = nullptr;      // [dim] exact H diagonal (field + couplings)
  double2* phase = nullptr;    // [dim] coupling phases of one layer (Strang: half), null if uncoupled
  double2* W = nullptr;        // replay accumulator
  double2* fac = nullptr;      // [steps][n][4]
  size_t fac_cap = 0;
  double* ctl = nullptr;       // staged controls [2][steps][n]
  size_t ctl_cap = 0;
  double2* part = nullptr;     // replay trace partials
  size_t part_cap = 0;
  double2* arr = nullptr;      // staged host accumulator
  size_t arr_cap = 0;
  int launches = 0;
};

namespace {

template <class T>
int ensure(T*& p, size_t& cap, size_t need) {
  if (need <= cap) return SQOC_OK;
  cudaFree(p);
  p = nullptr;
  cap = 0;
  TR_CUDA(cudaMalloc(&p, std::max<size_t>(need, 1) * sizeof(T)));
  cap = need;
  return SQOC_OK;
}

// controls to the device and the 2 x 2 factors of every step
int stage_factors(sqoc_trotter* t, const double* bx, const double* by, int n_steps, int memory, cudaStream_t st,
                  const double** bx_dev, const double** by_dev) {
  const size_t nn = (size_t)n_steps * t->n;
  int rc = ensure(t->fac, t->fac_cap, 4 * nn);
  if (rc) return rc;
  if (memory == SQOC_MEM_HOST) {
    if ((rc = ensure(t->ctl, t->ctl_cap, 2 * nn))) return rc;
    TR_CUDA(cudaMemcpyAsync(t->ctl, bx, nn * sizeof(double), cudaMemcpyHostToDevice, st));
    TR_CUDA(cudaMemcpyAsync(t->ctl + nn, by, nn * sizeof(double), cudaMemcpyHostToDevice, st));
    *bx_dev = t->ctl;
    *by_dev = t->ctl + nn;
  } else {
    *bx_dev = bx;
    *by_dev = by;
  }
  if (nn) {
    tr_factor_kernel<<<(unsigned)((nn + 255) / 256), 256, 0, st>>>(*bx_dev, *by_dev, n_steps, t->n, t->bz,
                                                                   t->strang ? 0.5 * t->tau : t->tau, t->fac);
    TR_CUDA(cudaGetLastError());
    t->launches++;
  }
  return SQOC_OK;
}

}  // namespace

extern "C" {

int sqoc_trotter_create(sqoc_trotter** out, int device, int n, double bz, const double* couplings, int n_couplings,
                        double tau, int strang) {
  if (!out) return report_error(SQOC_ERR_ARG, "out is NULL");
  *out = nullptr;
  if (n < kMinQubits || n > kMaxQubits) return report_error(SQOC_ERR_ARG, "Trotter plan needs 1 <= n <= 12");
  if (n_couplings < 0 || n_couplings > n / 2 || (n_couplings && !couplings))
    return report_error(SQOC_ERR_ARG, "at most floor(n/2) coupling offsets (model.py:31-33)");
  if (!std::isfinite(tau) || !std::isfinite(bz)) return report_error(SQOC_ERR_ARG, "tau and bz must be finite");
  TR_CUDA(cudaSetDevice(device));
  const int dim = 1 << n;
  std::vector<double> cpl(dim, 0.0), diag(dim, 0.0);
  bool coupled = false;
  for (int k = 1; k <= n_couplings; ++k) {
    const double c = couplings[k - 1];
    if (!std::isfinite(c)) return report_error(SQOC_ERR_ARG, "couplings must be finite");
    if (c == 0.0) continue;
    coupled = true;
    for (int i = 1; i <= n; ++i) {  // literal ring sums (model.py:66-70)
      const int j = (i - 1 + k) % n + 1;
      for (int x = 0; x < dim; ++x) {
        const int zi = 1 - 2 * ((x >> (n - i)) & 1), zj = 1 - 2 * ((x >> (n - j)) & 1);
        cpl[x] += 0.25 * c * zi * zj;
      }
    }
  }
  double dmax = 0.0;
  for (int x = 0; x < dim; ++x) {
    double f = 0.0;
    for (int i = 1; i <= n; ++i) f += 0.5 * bz * (1 - 2 * ((x >> (n - i)) & 1));
    diag[x] = f + cpl[x];
    dmax = std::max(dmax, std::fabs(diag[x]));
  }
  sqoc_trotter* t = new sqoc_trotter();
  t->device = device;
  t->n = n;
  t->dim = dim;
  t->bz = bz;
  t->tau = tau;
  t->strang = strang ? 1 : 0;
  t->coupled = coupled;
  t->dmax = dmax;
  auto fail = [&](cudaError_t e, const char* what) {
    cudaFree(t->diag);
    cudaFree(t->phase);
    delete t;
    return report_error(SQOC_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  };
  cudaError_t e = cudaMalloc(&t->diag, dim * sizeof(double));
  if (e != cudaSuccess) return fail(e, "cudaMalloc diag");
  e = cudaMemcpy(t->diag, diag.data(), dim * sizeof(double), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return fail(e, "copy diag");
  if (coupled) {  // exp(-i (tau / n) cpl) per layer; Strang: exp(-i (tau / 2n) cpl)  (trotter.py:110-111)
    const double a = (strang ? 0.5 * tau : tau) / n;
    std::vector<double2> ph(dim);
    for (int x = 0; x < dim; ++x) ph[x] = make_double2(std::cos(a * cpl[x]), -std::sin(a * cpl[x]));
    e = cudaMalloc(&t->phase, dim * sizeof(double2));
    if (e != cudaSuccess) return fail(e, "cudaMalloc phase");
    e = cudaMemcpy(t->phase, ph.data(), dim * sizeof(double2), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return fail(e, "copy phase");
  }
  *out = t;
  return SQOC_OK;
}

int sqoc_trotter_destroy(sqoc_trotter* t) {
  if (!t) return SQOC_OK;
  cudaSetDevice(t->device);
  cudaFree(t->diag);
  cudaFree(t->phase);
  cudaFree(t->W);
  cudaFree(t->fac);
  cudaFree(t->ctl);
  cudaFree(t->part);
  cudaFree(t->arr);
  delete t;
  return SQOC_OK;
}

int sqoc_trotter_apply(sqoc_trotter* t, double* arr, int cols, const double* bx, const double* by, int n_steps,
                       int memory, void* stream) {
  if (!t) return report_error(SQOC_ERR_ARG, "plan is NULL");
  if (memory != SQOC_MEM_HOST && memory != SQOC_MEM_DEVICE) return report_error(SQOC_ERR_ARG, "unknown memory kind");
  if (!arr || cols < 1 || n_steps < 0 || (n_steps && (!bx || !by)))
    return report_error(SQOC_ERR_ARG, "need arr, cols >= 1 and one control pair per site and step");
  TR_CUDA(cudaSetDevice(t->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  t->launches = 0;
  const double *bxd = nullptr, *byd = nullptr;
  int rc = stage_factors(t, bx, by, n_steps, memory, st, &bxd, &byd);
  if (rc) return rc;
  const size_t elems = (size_t)t->dim * cols;
  double2* A = reinterpret_cast<double2*>(arr);
  if (memory == SQOC_MEM_HOST) {
    if ((rc = ensure(t->arr, t->arr_cap, elems))) return rc;
    TR_CUDA(cudaMemcpyAsync(t->arr, arr, elems * sizeof(double2), cudaMemcpyHostToDevice, st));
    A = t->arr;
  }
  if (n_steps) {
    cudaError_t e = cudaSuccess;
#define TR_COLS(N) e = launch_cols<N>(A, cols, n_steps, t->fac, t->phase, t->strang, nullptr, st)
    TR_DISPATCH(t->n, TR_COLS)
#undef TR_COLS
    TR_CUDA(e);
    t->launches++;
  }
  if (memory == SQOC_MEM_HOST) TR_CUDA(cudaMemcpyAsync(arr, A, elems * sizeof(double2), cudaMemcpyDeviceToHost, st));
  TR_CUDA(cudaStreamSynchronize(st));
  return SQOC_OK;
}

int sqoc_trotter_replay(sqoc_trotter* t, const double* bx, const double* by, int n_steps, int record_every,
                        double* fids, int memory, void* stream) {
  if (!t) return report_error(SQOC_ERR_ARG, "plan is NULL");
  if (memory != SQOC_MEM_HOST && memory != SQOC_MEM_DEVICE) return report_error(SQOC_ERR_ARG, "unknown memory kind");
  if (n_steps < 1 || record_every < 1 || !bx || !by || !fids)
    return report_error(SQOC_ERR_ARG, "need n_steps >= 1, record_every >= 1, controls and fids");
  TR_CUDA(cudaSetDevice(t->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  t->launches = 0;
  const double *bxd = nullptr, *byd = nullptr;
  int rc = stage_factors(t, bx, by, n_steps, memory, st, &bxd, &byd);
  if (rc) return rc;
  const int dim = t->dim, n = t->n;
  const int n_rec = (n_steps + record_every - 1) / record_every;
  const int nct = (dim + 1) / 2;
  if (!t->W) TR_CUDA(cudaMalloc(&t->W, (size_t)dim * dim * sizeof(double2)));
  if ((rc = ensure(t->part, t->part_cap, (size_t)n_rec * nct))) return rc;
  tr_eye_kernel<<<std::min(4096, (dim * dim + 255) / 256), 256, 0, st>>>(t->W, dim);
  TR_CUDA(cudaGetLastError());
  t->launches++;
  int rec = 0;
  for (int j = 0; j < n_steps; ++j) {
    cudaError_t e = cudaSuccess;
#define TR_ROWS(N) e = launch_rows<N>(t->W, t->diag, t->dmax, bxd + (size_t)j * n, byd + (size_t)j * n, t->tau, st)
    TR_DISPATCH(n, TR_ROWS)
#undef TR_ROWS
    TR_CUDA(e);
    const bool record = (j + 1) % record_every == 0 || j == n_steps - 1;
    double2* tr = record ? t->part + (size_t)rec * nct : nullptr;
#define TR_COLS(N) e = launch_cols<N>(t->W, dim, 1, t->fac + (size_t)j * n * 4, t->phase, t->strang, tr, st)
    TR_DISPATCH(n, TR_COLS)
#undef TR_COLS
    TR_CUDA(e);
    rec += record;
    t->launches += 2;
  }
  double* fd = fids;
  double* tmp = nullptr;
  if (memory == SQOC_MEM_HOST) {
    TR_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&tmp), n_rec * sizeof(double), st));
    fd = tmp;
  }
  tr_trace_reduce_kernel<<<(n_rec + 127) / 128, 128, 0, st>>>(t->part, n_rec, nct, 1.0 / ((double)dim * dim), fd);
  TR_CUDA(cudaGetLastError());
  t->launches++;
  if (memory == SQOC_MEM_HOST) {
    TR_CUDA(cudaMemcpyAsync(fids, tmp, n_rec * sizeof(double), cudaMemcpyDeviceToHost, st));
    TR_CUDA(cudaFreeAsync(tmp, st));
  }
  TR_CUDA(cudaStreamSynchronize(st));
  return SQOC_OK;
}

int sqoc_trotter_last_launches(const sqoc_trotter* t) { return t ? t->launches : 0; }

}  // extern "C"
