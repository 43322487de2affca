// Fused on-chip GRAPE evaluation for tiny symmetry blocks (d <= 16).
//
// One group of d lanes owns one (control vector, block) problem; lane r owns
// row r of every d x d matrix.  Right-hand GEMM operands live in shared memory
// and are read as warp broadcasts; left operands are the lane's own row.
// FP64 on sm_100a: DFMA and DMMA run at the same 64 FMA/clk/SM (measured,
// profiles/r01_fp64_peak.txt), so a DFMA kernel that pads nothing beats a
// DMMA kernel that pads 13 -> 16.
//
// Per slice j (A_j = -i dt (H0 + sum_k u_kj H_k), U_j = R(A_j) with
// R = Taylor_m(A/2^s)^(2^s), Paterson-Stockmeyer with A^2, A^3):
//   forward : X_j = U_j X_{j-1}
//   backward: C_j = X_j Lam_j^dag,  (U_j, N_j) = (R(A_j), L_R(A_j, C_j)) by
//             forward-mode pairs,   D_j = U_j^dag N_j = L_R(A_j, X_{j-1} Lam_j^dag),
//             dtau/du_kj = Tr(D_j E_k),  X_{j-1} = U_j^dag X_j,  Lam_{j-1} = U_j^dag Lam_j.
// The identity Tr(B L(A,E)) = Tr(L(A,B) E) turns K Frechet derivatives into one.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace sqoc {

constexpr int kTinyMaxDim = 16;
constexpr int kTinyBuffers = 8;   // d x d matrices per problem in shared memory
constexpr int kMaxControls = 4;

struct TinyParams {
  int K, N, batch;
  const double2* gen;     // (K+1) d*d: a0 = -i dt H0, a_k = -i dt H_k
  const double2* x0;      // state: psi_0 (d); gate: unused (identity)
  const double2* target;  // gate: V (d*d); state: psi_f (d)
  const double* u;        // [batch][K][N]
  double weight;          // w_b
  double2* tau_out;       // tau of (problem, block) at tau_out[prob * tau_stride]
  int tau_stride;
  double* grad_out;       // [batch][K][N] contribution of this block
  double2* park;          // [batch][2][d*R] workspace (X, Lam between phases)
  int nwarps;             // warps per CTA
};

// Taylor coefficients 1/k!, k = 0..21
__constant__ double c_inv_fact[22] = {
    1.0, 1.0, 0.5, 1.6666666666666666e-01, 4.1666666666666664e-02, 8.3333333333333332e-03,
    1.3888888888888889e-03, 1.9841269841269841e-04, 2.4801587301587302e-05,
    2.7557319223985893e-06, 2.7557319223985888e-07, 2.5052108385441720e-08,
    2.0876756987868100e-09, 1.6059043836821613e-10, 1.1470745597729725e-11,
    7.6471637318198164e-13, 4.7794773323873853e-14, 2.8114572543455206e-15,
    1.5619206968586225e-16, 8.2206352466243295e-18, 4.1103176233121648e-19,
    1.9572941063391263e-20};

// Degree m = 3 nb, nb = 4..7: largest ||A|| with truncation <= 2^-53.
__device__ __forceinline__ void choose_taylor(double nrm, int& nb, int& s) {
  const double theta[4] = {0.33, 0.67, 1.10, 1.65};
  int best_cost = 1 << 30;
  nb = 4;
  s = 0;
  for (int i = 0; i < 4; ++i) {
    int si = 0;
    double x = nrm;
    while (x > theta[i] && si < 60) { x *= 0.5; ++si; }
    int cost = (4 + i) + 1 + si;
    if (cost < best_cost || (cost == best_cost && si < s)) { best_cost = cost; nb = 4 + i; s = si; }
  }
}

__device__ __forceinline__ void cfma(double2& acc, const double2 a, const double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 czero() { return make_double2(0.0, 0.0); }

// acc[c] = sum_k L[k] * M[k][c]      (L: own row, M: full matrix in smem, ld D)
template <int D, int NC>
__device__ __forceinline__ void row_mul(double2 (&acc)[NC], const double2* L, const double2* M) {
#pragma unroll
  for (int c = 0; c < NC; ++c) acc[c] = czero();
#pragma unroll 1
  for (int k = 0; k < D; ++k) {
    const double2 l = L[k];
    const double2* m = M + k * NC;
#pragma unroll
    for (int c = 0; c < NC; ++c) cfma(acc[c], l, m[c]);
  }
}

// acc[c] = sum_k conj(U[k][r]) * M[k][c]   (U^dag * M, U full in smem)
template <int D, int NC>
__device__ __forceinline__ void row_mul_adj(double2 (&acc)[NC], const double2* U, int r, const double2* M) {
#pragma unroll
  for (int c = 0; c < NC; ++c) acc[c] = czero();
#pragma unroll 1
  for (int k = 0; k < D; ++k) {
    const double2 l = cconj(U[k * D + r]);
    const double2* m = M + k * NC;
#pragma unroll
    for (int c = 0; c < NC; ++c) cfma(acc[c], l, m[c]);
  }
}

// (T, dT) = (L, dL) x (M, dM):  T = L M,  dT = L dM + dL M
template <int D>
__device__ __forceinline__ void row_mul_pair(double2 (&t)[D], double2 (&dt)[D], const double2* L,
                                             const double2* dL, const double2* M, const double2* dM) {
#pragma unroll
  for (int c = 0; c < D; ++c) { t[c] = czero(); dt[c] = czero(); }
#pragma unroll 1
  for (int k = 0; k < D; ++k) {
    const double2 l = L[k], dl = dL[k];
    const double2* m = M + k * D;
    const double2* dm = dM + k * D;
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const double2 mc = m[c];
      cfma(t[c], l, mc);
      cfma(dt[c], dl, mc);
      cfma(dt[c], l, dm[c]);
    }
  }
}

template <int NC>
__device__ __forceinline__ void store_row(double2* dst, const double2 (&v)[NC], bool wr) {
  if (wr) {
#pragma unroll
    for (int c = 0; c < NC; ++c) dst[c] = v[c];
  }
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Deterministic in-group sum: every lane writes its partial, the group's lanes
// then all read the d partials in order (same result in every lane).
template <int D>
__device__ __forceinline__ double2 group_sum(double2 v, double2* red, int r, bool wr) {
  __syncwarp();
  if (wr) red[r] = v;
  __syncwarp();
  double2 s = czero();
#pragma unroll
  for (int i = 0; i < D; ++i) s = cadd(s, red[i]);
  __syncwarp();
  return s;
}

template <int D, bool GATE>
__global__ void __launch_bounds__(256) grape_tiny_kernel(TinyParams p) {
  constexpr int R = GATE ? D : 1;  // columns of X and Lam
  constexpr int PG = 32 / D;       // problems per warp
  constexpr int DD = D * D;
  constexpr int PSTRIDE = kTinyBuffers * DD + D;  // per-problem smem (double2)
  extern __shared__ double2 smem[];

  const int K = p.K, N = p.N;
  double2* gen = smem;  // (K+1) DD
  for (int i = threadIdx.x; i < (K + 1) * DD; i += blockDim.x) gen[i] = p.gen[i];
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g_raw = lane / D;
  const bool lane_used = g_raw < PG;
  const int g = lane_used ? g_raw : 0;
  const int r = lane_used ? lane - g_raw * D : 0;
  const int slot = (blockIdx.x * p.nwarps + warp) * PG + g;  // problem slot (park is sized for all slots)
  const bool wr = lane_used && slot < p.batch;  // this lane owns a real problem and may store globally
  const int prob = slot < p.batch ? slot : p.batch - 1;  // padding slots replay the last problem's u

  double2* buf = gen + (K + 1) * DD + (size_t)(warp * PG + g) * PSTRIDE;
  double2* B0 = buf;           // X (fwd) | X, A2 (bwd)
  double2* B1 = B0 + DD;       // Lam, dA2
  double2* B2 = B1 + DD;       // A
  double2* B3 = B2 + DD;       // Adot
  double2* B4 = B3 + DD;       // A3
  double2* B5 = B4 + DD;       // dA3
  double2* B6 = B5 + DD;       // T  (-> U)
  double2* B7 = B6 + DD;       // dT (-> N)
  double2* red = B7 + DD;      // D partials
  const double* up = p.u + (size_t)prob * K * N;
  double2* parkX = p.park + (size_t)slot * 2 * D * R;
  double2* parkL = parkX + D * R;

  // ---- build A row r for slice j, return warp-uniform Taylor plan ----
  auto build_a = [&](int j, double2 (&arow)[D], int& nb, int& s) {
    double uk[kMaxControls];
#pragma unroll
    for (int k = 0; k < kMaxControls; ++k) uk[k] = (k < K) ? up[k * N + j] : 0.0;
    double nrm = 0.0;
#pragma unroll
    for (int c = 0; c < D; ++c) {
      double2 a = gen[r * D + c];
      for (int k = 0; k < K; ++k) {
        const double2 e = gen[(k + 1) * DD + r * D + c];
        a.x = fma(uk[k], e.x, a.x);
        a.y = fma(uk[k], e.y, a.y);
      }
      arow[c] = a;
      nrm += fabs(a.x) + fabs(a.y);
    }
    nrm = warp_max(wr ? nrm : 0.0);  // plan is warp-uniform, from real problems only
    choose_taylor(nrm, nb, s);
    const double sc = ldexp(1.0, -s);
#pragma unroll
    for (int c = 0; c < D; ++c) arow[c] = cscale(arow[c], sc);
  };

  // Q_t own row: c_{3t} I + c_{3t+1} A + c_{3t+2} A2
  auto q_row = [&](int t, int c, const double2* A, const double2* A2) {
    double2 v = cadd(cscale(A[r * D + c], c_inv_fact[3 * t + 1]), cscale(A2[r * D + c], c_inv_fact[3 * t + 2]));
    if (c == r) v.x += c_inv_fact[3 * t];
    return v;
  };
  auto dq_row = [&](int t, int c, const double2* dA, const double2* dA2) {
    return cadd(cscale(dA[r * D + c], c_inv_fact[3 * t + 1]), cscale(dA2[r * D + c], c_inv_fact[3 * t + 2]));
  };

  // ================= forward sweep: X_N =================
  double2 row[D];
  {
    double2* X = B0;
    if (GATE) {
#pragma unroll
      for (int c = 0; c < R; ++c) row[c] = make_double2(c == r ? 1.0 : 0.0, 0.0);
    } else {
      row[0] = p.x0[r];
    }
    store_row<R>(X + r * R, *reinterpret_cast<double2(*)[R]>(row), lane_used);
    __syncwarp();
    for (int j = 0; j < N; ++j) {
      int nb, s;
      build_a(j, row, nb, s);
      store_row<D>(B2 + r * D, row, lane_used);
      __syncwarp();
      row_mul<D, D>(row, B2 + r * D, B2);  // A2
      store_row<D>(B1 + r * D, row, lane_used);
      __syncwarp();
      row_mul<D, D>(row, B1 + r * D, B2);  // A3
      store_row<D>(B4 + r * D, row, lane_used);
      __syncwarp();
      // Horner in A3: T = c_{3nb} A3 + Q_{nb-1}
#pragma unroll
      for (int c = 0; c < D; ++c) row[c] = cadd(cscale(row[c], c_inv_fact[3 * nb]), q_row(nb - 1, c, B2, B1));
      for (int t = nb - 2; t >= 0; --t) {
        store_row<D>(B6 + r * D, row, lane_used);
        __syncwarp();
        row_mul<D, D>(row, B6 + r * D, B4);
#pragma unroll
        for (int c = 0; c < D; ++c) row[c] = cadd(row[c], q_row(t, c, B2, B1));
      }
      store_row<D>(B6 + r * D, row, lane_used);
      for (int q = 0; q < s; ++q) {
        __syncwarp();
        row_mul<D, D>(row, B6 + r * D, B6);
        __syncwarp();
        store_row<D>(B6 + r * D, row, lane_used);
      }
      __syncwarp();
      double2 xr[R];
      row_mul<D, R>(xr, B6 + r * D, X);  // X_j = U_j X_{j-1}
      __syncwarp();
      store_row<R>(X + r * R, xr, lane_used);
      __syncwarp();
    }
    // tau = <V, X_N>_F ; park X_N and Lam_N = V
    double2 part = czero();
#pragma unroll
    for (int c = 0; c < R; ++c) {
      const double2 v = p.target[r * R + c];
      const double2 x = X[r * R + c];
      part = cadd(part, cmul(cconj(v), x));
      if (lane_used) { parkX[r * R + c] = x; parkL[r * R + c] = v; }
    }
    const double2 tau = group_sum<D>(part, red, r, lane_used);
    if (wr && r == 0) p.tau_out[(size_t)prob * p.tau_stride] = tau;

    // ================= backward sweep: gradient =================
    const double2 ctw = cscale(cconj(tau), 2.0 * p.weight);  // dF/du = Re(2 w conj(tau) dtau/du)
    for (int j = N - 1; j >= 0; --j) {
      int nb, s;
      // stage X_j, Lam_j (own rows) into B0 / B1
      if (lane_used) {
#pragma unroll
        for (int c = 0; c < R; ++c) { B0[r * R + c] = parkX[r * R + c]; B1[r * R + c] = parkL[r * R + c]; }
      }
      build_a(j, row, nb, s);
      store_row<D>(B2 + r * D, row, lane_used);
      __syncwarp();
      {  // C = X Lam^dag (scaled by 2^-s) -> Adot
        const double sc = ldexp(1.0, -s);
        double2 crow[D];
#pragma unroll
        for (int c = 0; c < D; ++c) crow[c] = czero();
#pragma unroll 1
        for (int k = 0; k < R; ++k) {
          const double2 x = B0[r * R + k];
#pragma unroll
          for (int c = 0; c < D; ++c) cfma(crow[c], x, cconj(B1[c * R + k]));
        }
#pragma unroll
        for (int c = 0; c < D; ++c) crow[c] = cscale(crow[c], sc);
        store_row<D>(B3 + r * D, crow, lane_used);
      }
      __syncwarp();
      double2 drow[D];
      row_mul_pair<D>(row, drow, B2 + r * D, B3 + r * D, B2, B3);  // (A2, dA2)
      store_row<D>(B0 + r * D, row, lane_used);
      store_row<D>(B1 + r * D, drow, lane_used);
      __syncwarp();
      row_mul_pair<D>(row, drow, B0 + r * D, B1 + r * D, B2, B3);  // (A3, dA3)
      store_row<D>(B4 + r * D, row, lane_used);
      store_row<D>(B5 + r * D, drow, lane_used);
      __syncwarp();
#pragma unroll
      for (int c = 0; c < D; ++c) {
        row[c] = cadd(cscale(row[c], c_inv_fact[3 * nb]), q_row(nb - 1, c, B2, B0));
        drow[c] = cadd(cscale(drow[c], c_inv_fact[3 * nb]), dq_row(nb - 1, c, B3, B1));
      }
      for (int t = nb - 2; t >= 0; --t) {
        store_row<D>(B6 + r * D, row, lane_used);
        store_row<D>(B7 + r * D, drow, lane_used);
        __syncwarp();
        row_mul_pair<D>(row, drow, B6 + r * D, B7 + r * D, B4, B5);
#pragma unroll
        for (int c = 0; c < D; ++c) {
          row[c] = cadd(row[c], q_row(t, c, B2, B0));
          drow[c] = cadd(drow[c], dq_row(t, c, B3, B1));
        }
      }
      store_row<D>(B6 + r * D, row, lane_used);
      store_row<D>(B7 + r * D, drow, lane_used);
      for (int q = 0; q < s; ++q) {
        __syncwarp();
        row_mul_pair<D>(row, drow, B6 + r * D, B7 + r * D, B6, B7);
        __syncwarp();
        store_row<D>(B6 + r * D, row, lane_used);
        store_row<D>(B7 + r * D, drow, lane_used);
      }
      __syncwarp();
      // restage X_j, Lam_j (B0/B1 were reused)
      if (lane_used) {
#pragma unroll
        for (int c = 0; c < R; ++c) { B0[r * R + c] = parkX[r * R + c]; B1[r * R + c] = parkL[r * R + c]; }
      }
      __syncwarp();
      // D = U^dag N ; dtau/du_k = Tr(D E_k) = sum_q D[r][q] E_k[q][r]
      row_mul_adj<D, D>(row, B6, r, B7);
      for (int k = 0; k < K; ++k) {
        const double2* E = gen + (k + 1) * DD;
        double2 part2 = czero();
#pragma unroll
        for (int q = 0; q < D; ++q) cfma(part2, row[q], E[q * D + r]);
        const double2 dtau = group_sum<D>(part2, red, r, lane_used);
        if (wr && r == 0) p.grad_out[((size_t)prob * K + k) * N + j] = ctw.x * dtau.x - ctw.y * dtau.y;
      }
      // X_{j-1} = U^dag X_j, Lam_{j-1} = U^dag Lam_j  -> park
      double2 xr[R];
      row_mul_adj<D, R>(xr, B6, r, B0);
      if (lane_used) {
#pragma unroll
        for (int c = 0; c < R; ++c) parkX[r * R + c] = xr[c];
      }
      row_mul_adj<D, R>(xr, B6, r, B1);
      if (lane_used) {
#pragma unroll
        for (int c = 0; c < R; ++c) parkL[r * R + c] = xr[c];
      }
      __syncwarp();
    }
  }
}

inline size_t tiny_smem_bytes(int d, int K, int nwarps) {
  const int pg = 32 / d;
  return sizeof(double2) * ((size_t)(K + 1) * d * d + (size_t)nwarps * pg * (kTinyBuffers * d * d + d));
}

}  // namespace sqoc
