// Batched-GEMM path for large symmetry blocks (d > kTinyMaxDim): D_n blocks of
// cfg 2 / cfg 3 and the unsymmetrised 2^n space of cfg 4.
//
// All large blocks of a problem are advanced together: every step below is ONE
// launch whose work list holds one GEMM per block (zgemm.cuh), so the 16 D_14
// blocks (495..1179) fill the 148 SMs together.  Per slice j (same algebra as
// tiny.cuh; the propagator scheme -- degree 12 in 4 products or degree 18 in 5 -- and
// s squarings are chosen once per evaluation from the bound
// ||A_j|| <= ||a_0|| + sum_k |u_kj| ||a_k||, large.cu "propagator schemes"):
//
//   forward : A, scheme steps (P products) -> Y, T <- T T (s x), X <- U X
//   backward: gate objective -- one d x d carry Ad = 2^-s C_j, C_j = X_j Lam_j^dag (formed once
//             from X_N and Lam_N); scheme steps as forward-mode pairs seeded with Ad, squaring
//             pairs -> (U, N = L_R(A, C_j)); one launch forms M = U^dag Ad and the trace
//             dtau_k = Tr(U^dag N E_k); then Ad <- M U (C_{j-1} = U^dag C_j U).
//             State objective (vector X, Lam): Ad = 2^-s X Lam^dag per slice, the same pairs
//             and trace, X <- U^dag X, Lam <- U^dag Lam.
//
// Slice-chunk sharding runs the same sweeps on one rank's slices, split in two phases around the
// exchange of the chunk products (LargeGroup::chunk_phase).
#pragma once
#include <cuda_runtime.h>

#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "sparse.cuh"
#include "zgemm_tma.cuh"

namespace sqoc {

struct LargeArgs {
  const double* u;   // [batch][K][N]
  int batch;
  double2* tau_out;  // tau of (s, large block i) at tau_out[s * tau_stride + global_block[i]]
  int tau_stride;
  double* gradb;     // per-block contributions [global block][max_batch][K][N]
  size_t gradb_block_stride;
};

struct LargeBlockSpec {
  int global_index;
  int d;
  const double2* gen;     // (K+1) d*d
  const double2* x0;      // state objective: psi_0
  const double2* target;  // V or psi_f
  double weight;
  double gen_norm[5];     // inf-norm bounds of a_0..a_K
  // union pattern of a_0..a_K (host CSR) and the generator values on it, [(K+1)][nnz]
  std::vector<int> sp_rp, sp_ci;
  std::vector<double2> sp_gv;
};

struct SpListRef {
  SpItem* dev = nullptr;
  int n = 0, rows = 0;
};

struct ListRef {
  GemmItem* dev = nullptr;
  ItemMaps* maps = nullptr;  // TMA tensor maps per item (null: cp.async staging)
  TileRef* tref = nullptr;   // persistent kernel's tile list (cost-ordered)
  int n = 0, tiles = 0;
  int pt_tiles = -1;  // tiles in tref (fewer than `tiles` when Hermitian items skip their mirror tiles)
  double macs = 0.0;  // complex multiply-adds of the list (sum m n k nseg), for the executed-FLOP count
};

struct LargeGroup {
  int nblk = 0, K = 0, N = 0;  // X / Lam have d columns per block (gate) or 1 (state)
  bool gate = true;
  std::vector<LargeBlockSpec> blocks;
  std::vector<size_t> off;    // block offsets into square workspace arrays (double2 units)
  std::vector<size_t> offr;   // block offsets into d x R arrays
  size_t total = 0, totalr = 0;
  double2 *A = nullptr, *Ad = nullptr, *A2 = nullptr, *dA2 = nullptr, *A3 = nullptr, *dA3 = nullptr;
  double2 *xs[5] = {}, *dxs[5] = {};  // scheme slots 3..7 (A6, P, Q, W1, W2) and their derivatives
  double2 *T[2] = {nullptr, nullptr}, *dT[2] = {nullptr, nullptr};
  double2 *X[2] = {nullptr, nullptr}, *L[2] = {nullptr, nullptr};
  double2* trace_part = nullptr;  // [sum tiles][K]
  std::vector<int> trace_tile_off;
  int trace_tiles = 0;
  double2* tau_dev = nullptr;     // [nblk]
  double* norm_dev = nullptr;     // scalar (max bound)
  int* pt_counter = nullptr;      // persistent GEMM's dynamic tile counter (zeroed before each launch)
  double* gnorm_dev = nullptr;    // [nblk][K+1]
  // device copies of per-block info for elementwise kernels
  int* d_dev = nullptr;
  size_t* off_dev = nullptr;
  size_t* offr_dev = nullptr;
  const double2** gen_dev = nullptr;
  const double2** tgt_dev = nullptr;
  const double2** x0_dev = nullptr;
  double* w_dev = nullptr;
  int* gidx_dev = nullptr;
  // GEMM work lists, built once (device), keyed by op + buffer parities
  std::map<std::tuple<int, int, int, int>, ListRef> lists;
  std::vector<void*> list_mem;
  // GEMM timing (sqoc_set_timing): an event pair around every GEMM launch of the last evaluation
  bool timing = false;
  std::vector<cudaEvent_t> tev;
  size_t tev_used = 0;
  double gemm_macs = 0.0;  // complex MACs issued by the last evaluation's GEMMs
  int gemm_launches = 0;
  int* tile_off_dev = nullptr;    // [nblk + 1] trace tile offsets
  // ---- sparse generators (sparse.cuh): the scheme's products with A as a factor and the gradient
  // trace run as sparse x dense kernels in the slice-sequential schedule when every block's pattern is
  // sparse enough (sp_on; SQOC_SPARSE=0 disables) ----
  // dry pass: the slice-sequential driver runs once without launching anything so that every work list it
  // needs (tile lists, tensor maps, sparse items: cudaMalloc + host-to-device copies) exists before the
  // first kernel of an evaluation starts
  bool warmed = false;                     // first evaluation repeated once (large_eval)
  bool dry = false;
  int seq_ready_key = -1;                  // scheme degree * 100 + squarings the lists were prepared for
  bool sp_on = false;
  bool sp_a2 = false;                      // A2 = A A by spgemm_a2_kernel (SQOC_SPGEMM=0 disables)
  SpBlockDev* sp_dev = nullptr;            // [nblk]
  std::vector<void*> sp_mem;
  double2* sp_part = nullptr;              // [sum d][K] trace partials by row
  int* sp_rowoff_dev = nullptr;            // [nblk + 1] row offsets (trace_reduce_kernel's tile offsets)
  size_t sp_smem = 0;                      // bytes of one dense row (max d double2)
  int sp_w = 1;                            // rows / columns per sparse-kernel CTA
  int sp_trace_tiles = 0;
  std::map<std::tuple<int, int, int, int>, SpListRef> splists;
  std::vector<void*> splist_mem;
  SpTraceItem* sp_trace_dev = nullptr;     // per p parity: [2][nblk]
  // ---- history schedule: every slice resident, slice-batched GEMMs (chosen when memory allows) ----
  int h_deg = -1, h_s = -1, h_C = 0;
  double2* h_chain = nullptr;       // [C][N][total]: scheme slots 0..8 (A .. Y), S_1..S_s
  double2* h_X = nullptr;           // [N+1][totalr]
  double2* h_L = nullptr;           // [N+1][totalr]
  double2* h_d[8] = {};             // [N][total] derivatives of scheme slots 0..7 (dA = seed)
  double2* h_dH[2] = {nullptr, nullptr};  // [N][total] dY and the squaring derivatives
  double2* h_g = nullptr;           // [N][nblk][K] traces
  double2* h_I = nullptr;           // [totalr] identity per block (chunked scans)
  const double2** gent_dev = nullptr;  // per block a_k^T (K d*d), for the slice traces
  std::vector<void*> gent_mem;
  std::map<std::tuple<int, int, int, int>, ListRef> hlists;
  std::vector<void*> hlist_mem;
  // ---- state-vector schedule (state objective): U_j history, vector sweeps, augmented Taylor action ----
  double2* sv_U = nullptr;          // [N][total]
  double2* sv_chunk = nullptr;      // [10][S][total]: scheme slots 0..8, squaring partner
  int sv_S = 0;
  double2* sv_psi = nullptr;        // [N+1][totalr]
  double2* sv_chi = nullptr;        // [N+1][totalr]
  double2* sv_V = nullptr;          // per block b: [(K+1) N][d_b] rows y_i, x_1,i .. x_K,i
  double2* sv_W = nullptr;          // [K+1] x same shape as sv_V
  double2* sv_acc = nullptr;        // per block: [K N][d_b]
  double2* sv_g = nullptr;          // [N][nblk][K]
  double2* mf_t = nullptr;          // matrix-free schedule: Taylor term vectors [3][totalr]
  const double2** gentall_dev = nullptr;  // per block a_k^T for k = 0..K
  std::vector<void*> gentall_mem;
  int last_degree = 0, last_s = 0, last_taylor_terms = 0;
  // ---- slice-chunk sharding (sqoc_chunk_forward / sqoc_chunk_backward) ----
  // phase 1 writes this chunk's product C = U_{N-1} .. U_0 of every block, packed in block order
  // (block b at off[b], d_b x d_b row-major), to chunk_out.  Phase 2 reads the products of all P
  // chunks (chunk_in, [P][total], chunk order) and forms the boundary values on the device:
  //   gate : X_end = C_c C_{c-1} .. C_0, Lam_end = C_{c+1}^dag .. C_{P-1}^dag V, tau = <Lam_end, X_end>
  //          -> the slice-sequential backward sweep only (the forward ran in phase 1);
  //   state: psi_start = C_{c-1} .. C_0 psi_0, chi_end = C_{c+1}^dag .. C_{P-1}^dag psi_f,
  //          tau = <chi_end, C_c psi_start> -> vector sweeps + gradient over the U_j phase 1 kept.
  int chunk_phase = 0;                // 0 ordinary evaluation, 1 chunk forward, 2 chunk backward
  double2* chunk_out = nullptr;       // phase 1 output [total]
  const double2* chunk_in = nullptr;  // phase 2 input [P][total]
  int chunk_P = 0, chunk_c = 0;
  bool chunk_fwd_valid = false;       // state: sv_U holds the propagators of the last phase 1
  double2* chunk_vec = nullptr;       // state carries: [5][totalr]
  double2* chunk_tau = nullptr;       // [nblk]
  const double2** chunk_ptrs = nullptr;  // device [2][nblk]: X_start / Lam_end block pointers
  cudaEvent_t carry_ev[2] = {nullptr, nullptr};
  float carry_ms = 0.f;               // device time of the last phase 2's carries (timing on)
  int carry_gemms = 0;                // carry GEMM launches of the last phase 2
  // boundary values consumed by bc_init / bc_tau (set only inside a phase 2 evaluation)
  const double2** bc_x_dev = nullptr;
  const double2** bc_l_dev = nullptr;
  const double2* bc_tau = nullptr;
  // ---- propagator history of the slice-sequential gate schedule: U_j of every slice, written by the
  // forward sweep, so the backward sweep skips the value half of the product that forms U_j (one
  // d^3 GEMM-unit per slice); kept only when N sum d^2 fits the free memory (SQOC_UHIST=0 disables) ----
  double2* uh = nullptr;            // [N][total]
  bool uh_valid = false;            // uh holds the propagators of the last forward sweep (same u)
  int mode = -1;                    // last schedule used: 0 sequential, 1 history, 2 state-vector, 3 matrix-free
  int force_mode = -1;              // -1 auto, 0 sequential, 1 history, 2 state-vector, 3 matrix-free
  int launches = 0;
  std::string err;
};

int large_init(LargeGroup& g, const std::vector<LargeBlockSpec>& blocks, int K, int N, bool gate);
int large_eval(LargeGroup& g, const LargeArgs& a, cudaStream_t st);
int large_set_norms(LargeGroup& g, const std::vector<double>& gnorm);
int large_set_complex_gemm(int mults);
int large_complex_mults();  // 3 (Gauss) or 4
int large_set_staging(int mode);  // 3M GEMM: 1 persistent TMA + mbarrier ring (default), 0 cp.async
int large_staging();
// Device time of the last evaluation's GEMM launches (needs g.timing during it).
int large_gemm_time(LargeGroup& g, double* ms);
// Device time of the last chunk phase 2's boundary-value formation (needs g.timing during it).
int large_carry_time(LargeGroup& g, double* ms);
void large_free(LargeGroup& g);

}  // namespace sqoc
