/*
 * symqoc_b200.h -- C ABI of the B200 GRAPE fidelity+gradient engine.
 *
 * Drop-in boundary for the reference's hot path
 *   symqoc.qoc.gradient(psi0, psi_f, bx, by, backend, tau) -> (gx, gy, P)
 *   (/root/reference/pkg/src/symqoc/qoc.py:137-168)
 * generalised to many symmetry blocks, K controls, the gate-fidelity
 * objective and a batch of control vectors.
 *
 * Plain pointers and sizes only.  Complex numbers are interleaved
 * (re, im) float64 pairs, matrices row-major.  Controls are laid out
 * u[b][k][j] (batch, control, slice), exactly like the gradient.
 *
 * Error convention (reference: ValueError / DimensionError for bad shapes,
 * FloatingPointError for non-finite P, qoc.py:191-192, pauli.py:24-25):
 * every entry point returns an SQOC_* status; sqoc_last_error() gives the
 * message of the last failure on the calling thread.
 */
#ifndef SYMQOC_B200_H
#define SYMQOC_B200_H

#ifdef __cplusplus
extern "C" {
#endif

#define SQOC_ABI_VERSION 2

enum sqoc_status {
  SQOC_OK = 0,
  SQOC_ERR_ARG = 1,         /* bad argument / shape  (-> ValueError)          */
  SQOC_ERR_NONFINITE = 2,   /* non-finite F or grad  (-> FloatingPointError)  */
  SQOC_ERR_CUDA = 3,        /* CUDA runtime failure  (-> RuntimeError)        */
  SQOC_ERR_UNSUPPORTED = 4, /* block size / feature not built (-> RuntimeError) */
  SQOC_ERR_NCCL = 5         /* collective failure    (-> RuntimeError)        */
};

enum sqoc_objective {
  SQOC_OBJ_STATE = 0, /* tau_b = <psi_f|X_N|psi_0>, F = sum_b w_b |tau_b|^2          */
  SQOC_OBJ_GATE = 1   /* tau_b = Tr(V_b^dag X_N),   F = sum_b w_b |tau_b|^2, w_b default 1/(N_B d_b^2) */
};

enum sqoc_memory {
  SQOC_MEM_HOST = 0,  /* u / F / grad / tau are host pointers (copies inside the call) */
  SQOC_MEM_DEVICE = 1 /* u / F / grad / tau are device pointers on the problem's GPU   */
};

typedef struct sqoc_problem sqoc_problem;

/* Upload one problem (setup, once): per-block generators and targets.
 *   dims[b]            block dimension d_b
 *   h0[b]              d_b x d_b complex (2 d_b^2 doubles), Hermitian
 *   hk[b]              n_controls consecutive d_b x d_b complex matrices
 *   initial[b]         state objective: psi_0 (2 d_b doubles); gate: NULL
 *   target[b]          state: psi_f (2 d_b doubles); gate: V_b (2 d_b^2 doubles)
 *   weights            n_blocks doubles, or NULL for the objective's default
 *   n_slices, dt       piecewise-constant grid (TimeGrid, propagate.py:25-41)
 *   max_batch          largest batch passed to sqoc_eval
 * Replaces: propagate.Backend.__init__ (propagate.py:59-86) as the owner of
 * the dense per-block matrices. */
int sqoc_create(sqoc_problem** out, int device, int n_blocks, const int* dims, int n_controls,
                const double* const* h0, const double* const* hk, int objective,
                const double* const* initial, const double* const* target, const double* weights,
                int n_slices, double dt, int max_batch);

/* One fidelity+gradient evaluation for `batch` control vectors.
 *   u      [batch][n_controls][n_slices]
 *   F      [batch]                          (may be NULL)
 *   grad   [batch][n_controls][n_slices]    (may be NULL)
 *   tau    [batch][n_blocks][2]             (may be NULL) per-block complex overlaps
 *   stream cudaStream_t (NULL = legacy default stream)
 * Blocking: returns after the results are complete (and copied for SQOC_MEM_HOST).
 * Replaces: qoc.gradient (qoc.py:137-168) and qoc.objective (qoc.py:93-95). */
int sqoc_eval(sqoc_problem* p, const double* u, int batch, double* F, double* grad, double* tau,
              int memory, void* stream);

/* Optional tighter norm bounds for the propagator plan: bounds[b * (n_controls+1) + k]
 * >= ||H_k,b||_2 (k = 0 is H0).  A_j = -i dt (H0 + sum_k u_kj H_k) is normal, so
 * dt (||H0||_2 + sum_k |u_kj| ||H_k||_2) bounds ||A_j||_2 and the Taylor truncation
 * error rigorously.  Without this call the plan uses infinity-norms (also rigorous,
 * looser: more products per slice). */
int sqoc_set_norm_bounds(sqoc_problem* p, const double* bounds);

/* Large-block schedule: -1 auto (default), 0 slice-sequential (no history; memory
 * O(sum d_b^2)), 1 history (all slices resident, slice-batched GEMMs; memory
 * O(N sum d_b^2)), 2 state-vector (state objective only: U_j history, psi/chi
 * sweeps and an augmented Taylor action for the gradient; memory O(N sum d_b^2)),
 * 3 matrix-free (state objective only, opt-in: psi/chi sweeps by Taylor actions of A_j,
 * no propagator is formed; memory O(N sum d_b)).
 * sqoc_last_schedule reports what the last sqoc_eval used (-1 = no large blocks). */
int sqoc_set_schedule(sqoc_problem* p, int schedule);
int sqoc_last_schedule(const sqoc_problem* p);

/* Tiny-block (d <= 16) schedule: -1 auto (default: slice-parallel for batch <= 16, fused
 * otherwise), 0 fused (one lane group per problem runs every slice on chip), 1 slice-parallel
 * (a lane group per (problem, slice) for the propagators and the Frechet chains; only the
 * X / Lambda recurrences are sequential -- the latency path for single evaluations). */
int sqoc_set_tiny_schedule(sqoc_problem* p, int schedule);
int sqoc_last_tiny_schedule(const sqoc_problem* p);

/* Fused tiny schedule, histories kept in device memory between the forward and backward sweeps:
 * 0 none (the backward sweep recomputes X_{j-1} = U_j^dag X_j and re-runs the full forward-mode
 * pairs), 1 X history (X_{j-1} of every slice; the Frechet chain is seeded with
 * X_{j-1} Lam_j^dag: two GEMM-units per slice fewer), 2 X + chain history (also the propagator
 * chain A2, A3, Z, Y of every slice: only the derivative halves of the pairs run, four more units
 * fewer).  -1 auto (default): X histories when they fit in 40% of free memory, chain histories
 * for the largest blocks first while the total stays within 88%.
 * sqoc_last_tiny_history reports the highest level the last fused evaluation used (-1 none). */
int sqoc_set_tiny_history(sqoc_problem* p, int mode);
int sqoc_last_tiny_history(const sqoc_problem* p);

/* Fused tiny kernel: warps per CTA.  -1 auto (default: 4-warp CTAs when the problem has a single
 * tiny block -- several CTAs per SM, a shorter tail; one CTA filling an SM otherwise, which packs
 * the concurrent block kernels best), 0 always full, > 0 a cap. */
int sqoc_set_tiny_cta_warps(sqoc_problem* p, int warps);

/* Propagator plan of the last large-block evaluation: Taylor degree of the product scheme
 * (12: 4 products, 18: 5 products), `squarings` squarings, and the number of
 * augmented-action terms (state-vector). */
int sqoc_last_plan(const sqoc_problem* p, int* taylor_degree, int* squarings, int* action_terms);

/* Slice-chunk sharding of ONE evaluation over ranks (multi-GPU scan carry).
 * Replaces the reference's strictly sequential slice loops (qoc.py:128-134 forward, :156-167
 * backward) by P contiguous chunks.  A rank builds the problem for its own slice range [s, e)
 * (n_slices = e - s, the same dt; any subset of the blocks, weights of the full problem), then:
 *   sqoc_chunk_size     : length in doubles of one packed chunk product (sum_b 2 d_b^2);
 *   sqoc_chunk_forward  : packed[...] = C_b = U_{e-1} ... U_s of every block, block order,
 *                         each d_b x d_b complex row-major (the forward sweep of the chunk);
 *   (the caller all-gathers the packed products of the P chunks into gathered[P][...],
 *    e.g. ncclAllGather on device buffers -- the only data that crosses GPUs)
 *   sqoc_chunk_backward : on the device, the boundary values of chunk c from gathered:
 *                         gate  X_end = C_c .. C_0, Lam_end = C_{c+1}^dag .. C_{P-1}^dag V_b,
 *                         state psi_start = C_{c-1} .. C_0 psi_0, chi_end = C_{c+1}^dag .. psi_f,
 *                         the full-grid tau_b, then the backward sweep of the chunk's slices only
 *                         (the forward is not repeated): F = sum_b w_b |tau_b|^2 over this
 *                         problem's blocks, grad [K][e - s], tau [n_blocks][2] (any may be NULL).
 * Call sqoc_chunk_backward after sqoc_chunk_forward with the same u.  Every block must be large
 * (d > 16); tiny blocks shard by batch instead (seed-DP).  `memory` applies to every array. */
int sqoc_chunk_size(const sqoc_problem* p, long long* n_doubles);
int sqoc_chunk_forward(sqoc_problem* p, const double* u, double* packed, int memory, void* stream);
int sqoc_chunk_backward(sqoc_problem* p, const double* u, const double* gathered, int n_chunks, int chunk, double* F,
                        double* grad, double* tau, int memory, void* stream);
/* Last sqoc_chunk_backward: device time of the boundary-value formation (carry GEMMs + tau; needs
 * sqoc_set_timing) and the number of carry GEMM launches (each batched over the blocks). */
int sqoc_last_carry_stats(sqoc_problem* p, double* carry_ms, int* carry_gemms);

/* Complex GEMM algorithm of the large-block path (process-wide): 3 = Gauss/3M (three
 * real DMMA products per complex product, default), 4 = 4M (four).  Both are exact
 * algorithms; 3M rounds slightly differently (still ~1e-15 relative). */
int sqoc_set_complex_gemm(int mults);

/* Large-block 3M GEMM kernel (process-wide): 1 = persistent warp-specialised kernel, one CTA per SM,
 * a producer warp streaming TMA tensor-map loads into a 12-stage 128B-swizzled shared-memory ring
 * with full/empty mbarriers across tile boundaries (default); 0 = the per-tile kernel with per-thread
 * cp.async staging and a block barrier per K stage.  SQOC_GEMM_TMA=0/1 sets the initial mode. */
int sqoc_set_gemm_staging(int tma);
int sqoc_gemm_staging(void);

/* Free all device memory of the problem. */
int sqoc_destroy(sqoc_problem* p);

/* Single-block state-transfer gradient with the reference's exact signature
 * semantics: qoc.gradient(psi0, psi_f, bx, by, backend, tau) with
 * backend.h0/hx/hy dense d x d.  Host buffers; gx, gy [n_steps], P scalar. */
int sqoc_state_gradient(int device, int d, const double* h0, const double* hx, const double* hy,
                        const double* psi0, const double* psi_f, const double* bx, const double* by,
                        int n_steps, double tau, double* gx, double* gy, double* P);

/* Per-block device timing: when on, sqoc_eval records CUDA events around each
 * block's work on the stream that launches it; sqoc_block_time_ms returns the
 * last evaluation's duration for block `block` (large blocks share one group). */
int sqoc_set_timing(sqoc_problem* p, int on);
int sqoc_block_time_ms(const sqoc_problem* p, int block, double* ms);

/* Large-block GEMMs of the last sqoc_eval: device time of their launches (summed CUDA-event
 * pairs around every GEMM launch on the launching stream; 0 unless sqoc_set_timing was on),
 * complex multiply-adds issued (sum m n k over the work lists; tile padding not counted) and
 * the number of GEMM launches.  The DMMA pipe executes sqoc_complex_gemm_mults() real FMAs
 * (3 for Gauss/3M, 4 for 4M) per complex MAC. */
int sqoc_last_gemm_stats(sqoc_problem* p, double* gemm_ms, double* complex_macs, int* launches);
int sqoc_complex_gemm_mults(void);

/* Device kernel launches issued by the last sqoc_eval on this problem. */
int sqoc_last_launch_count(const sqoc_problem* p);

/* On-GPU D_n symmetry-adapted basis.  Builds, on `device`, the full
 * D_n block basis of n spins (3 <= n <= 16) with the reference's block order and column order
 * (adjoint._dn_full_projected, adjoint.py:198-220: irrep rows A1, A2, (B1, B2), E_k(j); each
 * row's matrix-element projector applied to Fock states, Gram-Schmidt with tolerance 1e-8,
 * columns sorted by (Hamming weight, generating index)); every column is supported on one
 * D_n orbit.  The reference refuses n > 10 (adjoint.py:231-232).
 *   sqoc_basis_info     : number of blocks, dims[b], irrep row of each block
 *                         (0 A1, 1 A2, then B1, B2 for even n, then E_k rows j = 1, 2)
 *   sqoc_basis_nnz      : stored entries of block b's columns
 *   sqoc_basis_columns  : keys[i] = generating Fock index of column i, col_nnz[i] = its support size;
 *                         rows/vals = the support (ascending Fock index) and real entries, column by column
 *   sqoc_basis_compress : A_b^T H A_b for every block b (AdjointMatrix.compress, adjoint.py:61-64)
 *                         of H = sum_t coef_t P_t, P_t e_x = (-1)^popcount(x & sign[t]) e_{x ^ flip[t]}
 *                         (coef complex interleaved; a Pauli string with X/Y letters in flip, Z/Y letters
 *                         in sign and the factor i^#Y folded into coef); out[b] = d_b x d_b complex
 *                         host buffers.  Deterministic (one thread per block column, fixed order). */
typedef struct sqoc_basis sqoc_basis;
int sqoc_dn_basis_create(sqoc_basis** out, int device, int n);
int sqoc_basis_info(const sqoc_basis* b, int* n_blocks, int* dims, int* irrep_rows);
int sqoc_basis_nnz(const sqoc_basis* b, int block, long long* nnz);
int sqoc_basis_columns(const sqoc_basis* b, int block, int* keys, int* col_nnz, int* rows, double* vals);
int sqoc_basis_compress(const sqoc_basis* b, int n_terms, const int* flip, const int* sign, const double* coef,
                        double* const* out);
int sqoc_basis_destroy(sqoc_basis* b);

/* Trotterised per-qubit propagator (reference trotter.py:68-225).
 * Model (model.py:59-92, per-qubit controls): H = sum_i bz/2 Z_i + sum_k c_k/4 sum_i Z_i Z_{i+k}
 * + sum_i (bx_i X_i + by_i Y_i)/2 on n <= 12 spins, site 1 = most significant bit.
 *   sqoc_trotter_create  : PerQubitPlan(cfg, tau, strang) (trotter.py:77-114): coupling phases and
 *                          the exact-H diagonal precomputed on the device
 *   sqoc_trotter_apply   : n_steps Trotter steps (PerQubitPlan.apply_step, trotter.py:138-152) on the
 *                          rows of arr [2^n][cols] complex row-major (a state: cols = 1), in place;
 *                          controls bx, by [n_steps][n]
 *   sqoc_trotter_replay  : fidelity_replay (trotter.py:196-225): W <- U_trotter (W U_exact^dag) per
 *                          step from W = I, fids[r] = |Tr W|^2 / 4^n after every record_every-th step
 *                          and the last (ceil(n_steps / record_every) values)
 * `memory` applies to arr / bx / by / fids. */
typedef struct sqoc_trotter sqoc_trotter;
int sqoc_trotter_create(sqoc_trotter** out, int device, int n, double bz, const double* couplings, int n_couplings,
                        double tau, int strang);
int sqoc_trotter_apply(sqoc_trotter* t, double* arr, int cols, const double* bx, const double* by, int n_steps,
                       int memory, void* stream);
int sqoc_trotter_replay(sqoc_trotter* t, const double* bx, const double* by, int n_steps, int record_every,
                        double* fids, int memory, void* stream);
int sqoc_trotter_last_launches(const sqoc_trotter* t);
int sqoc_trotter_destroy(sqoc_trotter* t);

/* Largest block dimension the fused on-chip (tiny) path handles. */
int sqoc_tiny_max_dim(void);

const char* sqoc_last_error(void);
int sqoc_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SYMQOC_B200_H */
