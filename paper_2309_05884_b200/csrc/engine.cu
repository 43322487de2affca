// C-ABI implementation of the GRAPE fidelity+gradient engine (include/symqoc_b200.h).
//
// Host responsibilities: own the per-block generators / targets on the device,
// pick a kernel family per block (tiny fused kernel for d <= 16, batched-GEMM
// path for larger blocks), fork one stream per block off the caller's stream,
// and reduce per-block contributions in a fixed order (deterministic F / grad).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/symqoc_b200.h"
#include "devonce.h"
#include "large.cuh"
#include "tiny.cuh"

namespace sqoc {

static thread_local std::string g_last_error;

static int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
int report_error(int code, const std::string& msg) { return fail(code, msg); }  // other translation units

#define SQOC_CUDA(call)                                                                      \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess)                                                                   \
      return fail(SQOC_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));        \
  } while (0)

constexpr size_t kMaxSmem = 227 * 1024;

struct BlockPlan {
  int d = 0;
  bool tiny = false;
  double weight = 1.0;
  double2* gen = nullptr;     // (K+1) d*d, -i dt H
  double2* x0 = nullptr;      // state objective
  double2* target = nullptr;  // V or psi_f
  double2* park = nullptr;    // tiny: [slots][2][d*R]
  size_t park_slots = 0;
  double2* xhist = nullptr;   // tiny fused: [slots][N][d*R] X history (allocated on first use)
  double2* chist = nullptr;   // tiny fused: [slots][N][4][d*d] propagator-chain history
  int hist_level = -1;        // auto decision per block: 0 none, 1 X, 2 X + chain
  double2 *sp_U = nullptr, *sp_X = nullptr, *sp_L = nullptr;  // slice-parallel histories
  int sp_batch = 0;
  int nwarps = 1;       // fused kernel warps per CTA (capped by max_batch)
  int nwarps_max = 1;   // smem-limited warps per CTA
  cudaStream_t stream = nullptr;
  cudaEvent_t done = nullptr;
  cudaEvent_t t0 = nullptr, t1 = nullptr;  // per-block device timing (sqoc_set_timing)
};

}  // namespace sqoc

struct sqoc_problem {
  int device = 0;
  int nblocks = 0, K = 0, N = 0, objective = 0, max_batch = 0;
  double dt = 0.0;
  std::vector<sqoc::BlockPlan> blocks;
  double* u_dev = nullptr;      // [max_batch][K][N] staging for host-memory calls
  double* grad_dev = nullptr;   // [max_batch][K][N]
  double* gradb = nullptr;      // [nblocks][max_batch][K][N] per-block contributions
  double2* tau_dev = nullptr;   // [max_batch][nblocks]
  double* F_dev = nullptr;      // [max_batch]
  double* w_dev = nullptr;      // [nblocks]
  int* flag_dev = nullptr;      // non-finite flag
  int* flag_host = nullptr;     // pinned copy (the read-back does not serialise the result copies)
  cudaEvent_t fork = nullptr;
  sqoc::LargeGroup* large = nullptr;  // all blocks with d > kTinyMaxDim, advanced together
  cudaStream_t large_stream = nullptr;
  cudaEvent_t large_done = nullptr;
  cudaEvent_t large_t0 = nullptr, large_t1 = nullptr;
  bool timing = false;
  int tiny_mode = -1;  // -1 auto, 0 fused, 1 slice-parallel
  int last_tiny_mode = -1;
  int tiny_hist = -1;  // -1 auto, 0 off, 1 X history, 2 X + chain history
  int tiny_cta = -1;   // fused-kernel warps per CTA: -1 auto, 0 full (one CTA fills an SM), > 0 cap
  int last_tiny_hist = -1;
  bool hist_planned = false;  // auto levels decided (once, from free memory)
  int launches = 0;
};

namespace sqoc {

// ---------------------------------------------------------------- finalize
__global__ void finalize_kernel(int batch, int nblocks, int KN, const double2* __restrict__ tau,
                                const double* __restrict__ w, const double* __restrict__ gradb,
                                size_t gradb_stride, double* __restrict__ F, double* __restrict__ grad,
                                int* flag) {
  const size_t total = (size_t)batch * KN;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    double g = 0.0;
    for (int b = 0; b < nblocks; ++b) g += gradb[b * gradb_stride + i];
    if (!isfinite(g)) atomicOr(flag, 1);
    grad[i] = g;
  }
  for (size_t s = blockIdx.x * (size_t)blockDim.x + threadIdx.x; s < (size_t)batch; s += (size_t)gridDim.x * blockDim.x) {
    double f = 0.0;
    for (int b = 0; b < nblocks; ++b) {
      const double2 t = tau[s * nblocks + b];
      f += w[b] * (t.x * t.x + t.y * t.y);
    }
    if (!isfinite(f)) atomicOr(flag, 1);
    F[s] = f;
  }
}

// ---------------------------------------------------------------- tiny dispatch
enum TinyKernel { TK_FUSED = 0, TK_SP_EXPM = 1, TK_SP_SWEEP = 2, TK_SP_GRAD = 3 };

template <int D, bool GATE>
static int launch_tiny_t(int which, const TinySliceParams& sp, int grid, int nwarps, size_t smem, cudaStream_t st) {
  static std::mutex mu;
  static uint64_t done = 0;
  SQOC_CUDA(once_per_device(mu, done, [] {
    const cudaFuncAttribute a = cudaFuncAttributeMaxDynamicSharedMemorySize;
    cudaError_t e = cudaFuncSetAttribute(grape_tiny_kernel<D, GATE>, a, (int)kMaxSmem);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(tiny_sp_expm_kernel<D, GATE>, a, (int)kMaxSmem);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(tiny_sp_sweep_kernel<D, GATE>, a, (int)kMaxSmem);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(tiny_sp_grad_kernel<D, GATE>, a, (int)kMaxSmem);
    return e;
  }));
  switch (which) {
    case TK_FUSED: grape_tiny_kernel<D, GATE><<<grid, nwarps * 32, smem, st>>>(sp.p); break;
    case TK_SP_EXPM: tiny_sp_expm_kernel<D, GATE><<<grid, nwarps * 32, smem, st>>>(sp); break;
    case TK_SP_SWEEP: tiny_sp_sweep_kernel<D, GATE><<<grid, nwarps * 32, smem, st>>>(sp); break;
    default: tiny_sp_grad_kernel<D, GATE><<<grid, nwarps * 32, smem, st>>>(sp); break;
  }
  SQOC_CUDA(cudaGetLastError());
  return SQOC_OK;
}

template <bool GATE>
static int launch_tiny(int d, int which, const TinySliceParams& sp, int grid, int nwarps, size_t smem,
                       cudaStream_t st) {
  switch (d) {
#define SQOC_CASE(D) \
  case D:            \
    return launch_tiny_t<D, GATE>(which, sp, grid, nwarps, smem, st);
    SQOC_CASE(1) SQOC_CASE(2) SQOC_CASE(3) SQOC_CASE(4) SQOC_CASE(5) SQOC_CASE(6) SQOC_CASE(7) SQOC_CASE(8)
    SQOC_CASE(9) SQOC_CASE(10) SQOC_CASE(11) SQOC_CASE(12) SQOC_CASE(13) SQOC_CASE(14) SQOC_CASE(15) SQOC_CASE(16)
#undef SQOC_CASE
    default:
      return fail(SQOC_ERR_UNSUPPORTED, "tiny path supports d <= 16");
  }
}

constexpr double kChainBudget = 0.88;  // fraction of free device memory the tiny histories may take

static int choose_nwarps(int d, int K, int batch, bool mma, int max_warps = kTinyMaxWarps) {
  const int pg = 32 / tiny_lanes(d, mma);
  const int need = (batch + pg - 1) / pg;
  int nw = max_warps;
  while (nw > 1 && tiny_smem_bytes(d, K, nw, mma) > kMaxSmem) --nw;
  return std::max(1, std::min(nw, need));
}

static std::vector<double2> to_generator(const double* h, int d, double dt) {
  // a = -i dt H : (x + i y) -> (dt y) - i (dt x)
  std::vector<double2> a((size_t)d * d);
  for (size_t i = 0; i < a.size(); ++i) a[i] = make_double2(dt * h[2 * i + 1], -dt * h[2 * i]);
  return a;
}

static void free_problem(sqoc_problem* p) {
  if (!p) return;
  cudaSetDevice(p->device);
  for (auto& b : p->blocks) {
    cudaFree(b.gen);
    cudaFree(b.x0);
    cudaFree(b.target);
    cudaFree(b.park);
    cudaFree(b.xhist);
    cudaFree(b.chist);
    cudaFree(b.sp_U);
    cudaFree(b.sp_X);
    cudaFree(b.sp_L);
    if (b.stream) cudaStreamDestroy(b.stream);
    if (b.done) cudaEventDestroy(b.done);
    if (b.t0) cudaEventDestroy(b.t0);
    if (b.t1) cudaEventDestroy(b.t1);
  }
  cudaFree(p->u_dev);
  cudaFree(p->grad_dev);
  cudaFree(p->gradb);
  cudaFree(p->tau_dev);
  cudaFree(p->F_dev);
  cudaFree(p->w_dev);
  cudaFree(p->flag_dev);
  cudaFreeHost(p->flag_host);
  if (p->fork) cudaEventDestroy(p->fork);
  if (p->large) {
    large_free(*p->large);
    delete p->large;
  }
  if (p->large_stream) cudaStreamDestroy(p->large_stream);
  if (p->large_done) cudaEventDestroy(p->large_done);
  if (p->large_t0) cudaEventDestroy(p->large_t0);
  if (p->large_t1) cudaEventDestroy(p->large_t1);
  delete p;
}

}  // namespace sqoc

using namespace sqoc;

extern "C" {

const char* sqoc_last_error(void) { return g_last_error.c_str(); }
int sqoc_abi_version(void) { return SQOC_ABI_VERSION; }
int sqoc_tiny_max_dim(void) { return kTinyMaxDim; }
int sqoc_last_launch_count(const sqoc_problem* p) { return p ? p->launches : 0; }

int sqoc_create(sqoc_problem** out, int device, int n_blocks, const int* dims, int n_controls,
                const double* const* h0, const double* const* hk, int objective,
                const double* const* initial, const double* const* target, const double* weights,
                int n_slices, double dt, int max_batch) {
  if (!out) return fail(SQOC_ERR_ARG, "out is NULL");
  *out = nullptr;
  if (n_blocks < 1 || !dims || !h0 || !hk || !target) return fail(SQOC_ERR_ARG, "missing block arrays");
  if (n_controls < 1 || n_controls > kMaxControls) return fail(SQOC_ERR_ARG, "n_controls must be in 1..4");
  if (objective != SQOC_OBJ_STATE && objective != SQOC_OBJ_GATE) return fail(SQOC_ERR_ARG, "unknown objective");
  if (objective == SQOC_OBJ_STATE && !initial) return fail(SQOC_ERR_ARG, "state objective needs initial states");
  if (n_slices < 0 || max_batch < 1 || !(dt > 0.0) || !std::isfinite(dt)) return fail(SQOC_ERR_ARG, "bad grid or batch");
  for (int b = 0; b < n_blocks; ++b)
    if (dims[b] < 1) return fail(SQOC_ERR_ARG, "block dimension must be >= 1");

  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return fail(SQOC_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  sqoc_problem* p = new sqoc_problem();
  p->device = device;
  p->nblocks = n_blocks;
  p->K = n_controls;
  p->N = n_slices;
  p->objective = objective;
  p->max_batch = max_batch;
  p->dt = dt;
  p->blocks.resize(n_blocks);
  const size_t KN = (size_t)n_controls * n_slices;
  std::vector<double> w(n_blocks);
  std::vector<LargeBlockSpec> large_specs;
  int rc = SQOC_OK;
  auto chk = [&](cudaError_t ce, const char* what) {
    if (ce != cudaSuccess && rc == SQOC_OK) rc = fail(SQOC_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(ce));
  };
  for (int b = 0; b < n_blocks && rc == SQOC_OK; ++b) {
    BlockPlan& bp = p->blocks[b];
    const int d = dims[b];
    bp.d = d;
    bp.tiny = d <= kTinyMaxDim;
    w[b] = weights ? weights[b]
                   : (objective == SQOC_OBJ_GATE ? 1.0 / ((double)n_blocks * d * d) : 1.0);
    std::vector<double2> g;
    g.reserve((size_t)(n_controls + 1) * d * d);
    auto a0 = to_generator(h0[b], d, dt);
    g.insert(g.end(), a0.begin(), a0.end());
    for (int k = 0; k < n_controls; ++k) {
      auto ak = to_generator(hk[b] + (size_t)k * 2 * d * d, d, dt);
      g.insert(g.end(), ak.begin(), ak.end());
    }
    chk(cudaMalloc(&bp.gen, g.size() * sizeof(double2)), "cudaMalloc gen");
    if (rc) break;
    chk(cudaMemcpy(bp.gen, g.data(), g.size() * sizeof(double2), cudaMemcpyHostToDevice), "copy gen");
    const size_t tsz = (objective == SQOC_OBJ_GATE ? (size_t)d * d : (size_t)d) * sizeof(double2);
    chk(cudaMalloc(&bp.target, tsz), "cudaMalloc target");
    if (rc) break;
    chk(cudaMemcpy(bp.target, target[b], tsz, cudaMemcpyHostToDevice), "copy target");
    if (objective == SQOC_OBJ_STATE) {
      chk(cudaMalloc(&bp.x0, d * sizeof(double2)), "cudaMalloc x0");
      if (rc) break;
      chk(cudaMemcpy(bp.x0, initial[b], d * sizeof(double2), cudaMemcpyHostToDevice), "copy x0");
    }
    {
      // Longest-first CTA dispatch among the concurrent block kernels: the larger the block, the
      // higher its stream priority (distinct larger dims ranked; ties share a level).
      int least = 0, greatest = 0;
      cudaDeviceGetStreamPriorityRange(&least, &greatest);
      std::vector<int> larger;
      for (int o = 0; o < n_blocks; ++o)
        if (dims[o] > d && std::find(larger.begin(), larger.end(), dims[o]) == larger.end()) larger.push_back(dims[o]);
      const int prio = std::min(least, greatest + (int)larger.size());
      chk(cudaStreamCreateWithPriority(&bp.stream, cudaStreamNonBlocking, prio), "stream");
    }
    chk(cudaEventCreateWithFlags(&bp.done, cudaEventDisableTiming), "event");
    chk(cudaEventCreate(&bp.t0), "event");
    chk(cudaEventCreate(&bp.t1), "event");
    if (bp.tiny) {
      const int R = objective == SQOC_OBJ_GATE ? d : 1;
      const int pg = 32 / tiny_lanes(d, tiny_mma(d));
      // r01: 24 warps for the <= 80-register instantiations beat 12 in the concurrent cfg 1 step
      // (212.8 vs 215.6 ms) although each sector alone is slower (fewer, larger CTAs)
      bp.nwarps = choose_nwarps(d, n_controls, max_batch, tiny_mma(d), tiny_fused_max_warps(d));
      // One CTA fills an SM (12 or 8 warps).  r01: 4-warp CTAs (3 per SM) run the d = 13 sector alone
      // in 79.0 instead of 90.7 ms (shorter tail) but spend 10% more active SM time (77.3 vs 69.9
      // SM-ms: SMs partly filled between CTAs), so the concurrent cfg 1 step slows to 212.9 ms.
      bp.nwarps_max = choose_nwarps(d, n_controls, 1 << 30, false);
      const int per_cta = pg * bp.nwarps;
      // room for any CTA size up to per_cta (sqoc_set_tiny_cta_warps): the last CTA's padding slots
      bp.park_slots = (size_t)((max_batch + per_cta - 1) / per_cta) * per_cta + per_cta;
      chk(cudaMalloc(&bp.park, bp.park_slots * 2 * d * R * sizeof(double2)), "cudaMalloc park");
    } else {
      LargeBlockSpec ls{};
      ls.global_index = b;
      ls.d = d;
      ls.gen = bp.gen;
      ls.x0 = bp.x0;
      ls.target = bp.target;
      ls.weight = w[b];
      for (int k = 0; k <= n_controls; ++k) {  // inf-norm of a_k (max row sum of |re| + |im|)
        double best = 0.0;
        for (int i = 0; i < d; ++i) {
          double rs = 0.0;
          for (int c = 0; c < d; ++c) {
            const double2 z = g[(size_t)k * d * d + (size_t)i * d + c];
            rs += std::fabs(z.x) + std::fabs(z.y);
          }
          best = std::max(best, rs);
        }
        ls.gen_norm[k] = best;
      }
      // union pattern of a_0..a_K (exact nonzeros; no threshold) and the values on it
      ls.sp_rp.assign(d + 1, 0);
      for (int i = 0; i < d; ++i) {
        for (int c = 0; c < d; ++c) {
          bool nz = false;
          for (int k = 0; k <= n_controls && !nz; ++k) {
            const double2 z = g[(size_t)k * d * d + (size_t)i * d + c];
            nz = z.x != 0.0 || z.y != 0.0;
          }
          if (nz) ls.sp_ci.push_back(c);
        }
        ls.sp_rp[i + 1] = (int)ls.sp_ci.size();
      }
      const size_t nnz = ls.sp_ci.size();
      ls.sp_gv.resize((size_t)(n_controls + 1) * nnz);
      for (int k = 0; k <= n_controls; ++k)
        for (int i = 0; i < d; ++i)
          for (int e = ls.sp_rp[i]; e < ls.sp_rp[i + 1]; ++e)
            ls.sp_gv[(size_t)k * nnz + e] = g[(size_t)k * d * d + (size_t)i * d + ls.sp_ci[e]];
      large_specs.push_back(ls);
    }
  }
  if (rc == SQOC_OK && !large_specs.empty()) {
    p->large = new LargeGroup();
    int lrc = large_init(*p->large, large_specs, n_controls, n_slices, objective == SQOC_OBJ_GATE);
    if (lrc != SQOC_OK) rc = fail(lrc, p->large->err);
    chk(cudaStreamCreateWithFlags(&p->large_stream, cudaStreamNonBlocking), "stream");
    chk(cudaEventCreateWithFlags(&p->large_done, cudaEventDisableTiming), "event");
    chk(cudaEventCreate(&p->large_t0), "event");
    chk(cudaEventCreate(&p->large_t1), "event");
  }
  if (rc == SQOC_OK) {
    chk(cudaMalloc(&p->u_dev, std::max<size_t>(1, max_batch * KN) * sizeof(double)), "cudaMalloc u");
    chk(cudaMalloc(&p->grad_dev, std::max<size_t>(1, max_batch * KN) * sizeof(double)), "cudaMalloc grad");
    chk(cudaMalloc(&p->gradb, std::max<size_t>(1, n_blocks * max_batch * KN) * sizeof(double)), "cudaMalloc gradb");
    chk(cudaMalloc(&p->tau_dev, (size_t)max_batch * n_blocks * sizeof(double2)), "cudaMalloc tau");
    chk(cudaMalloc(&p->F_dev, max_batch * sizeof(double)), "cudaMalloc F");
    chk(cudaMalloc(&p->w_dev, n_blocks * sizeof(double)), "cudaMalloc w");
    chk(cudaMalloc(&p->flag_dev, sizeof(int)), "cudaMalloc flag");
    chk(cudaMallocHost(&p->flag_host, sizeof(int)), "cudaMallocHost flag");
    if (rc == SQOC_OK) chk(cudaMemcpy(p->w_dev, w.data(), n_blocks * sizeof(double), cudaMemcpyHostToDevice), "copy w");
    chk(cudaEventCreateWithFlags(&p->fork, cudaEventDisableTiming), "event");
    for (int b = 0; b < n_blocks; ++b) p->blocks[b].weight = w[b];
  }
  if (rc != SQOC_OK) {
    free_problem(p);
    return rc;
  }
  // setup copies come from pageable host memory (staged DMA on the legacy stream); evaluations run on
  // non-blocking streams that do not wait for it
  if (cudaDeviceSynchronize() != cudaSuccess) {
    free_problem(p);
    return report_error(SQOC_ERR_CUDA, "sqoc_create: device synchronisation failed");
  }
  *out = p;
  return SQOC_OK;
}

int sqoc_destroy(sqoc_problem* p) {
  free_problem(p);
  return SQOC_OK;
}

int sqoc_eval(sqoc_problem* p, const double* u, int batch, double* F, double* grad, double* tau, int memory,
              void* stream) {
  if (!p) return fail(SQOC_ERR_ARG, "problem is NULL");
  if (batch < 1 || batch > p->max_batch) return fail(SQOC_ERR_ARG, "batch outside 1..max_batch");
  if (memory != SQOC_MEM_HOST && memory != SQOC_MEM_DEVICE) return fail(SQOC_ERR_ARG, "unknown memory kind");
  if (!u && p->N > 0) return fail(SQOC_ERR_ARG, "u is NULL");
  SQOC_CUDA(cudaSetDevice(p->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t KN = (size_t)p->K * p->N;
  const bool dev = memory == SQOC_MEM_DEVICE;
  const double* u_dev = u;
  p->launches = 0;
  p->last_tiny_hist = -1;
  if (!dev && KN) {
    SQOC_CUDA(cudaMemcpyAsync(p->u_dev, u, batch * KN * sizeof(double), cudaMemcpyHostToDevice, st));
    u_dev = p->u_dev;
  }
  double* grad_dev = (dev && grad) ? grad : p->grad_dev;
  double* F_dev = (dev && F) ? F : p->F_dev;
  SQOC_CUDA(cudaMemsetAsync(p->flag_dev, 0, sizeof(int), st));
  SQOC_CUDA(cudaEventRecord(p->fork, st));
  const bool gate = p->objective == SQOC_OBJ_GATE;
  for (int b = 0; b < p->nblocks; ++b) {
    BlockPlan& bp = p->blocks[b];
    SQOC_CUDA(cudaStreamWaitEvent(bp.stream, p->fork, 0));
    double* gout = p->gradb + (size_t)b * p->max_batch * KN;
    if (p->N == 0) {
      // empty grid: X_N = X_0 (qoc.py test_empty_grid_gives_empty_gradient)
    }
    if (!bp.tiny) continue;
    if (p->timing) SQOC_CUDA(cudaEventRecord(bp.t0, bp.stream));
    {
      TinySliceParams sp{};
      TinyParams& tp = sp.p;
      tp.K = p->K;
      tp.N = p->N;
      tp.batch = batch;
      tp.gen = bp.gen;
      tp.x0 = bp.x0;
      tp.target = bp.target;
      tp.u = u_dev;
      tp.weight = bp.weight;
      tp.tau_out = p->tau_dev + b;
      tp.tau_stride = p->nblocks;
      tp.grad_out = gout;
      tp.park = bp.park;
      const size_t R = gate ? bp.d : 1;
      // slice-parallel latency path for small batches (every (problem, slice) its own lane group)
      const bool sp_mode = p->N > 0 && (p->tiny_mode == 1 || (p->tiny_mode == -1 && batch <= kTinySliceParallelMaxBatch));
      p->last_tiny_mode = sp_mode ? 1 : 0;
      if (sp_mode) p->last_tiny_hist = -1;
      int rc = SQOC_OK;
      if (sp_mode) {
        if (bp.sp_batch < batch) {
          cudaFree(bp.sp_U);
          cudaFree(bp.sp_X);
          cudaFree(bp.sp_L);
          bp.sp_U = bp.sp_X = bp.sp_L = nullptr;
          const int nb_alloc = std::max(batch, std::min(p->max_batch, kTinySliceParallelMaxBatch));
          SQOC_CUDA(cudaMalloc(&bp.sp_U, (size_t)nb_alloc * p->N * bp.d * bp.d * sizeof(double2)));
          SQOC_CUDA(cudaMalloc(&bp.sp_X, (size_t)nb_alloc * (p->N + 1) * bp.d * R * sizeof(double2)));
          SQOC_CUDA(cudaMalloc(&bp.sp_L, (size_t)nb_alloc * (p->N + 1) * bp.d * R * sizeof(double2)));
          bp.sp_batch = nb_alloc;
        }
        sp.Uh = bp.sp_U;
        sp.Xh = bp.sp_X;
        sp.Lh = bp.sp_L;
        sp.units = batch * p->N;
        const int pg = 32 / tiny_lanes(bp.d, false);
        // phases 1 and 3: lane group per (problem, slice); phase 2: per problem
        const int warps_units = (sp.units + pg - 1) / pg;
        const int nw = std::max(1, std::min(bp.nwarps_max, warps_units));
        tp.nwarps = nw;
        const size_t smem = tiny_smem_bytes(bp.d, p->K, nw, false);
        const int grid_units = (warps_units + nw - 1) / nw;
        const int warps_b = (batch + pg - 1) / pg;
        const int nw_b = 1;  // one warp per CTA: room for the sweep's U_j prefetch ring
        const int grid_b = warps_b;
        rc = gate ? launch_tiny<true>(bp.d, TK_SP_EXPM, sp, grid_units, nw, smem, bp.stream)
                  : launch_tiny<false>(bp.d, TK_SP_EXPM, sp, grid_units, nw, smem, bp.stream);
        if (rc == SQOC_OK) {
          TinySliceParams sp2 = sp;
          sp2.p.nwarps = nw_b;
          const size_t smem_b = tiny_sweep_smem_bytes(bp.d, p->K, nw_b);
          rc = gate ? launch_tiny<true>(bp.d, TK_SP_SWEEP, sp2, grid_b, nw_b, smem_b, bp.stream)
                    : launch_tiny<false>(bp.d, TK_SP_SWEEP, sp2, grid_b, nw_b, smem_b, bp.stream);
        }
        if (rc == SQOC_OK)
          rc = gate ? launch_tiny<true>(bp.d, TK_SP_GRAD, sp, grid_units, nw, smem, bp.stream)
                    : launch_tiny<false>(bp.d, TK_SP_GRAD, sp, grid_units, nw, smem, bp.stream);
        p->launches += 3;
      } else {
        const int pg = 32 / tiny_lanes(bp.d, tiny_mma(bp.d));
        // auto: a problem with a single tiny block launches 4-warp CTAs (several per SM: a shorter
        // tail -- r01 d = 13 alone 79.0 vs 90.7 ms); with several blocks one CTA fills an SM, which
        // packs the concurrent sector kernels best (r01 cfg 1: 198 vs 213 ms with 4-warp CTAs)
        int ntiny = 0;
        for (auto& ob : p->blocks) ntiny += ob.tiny;
        const int cap = p->tiny_cta > 0 ? p->tiny_cta : (p->tiny_cta == -1 && ntiny == 1) ? 4 : bp.nwarps;
        int nw = std::max(1, std::min(std::min(bp.nwarps, cap), (batch + pg - 1) / pg));
        tp.nwarps = nw;
        if (!p->hist_planned) {
          // auto: X histories of all tiny blocks if they fit in 40% of free memory, then chain
          // histories for the largest blocks first while the total stays within kChainBudget
          // (cfg 1: 149 GB for all seven sectors, 84% of a free B200)
          size_t free_b = 0, total_b = 0, used = 0;
          SQOC_CUDA(cudaMemGetInfo(&free_b, &total_b));
          for (auto& ob : p->blocks)
            if (ob.tiny) used += ob.park_slots * p->N * ob.d * (gate ? ob.d : 1) * sizeof(double2);
          const bool x_ok = used <= (size_t)(0.4 * (double)free_b);
          std::vector<int> order;
          for (int i = 0; i < p->nblocks; ++i)
            if (p->blocks[i].tiny) order.push_back(i);
          std::sort(order.begin(), order.end(), [&](int a, int b) { return p->blocks[a].d > p->blocks[b].d; });
          for (int i : order) {
            BlockPlan& ob = p->blocks[i];
            ob.hist_level = x_ok ? 1 : 0;
            const size_t cb = ob.park_slots * p->N * 4 * ob.d * ob.d * sizeof(double2);
            if (x_ok && used + cb <= (size_t)(kChainBudget * (double)free_b)) {
              ob.hist_level = 2;
              used += cb;
            }
          }
          p->hist_planned = true;
        }
        int level = p->N == 0 ? 0 : p->tiny_hist >= 0 ? p->tiny_hist : bp.hist_level;
        // histories are an optimisation: if the device cannot hold them, run with less history
        if (level >= 1 && !bp.xhist &&
            cudaMalloc(&bp.xhist, bp.park_slots * p->N * bp.d * R * sizeof(double2)) != cudaSuccess) {
          (void)cudaGetLastError();
          bp.xhist = nullptr;
          bp.hist_level = level = 0;
        }
        if (level >= 2 && !bp.chist &&
            cudaMalloc(&bp.chist, bp.park_slots * p->N * 4 * bp.d * bp.d * sizeof(double2)) != cudaSuccess) {
          (void)cudaGetLastError();
          bp.chist = nullptr;
          bp.hist_level = level = 1;
        }
        tp.xhist = level >= 1 ? bp.xhist : nullptr;
        tp.chist = level >= 2 ? bp.chist : nullptr;
        p->last_tiny_hist = std::max(p->last_tiny_hist, level);
        const int grid = (batch + pg * nw - 1) / (pg * nw);
        const size_t smem = tiny_smem_bytes(bp.d, p->K, nw, tiny_mma(bp.d));
        rc = gate ? launch_tiny<true>(bp.d, TK_FUSED, sp, grid, nw, smem, bp.stream)
                  : launch_tiny<false>(bp.d, TK_FUSED, sp, grid, nw, smem, bp.stream);
        p->launches += 1;
      }
      if (rc != SQOC_OK) return rc;
    }
    if (p->timing) SQOC_CUDA(cudaEventRecord(bp.t1, bp.stream));
    SQOC_CUDA(cudaEventRecord(bp.done, bp.stream));
    SQOC_CUDA(cudaStreamWaitEvent(st, bp.done, 0));
  }
  if (p->large) {
    SQOC_CUDA(cudaStreamWaitEvent(p->large_stream, p->fork, 0));
    LargeArgs la;
    la.u = u_dev;
    la.batch = batch;
    la.tau_out = p->tau_dev;
    la.tau_stride = p->nblocks;
    la.gradb = p->gradb;
    la.gradb_block_stride = (size_t)p->max_batch * KN;
    if (p->timing) SQOC_CUDA(cudaEventRecord(p->large_t0, p->large_stream));
    int rc = large_eval(*p->large, la, p->large_stream);
    if (rc != SQOC_OK) return fail(rc, p->large->err);
    if (p->timing) SQOC_CUDA(cudaEventRecord(p->large_t1, p->large_stream));
    p->launches += p->large->launches;
    SQOC_CUDA(cudaEventRecord(p->large_done, p->large_stream));
    SQOC_CUDA(cudaStreamWaitEvent(st, p->large_done, 0));
  }
  {
    const size_t total = std::max<size_t>(batch * KN, batch);
    const int threads = 256;
    const int grid = (int)std::min<size_t>((total + threads - 1) / threads, 148 * 8);
    finalize_kernel<<<std::max(grid, 1), threads, 0, st>>>(batch, p->nblocks, (int)KN, p->tau_dev, p->w_dev,
                                                           p->gradb, (size_t)p->max_batch * KN, F_dev, grad_dev,
                                                           p->flag_dev);
    SQOC_CUDA(cudaGetLastError());
    p->launches += 1;
  }
  *p->flag_host = 0;
  SQOC_CUDA(cudaMemcpyAsync(p->flag_host, p->flag_dev, sizeof(int), cudaMemcpyDeviceToHost, st));
  if (!dev) {
    if (F) SQOC_CUDA(cudaMemcpyAsync(F, F_dev, batch * sizeof(double), cudaMemcpyDeviceToHost, st));
    if (grad && KN) SQOC_CUDA(cudaMemcpyAsync(grad, grad_dev, batch * KN * sizeof(double), cudaMemcpyDeviceToHost, st));
    if (tau)
      SQOC_CUDA(cudaMemcpyAsync(tau, p->tau_dev, (size_t)batch * p->nblocks * sizeof(double2), cudaMemcpyDeviceToHost, st));
  } else if (tau) {
    SQOC_CUDA(cudaMemcpyAsync(tau, p->tau_dev, (size_t)batch * p->nblocks * sizeof(double2), cudaMemcpyDeviceToDevice, st));
  }
  SQOC_CUDA(cudaStreamSynchronize(st));
  if (*p->flag_host) return fail(SQOC_ERR_NONFINITE, "objective or gradient became non-finite");
  return SQOC_OK;
}

// ---------------------------------------------------------------- slice-chunk sharding
static int chunk_checks(sqoc_problem* p, int memory) {
  if (!p) return fail(SQOC_ERR_ARG, "problem is NULL");
  if (memory != SQOC_MEM_HOST && memory != SQOC_MEM_DEVICE) return fail(SQOC_ERR_ARG, "unknown memory kind");
  if (!p->large) return fail(SQOC_ERR_UNSUPPORTED, "slice-chunk sharding needs large blocks (d > 16)");
  for (auto& b : p->blocks)
    if (b.tiny) return fail(SQOC_ERR_UNSUPPORTED, "slice-chunk sharding is not built for tiny blocks (use seed-DP)");
  return SQOC_OK;
}

int sqoc_chunk_size(const sqoc_problem* p, long long* n_doubles) {
  if (!p || !n_doubles) return fail(SQOC_ERR_ARG, "problem or n_doubles is NULL");
  long long n = 0;
  for (auto& b : p->blocks) n += 2LL * b.d * b.d;
  *n_doubles = n;
  return SQOC_OK;
}

int sqoc_chunk_forward(sqoc_problem* p, const double* u, double* packed, int memory, void* stream) {
  int rc = chunk_checks(p, memory);
  if (rc != SQOC_OK) return rc;
  if (!packed || (!u && p->N > 0)) return fail(SQOC_ERR_ARG, "u or packed is NULL");
  SQOC_CUDA(cudaSetDevice(p->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t KN = (size_t)p->K * p->N;
  const size_t total = p->large->total;
  const double* u_dev = u;
  double2* out = reinterpret_cast<double2*>(packed);
  if (memory == SQOC_MEM_HOST) {
    if (KN) SQOC_CUDA(cudaMemcpyAsync(p->u_dev, u, KN * sizeof(double), cudaMemcpyHostToDevice, st));
    u_dev = p->u_dev;
    SQOC_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&out), total * sizeof(double2), st));
  }
  LargeArgs la;
  la.u = u_dev;
  la.batch = 1;
  la.tau_out = p->tau_dev;
  la.tau_stride = p->nblocks;
  la.gradb = p->gradb;
  la.gradb_block_stride = (size_t)p->max_batch * KN;
  p->large->chunk_phase = 1;
  p->large->chunk_out = out;
  rc = large_eval(*p->large, la, st);
  p->large->chunk_phase = 0;
  p->large->chunk_out = nullptr;
  p->launches = p->large->launches;
  if (rc == SQOC_OK && memory == SQOC_MEM_HOST)
    SQOC_CUDA(cudaMemcpyAsync(packed, out, total * sizeof(double2), cudaMemcpyDeviceToHost, st));
  if (memory == SQOC_MEM_HOST) cudaFreeAsync(out, st);
  if (rc != SQOC_OK) return fail(rc, p->large->err);
  SQOC_CUDA(cudaStreamSynchronize(st));
  return SQOC_OK;
}

int sqoc_chunk_backward(sqoc_problem* p, const double* u, const double* gathered, int n_chunks, int chunk, double* F,
                        double* grad, double* tau, int memory, void* stream) {
  int rc = chunk_checks(p, memory);
  if (rc != SQOC_OK) return rc;
  if (!gathered) return fail(SQOC_ERR_ARG, "gathered is NULL");
  if (n_chunks < 1 || chunk < 0 || chunk >= n_chunks) return fail(SQOC_ERR_ARG, "chunk outside 0..n_chunks-1");
  SQOC_CUDA(cudaSetDevice(p->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t total = p->large->total;
  const double2* in = reinterpret_cast<const double2*>(gathered);
  double2* staged = nullptr;
  if (memory == SQOC_MEM_HOST) {
    SQOC_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&staged), (size_t)n_chunks * total * sizeof(double2), st));
    SQOC_CUDA(cudaMemcpyAsync(staged, gathered, (size_t)n_chunks * total * sizeof(double2), cudaMemcpyHostToDevice,
                              st));
    in = staged;
  }
  p->large->chunk_phase = 2;
  p->large->chunk_in = in;
  p->large->chunk_P = n_chunks;
  p->large->chunk_c = chunk;
  rc = sqoc_eval(p, u, 1, F, grad, tau, memory, stream);
  p->large->chunk_phase = 0;
  p->large->chunk_in = nullptr;
  if (staged) {
    cudaFreeAsync(staged, st);
    cudaStreamSynchronize(st);
  }
  return rc;
}

int sqoc_last_carry_stats(sqoc_problem* p, double* carry_ms, int* carry_gemms) {
  if (!p || !carry_ms || !carry_gemms) return fail(SQOC_ERR_ARG, "NULL argument");
  *carry_ms = 0.0;
  *carry_gemms = 0;
  if (!p->large) return SQOC_OK;
  *carry_gemms = p->large->carry_gemms;
  if (p->timing) large_carry_time(*p->large, carry_ms);
  return SQOC_OK;
}

int sqoc_set_norm_bounds(sqoc_problem* p, const double* bounds) {
  if (!p || !bounds) return fail(SQOC_ERR_ARG, "problem or bounds is NULL");
  const int K1 = p->K + 1;
  for (int i = 0; i < p->nblocks * K1; ++i)
    if (!(bounds[i] >= 0.0) || !std::isfinite(bounds[i])) return fail(SQOC_ERR_ARG, "bounds must be finite and >= 0");
  if (p->large) {
    std::vector<double> gn;
    for (const auto& ls : p->large->blocks)
      for (int k = 0; k < K1; ++k) gn.push_back(p->dt * bounds[ls.global_index * K1 + k]);
    int rc = large_set_norms(*p->large, gn);
    if (rc != SQOC_OK) return fail(rc, p->large->err);
  }
  return SQOC_OK;
}

int sqoc_set_schedule(sqoc_problem* p, int schedule) {
  if (!p || schedule < -1 || schedule > 3) return fail(SQOC_ERR_ARG, "schedule must be -1 (auto), 0, 1, 2 or 3");
  if (schedule == 3 && p->objective != SQOC_OBJ_STATE) return fail(SQOC_ERR_ARG, "matrix-free needs the state objective");
  if (p->large) p->large->force_mode = schedule;
  return SQOC_OK;
}

int sqoc_last_schedule(const sqoc_problem* p) { return (p && p->large) ? p->large->mode : -1; }

int sqoc_set_tiny_schedule(sqoc_problem* p, int schedule) {
  if (!p || schedule < -1 || schedule > 1) return fail(SQOC_ERR_ARG, "tiny schedule must be -1, 0 or 1");
  p->tiny_mode = schedule;
  return SQOC_OK;
}

int sqoc_last_tiny_schedule(const sqoc_problem* p) { return p ? p->last_tiny_mode : -1; }

int sqoc_set_tiny_history(sqoc_problem* p, int mode) {
  if (!p || mode < -1 || mode > 2) return fail(SQOC_ERR_ARG, "tiny history mode must be -1, 0, 1 or 2");
  p->tiny_hist = mode;
  return SQOC_OK;
}

int sqoc_last_tiny_history(const sqoc_problem* p) { return p ? p->last_tiny_hist : -1; }

int sqoc_set_tiny_cta_warps(sqoc_problem* p, int warps) {
  if (!p || warps < -1 || warps > 32) return fail(SQOC_ERR_ARG, "tiny CTA warps must be -1, 0 or 1..32");
  p->tiny_cta = warps;
  return SQOC_OK;
}

int sqoc_last_plan(const sqoc_problem* p, int* taylor_degree, int* squarings, int* action_terms) {
  if (!p || !taylor_degree || !squarings || !action_terms) return fail(SQOC_ERR_ARG, "NULL argument");
  *taylor_degree = p->large ? p->large->last_degree : 0;
  *squarings = p->large ? p->large->last_s : 0;
  *action_terms = p->large ? p->large->last_taylor_terms : 0;
  return SQOC_OK;
}

int sqoc_set_complex_gemm(int mults) {
  if (large_set_complex_gemm(mults) != SQOC_OK) return fail(SQOC_ERR_ARG, "mults must be 3 or 4");
  return SQOC_OK;
}

int sqoc_set_timing(sqoc_problem* p, int on) {
  if (!p) return fail(SQOC_ERR_ARG, "problem is NULL");
  p->timing = on != 0;
  if (p->large) p->large->timing = p->timing;
  return SQOC_OK;
}

int sqoc_last_gemm_stats(sqoc_problem* p, double* gemm_ms, double* complex_macs, int* launches) {
  if (!p || !gemm_ms || !complex_macs || !launches) return fail(SQOC_ERR_ARG, "NULL argument");
  *gemm_ms = 0.0;
  *complex_macs = 0.0;
  *launches = 0;
  if (!p->large) return SQOC_OK;
  SQOC_CUDA(cudaSetDevice(p->device));
  *complex_macs = p->large->gemm_macs;
  *launches = p->large->gemm_launches;
  if (p->large->timing) {
    int rc = large_gemm_time(*p->large, gemm_ms);
    if (rc != SQOC_OK) return fail(rc, p->large->err);
  }
  return SQOC_OK;
}

int sqoc_complex_gemm_mults(void) { return large_complex_mults(); }

int sqoc_set_gemm_staging(int tma) {
  if (large_set_staging(tma) != SQOC_OK) return fail(SQOC_ERR_ARG, "staging must be 0 (cp.async), 1 or 2 (TMA)");
  return SQOC_OK;
}
int sqoc_gemm_staging(void) { return large_staging(); }

int sqoc_block_time_ms(const sqoc_problem* p, int block, double* ms) {
  if (!p || !ms || block < 0 || block >= p->nblocks) return fail(SQOC_ERR_ARG, "bad block index");
  const BlockPlan& bp = p->blocks[block];
  float t = 0.f;
  cudaError_t e = bp.tiny ? cudaEventElapsedTime(&t, bp.t0, bp.t1) : cudaEventElapsedTime(&t, p->large_t0, p->large_t1);
  if (e != cudaSuccess) return fail(SQOC_ERR_CUDA, std::string("cudaEventElapsedTime: ") + cudaGetErrorString(e));
  *ms = t;
  return SQOC_OK;
}

int sqoc_state_gradient(int device, int d, const double* h0, const double* hx, const double* hy,
                        const double* psi0, const double* psi_f, const double* bx, const double* by,
                        int n_steps, double tau, double* gx, double* gy, double* P) {
  if (d < 1 || !h0 || !hx || !hy || !psi0 || !psi_f || n_steps < 0) return fail(SQOC_ERR_ARG, "bad arguments");
  if (n_steps > 0 && !(tau > 0.0)) return fail(SQOC_ERR_ARG, "tau must be > 0");
  std::vector<double> hk((size_t)4 * d * d);
  std::memcpy(hk.data(), hx, sizeof(double) * 2 * d * d);
  std::memcpy(hk.data() + 2 * (size_t)d * d, hy, sizeof(double) * 2 * d * d);
  const double* h0s[1] = {h0};
  const double* hks[1] = {hk.data()};
  const double* ini[1] = {psi0};
  const double* tgt[1] = {psi_f};
  const double w = 1.0;
  sqoc_problem* p = nullptr;
  int rc = sqoc_create(&p, device, 1, &d, 2, h0s, hks, SQOC_OBJ_STATE, ini, tgt, &w, n_steps,
                       n_steps > 0 ? tau : 1.0, 1);
  if (rc != SQOC_OK) return rc;
  std::vector<double> u((size_t)2 * n_steps), g((size_t)2 * n_steps);
  for (int j = 0; j < n_steps; ++j) {
    u[j] = bx[j];
    u[n_steps + j] = by[j];
  }
  double F = 0.0;
  rc = sqoc_eval(p, u.data(), 1, &F, g.data(), nullptr, SQOC_MEM_HOST, nullptr);
  if (rc == SQOC_OK) {
    for (int j = 0; j < n_steps; ++j) {
      gx[j] = g[j];
      gy[j] = g[n_steps + j];
    }
    *P = F;
  }
  std::string keep = g_last_error;
  sqoc_destroy(p);
  g_last_error = keep;
  return rc;
}

}  // extern "C"
