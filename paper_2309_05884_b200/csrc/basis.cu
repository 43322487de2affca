// On-GPU D_n symmetry-adapted basis and block compression.
//
// Restates, on the device, the reference's full D_n adjoint builder
//   adjoint._dn_full_projected   (pkg/src/symqoc/adjoint.py:198-220)
//   groups.build_projector       (pkg/src/symqoc/groups.py:331-349)
//   AdjointMatrix.compress       (pkg/src/symqoc/adjoint.py:61-64)
// in the orbit-local form of paper_2309_05884_b200/symmetry.py (the host restatement that the
// tests pin to the reference at n = 6, 8, 10):
//   * orbit_kernel: one thread per Fock state x computes its 2n dihedral images (fock_map of
//     rotations r^m and reflections s r^m, groups.py:104-116), the orbit representative (the
//     minimum), the orbit size and x's position inside its ascending orbit;
//   * project_kernel: one warp per (irrep row, orbit): lane l holds entry l of the projected
//     vector P e_x = (dim/|G|) sum_g A_jj(g) e_{g x} for every member x in ascending order
//     (the element sum accumulates in element order, as the reference's csr sum / bincount),
//     Gram-Schmidt against the vectors already kept on this orbit (rank tolerance 1e-8,
//     adjoint.py:24), kept vectors normalised -- orbits have disjoint support, so this is the
//     reference's global Gram-Schmidt;
//   * the host sorts each row's kept vectors by (Hamming weight, generating index) -- the
//     reference's column order -- and uploads column tables;
//   * compress_kernel: one thread per block column c computes column c of A_b^T H A_b for a
//     Pauli sum H (terms: flip mask, sign mask, complex coefficient), sequentially in a fixed
//     order (deterministic, no atomics): for every member x of c's orbit and every term,
//     y = x ^ flip, and the contribution lands on the block's columns that live on y's orbit.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "../../include/symqoc_b200.h"

namespace sqoc {
int report_error(int code, const std::string& msg);  // engine.cu (sqoc_last_error)
}
using sqoc::report_error;

namespace {

constexpr double kGsRankTol = 1e-8;  // adjoint.py:24
constexpr int kMaxBasisQubits = 16;  // orbit size <= 2n <= 32: one lane per orbit entry

#define BASIS_CUDA(call)                                                                        \
  do {                                                                                          \
    cudaError_t e_ = (call);                                                                    \
    if (e_ != cudaSuccess) return report_error(SQOC_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// image of Fock index x under element g (g < n: rotation r^g; g >= n: reflection s r^(g-n)),
// perm[i-1] = image of site i; bit of site i is x >> (n - i)
__host__ __device__ inline int dn_image(int x, int g, int n) {
  int y = 0;
  const bool refl = g >= n;
  const int m = refl ? g - n : g;
  for (int i = 1; i <= n; ++i) {
    const int pi = refl ? n - (i - 1 + m) % n : (i - 1 + m) % n + 1;
    y |= ((x >> (n - i)) & 1) << (n - pi);
  }
  return y;
}

__global__ void orbit_kernel(int n, int* rep, int* size, int* local) {
  const int dim = 1 << n;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= dim) return;
  int img[2 * kMaxBasisQubits];
  int r = x;
  for (int g = 0; g < 2 * n; ++g) {
    img[g] = dn_image(x, g, n);
    r = min(r, img[g]);
  }
  int s = 0, below = 0;
  for (int g = 0; g < 2 * n; ++g) {
    bool first = true;
    for (int h = 0; h < g; ++h) first = first && img[h] != img[g];
    if (first) {
      ++s;
      below += img[g] < x;
    }
  }
  rep[x] = r;
  size[x] = s;
  local[x] = below;
}

struct ProjectArgs {
  int n, n_orbits, n_rows;
  const int* orb_off;     // [n_orbits + 1] member offsets
  const int* members;     // ascending members of every orbit
  const int* local;       // [2^n] position inside the orbit
  const double* coef;     // [n_rows][2n] diagonal irrep entries A_jj(g)
  const double* scale;    // [n_rows] dim_irrep / |G|
  const long long* vec_base;  // [n_orbits] offset of the orbit's slot area (sum of size^2)
  long long vec_row_stride;   // sum_o size_o^2
  int* count;             // [n_rows][n_orbits] kept vectors
  int* key;               // [n_rows][2^n] generating Fock index of kept vector k: at orb_off[o] + k
  double* vec;            // [n_rows][vec_row_stride]: kept vector k of (row, o) at vec_base[o] + k * size
};

__global__ void project_kernel(ProjectArgs a) {
  const int warps = blockDim.x / 32;
  const int item = blockIdx.x * warps + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (item >= a.n_rows * a.n_orbits) return;
  const int row = item / a.n_orbits, o = item % a.n_orbits;
  const int n = a.n, G = 2 * n;
  const int beg = a.orb_off[o], s = a.orb_off[o + 1] - beg;
  const double* c = a.coef + (size_t)row * G;
  const double sc = a.scale[row];
  double* out = a.vec + (size_t)row * a.vec_row_stride + a.vec_base[o];
  int* keys = a.key + ((size_t)row << n) + beg;
  int kept = 0;
  for (int m = 0; m < s; ++m) {
    const int x = a.members[beg + m];
    double acc = 0.0;
    for (int g = 0; g < G; ++g) {
      const double cg = c[g];
      if (fabs(cg) < 1e-15) continue;  // groups.py:343
      if (a.local[dn_image(x, g, n)] == lane) acc += cg;
    }
    double v = lane < s ? acc * sc : 0.0;
    for (int k = 0; k < kept; ++k) {
      const double u = lane < s ? out[(size_t)k * s + lane] : 0.0;
      double d = u * v;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) d += __shfl_xor_sync(0xffffffffu, d, off);
      v -= d * u;
    }
    double q = v * v;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) q += __shfl_xor_sync(0xffffffffu, q, off);
    const double nrm = sqrt(q);
    if (nrm > kGsRankTol) {  // warp-uniform
      if (lane < s) out[(size_t)kept * s + lane] = v / nrm;
      if (lane == 0) keys[kept] = x;
      ++kept;
      __syncwarp();
    }
  }
  if (lane == 0) a.count[(size_t)row * a.n_orbits + o] = kept;
}

struct CompressArgs {
  int n_cols;              // all block columns
  const int* col_block;    // [n_cols] block of column
  const int* col_index;    // [n_cols] index inside the block
  const int* col_orbit;    // [n_cols]
  const long long* col_vec;  // [n_cols] offset of the column's orbit vector in vec
  const double* vec;
  const int* orb_off;
  const int* members;
  const int* orbit_of;     // [2^n] orbit id
  const int* local;
  const int* bo_off;       // [n_blocks][n_orbits + 1] CSR: columns of block b on orbit o
  const int* bo_cols;      // global column ids
  int n_orbits;
  const int* block_dim;
  const long long* block_off;  // [n_blocks] offset of H_b in out (double2 units)
  int n_terms;
  const int* flip;         // [n_terms]
  const int* sign;         // [n_terms]
  const double2* coef;     // [n_terms]
  double2* out;            // per block d_b x d_b row-major, zeroed
};

__global__ void compress_kernel(CompressArgs a) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= a.n_cols) return;
  const int b = a.col_block[c], ci = a.col_index[c], o = a.col_orbit[c];
  const int d = a.block_dim[b];
  const int beg = a.orb_off[o], s = a.orb_off[o + 1] - beg;
  const double* va = a.vec + a.col_vec[c];
  double2* H = a.out + a.block_off[b];
  const int* boff = a.bo_off + (size_t)b * (a.n_orbits + 1);
  for (int m = 0; m < s; ++m) {
    const int x = a.members[beg + m];
    const double ax = va[m];
    for (int t = 0; t < a.n_terms; ++t) {
      const int y = x ^ a.flip[t];
      const double sg = (__popc(x & a.sign[t]) & 1) ? -ax : ax;
      const double2 cf = a.coef[t];
      const int oy = a.orbit_of[y], ly = a.local[y];
      for (int q = boff[oy]; q < boff[oy + 1]; ++q) {
        const int cp = a.bo_cols[q];
        const double w = a.vec[a.col_vec[cp] + ly] * sg;
        double2& h = H[(size_t)a.col_index[cp] * d + ci];
        h.x += w * cf.x;
        h.y += w * cf.y;
      }
    }
  }
}

}  // namespace

struct sqoc_basis {
  int n = 0, device = 0, n_orbits = 0, n_cols = 0;
  std::vector<int> dims, rows, orb_off, members;
  std::vector<int> col_orbit, col_key;  // per global column (block-major)
  std::vector<long long> col_vec, block_off;
  std::vector<double> vec_host;  // kept vectors (for export)
  std::vector<std::string> labels;
  // device
  int *d_orb_off = nullptr, *d_members = nullptr, *d_orbit_of = nullptr, *d_local = nullptr;
  int *d_col_block = nullptr, *d_col_index = nullptr, *d_col_orbit = nullptr;
  long long *d_col_vec = nullptr, *d_block_off = nullptr;
  int *d_bo_off = nullptr, *d_bo_cols = nullptr, *d_block_dim = nullptr;
  double* d_vec = nullptr;
};

static void basis_free(sqoc_basis* B) {
  if (!B) return;
  cudaSetDevice(B->device);
  for (void* p : {(void*)B->d_orb_off, (void*)B->d_members, (void*)B->d_orbit_of, (void*)B->d_local,
                  (void*)B->d_col_block, (void*)B->d_col_index, (void*)B->d_col_orbit, (void*)B->d_col_vec,
                  (void*)B->d_block_off, (void*)B->d_bo_off, (void*)B->d_bo_cols, (void*)B->d_block_dim,
                  (void*)B->d_vec})
    cudaFree(p);
  delete B;
}

template <class T>
static cudaError_t upload(T** dst, const std::vector<T>& v) {
  cudaError_t e = cudaMalloc(dst, std::max<size_t>(1, v.size()) * sizeof(T));
  if (e != cudaSuccess) return e;
  return v.empty() ? cudaSuccess : cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
}

static int build(sqoc_basis* B) {
  const int n = B->n, dim = 1 << n, G = 2 * n;
  BASIS_CUDA(cudaSetDevice(B->device));
  // ---- orbits
  int *d_rep = nullptr, *d_size = nullptr;
  BASIS_CUDA(cudaMalloc(&d_rep, dim * sizeof(int)));
  BASIS_CUDA(cudaMalloc(&d_size, dim * sizeof(int)));
  BASIS_CUDA(cudaMalloc(&B->d_local, dim * sizeof(int)));
  orbit_kernel<<<(dim + 255) / 256, 256>>>(n, d_rep, d_size, B->d_local);
  BASIS_CUDA(cudaGetLastError());
  std::vector<int> rep(dim);
  BASIS_CUDA(cudaMemcpy(rep.data(), d_rep, dim * sizeof(int), cudaMemcpyDeviceToHost));
  cudaFree(d_rep);
  cudaFree(d_size);
  // orbit ids in ascending representative order (= first appearance); members ascending
  std::vector<int> orbit_of(dim), count;
  std::vector<int> id_of_rep(dim, -1);
  for (int x = 0; x < dim; ++x)
    if (rep[x] == x) {
      id_of_rep[x] = (int)count.size();
      count.push_back(0);
    }
  B->n_orbits = (int)count.size();
  for (int x = 0; x < dim; ++x) count[orbit_of[x] = id_of_rep[rep[x]]]++;
  B->orb_off.assign(B->n_orbits + 1, 0);
  for (int o = 0; o < B->n_orbits; ++o) B->orb_off[o + 1] = B->orb_off[o] + count[o];
  B->members.assign(dim, 0);
  {
    std::vector<int> fill(B->orb_off.begin(), B->orb_off.end() - 1);
    for (int x = 0; x < dim; ++x) B->members[fill[orbit_of[x]]++] = x;
  }
  BASIS_CUDA(upload(&B->d_orb_off, B->orb_off));
  BASIS_CUDA(upload(&B->d_members, B->members));
  BASIS_CUDA(upload(&B->d_orbit_of, orbit_of));
  // ---- irrep rows in the reference table order (groups.py:298-307): A1, A2, (B1, B2), E_k (j = 1, 2)
  struct Row { std::string label; int dim; int kind; int k; int j; };
  std::vector<Row> rows = {{"A1", 1, 0, 0, 0}, {"A2", 1, 1, 0, 0}};
  if (n % 2 == 0) {
    rows.push_back({"B1", 1, 2, 0, 0});
    rows.push_back({"B2", 1, 3, 0, 0});
  }
  for (int k = 1; k <= (n - 1) / 2; ++k)
    for (int j = 0; j < 2; ++j) rows.push_back({"E" + std::to_string(k) + "(j=" + std::to_string(j + 1) + ")", 2, 4, k, j});
  const int R = (int)rows.size();
  std::vector<double> coef((size_t)R * G), scale(R);
  for (int r = 0; r < R; ++r) {
    scale[r] = (double)rows[r].dim / G;
    for (int g = 0; g < G; ++g) {
      const bool refl = g >= n;
      const int m = refl ? g - n : g;
      double v = 1.0;  // diagonal entries of the irrep matrices (groups.py:153-171)
      switch (rows[r].kind) {
        case 0: v = 1.0; break;
        case 1: v = refl ? -1.0 : 1.0; break;
        case 2: v = (m & 1) ? -1.0 : 1.0; break;
        case 3: v = ((m & 1) ? -1.0 : 1.0) * (refl ? -1.0 : 1.0); break;
        default: {
          const double cth = std::cos(2.0 * M_PI * rows[r].k * m / n);
          v = (refl && rows[r].j == 1) ? -cth : cth;
        }
      }
      coef[(size_t)r * G + g] = v;
    }
  }
  std::vector<long long> vec_base(B->n_orbits);
  long long stride = 0;
  for (int o = 0; o < B->n_orbits; ++o) {
    vec_base[o] = stride;
    stride += (long long)count[o] * count[o];
  }
  double *d_coef = nullptr, *d_scale = nullptr;
  long long* d_vec_base = nullptr;
  int *d_count = nullptr, *d_key = nullptr;
  BASIS_CUDA(upload(&d_coef, coef));
  BASIS_CUDA(upload(&d_scale, scale));
  BASIS_CUDA(upload(&d_vec_base, vec_base));
  BASIS_CUDA(cudaMalloc(&d_count, (size_t)R * B->n_orbits * sizeof(int)));
  BASIS_CUDA(cudaMalloc(&d_key, ((size_t)R << n) * sizeof(int)));
  BASIS_CUDA(cudaMalloc(&B->d_vec, (size_t)R * stride * sizeof(double)));
  ProjectArgs pa{n, B->n_orbits, R, B->d_orb_off, B->d_members, B->d_local, d_coef, d_scale, d_vec_base, stride,
                 d_count, d_key, B->d_vec};
  const int items = R * B->n_orbits;
  project_kernel<<<(items + 3) / 4, 128>>>(pa);
  BASIS_CUDA(cudaGetLastError());
  std::vector<int> kcount((size_t)R * B->n_orbits), keys((size_t)R << n);
  BASIS_CUDA(cudaMemcpy(kcount.data(), d_count, kcount.size() * sizeof(int), cudaMemcpyDeviceToHost));
  BASIS_CUDA(cudaMemcpy(keys.data(), d_key, keys.size() * sizeof(int), cudaMemcpyDeviceToHost));
  B->vec_host.resize((size_t)R * stride);
  BASIS_CUDA(cudaMemcpy(B->vec_host.data(), B->d_vec, B->vec_host.size() * sizeof(double), cudaMemcpyDeviceToHost));
  cudaFree(d_coef);
  cudaFree(d_scale);
  cudaFree(d_vec_base);
  cudaFree(d_count);
  cudaFree(d_key);
  // ---- blocks: each row's kept vectors sorted by (weight(key), key) (adjoint.py:200-201)
  std::vector<int> col_block, col_index;
  std::vector<std::vector<std::pair<int, int>>> bo;  // per block: (orbit, global column)
  for (int r = 0; r < R; ++r) {
    struct Col { int w, key, o, k; };
    std::vector<Col> cols;
    for (int o = 0; o < B->n_orbits; ++o)
      for (int k = 0; k < kcount[(size_t)r * B->n_orbits + o]; ++k) {
        const int key = keys[((size_t)r << n) + B->orb_off[o] + k];
        cols.push_back({__builtin_popcount(key), key, o, k});
      }
    if (cols.empty()) continue;
    std::sort(cols.begin(), cols.end(), [](const Col& a, const Col& b) { return a.w != b.w ? a.w < b.w : a.key < b.key; });
    const int b = (int)B->dims.size();
    B->dims.push_back((int)cols.size());
    B->rows.push_back(r);
    B->labels.push_back(rows[r].label);
    bo.emplace_back();
    for (int i = 0; i < (int)cols.size(); ++i) {
      const int s = count[cols[i].o];
      B->col_orbit.push_back(cols[i].o);
      B->col_key.push_back(cols[i].key);
      B->col_vec.push_back((long long)r * stride + vec_base[cols[i].o] + (long long)cols[i].k * s);
      col_block.push_back(b);
      col_index.push_back(i);
      bo[b].push_back({cols[i].o, (int)B->col_orbit.size() - 1});
    }
  }
  B->n_cols = (int)B->col_orbit.size();
  if (B->n_cols != dim) return report_error(SQOC_ERR_ARG, "rank deficiency: block columns do not span the space");
  const int nb = (int)B->dims.size();
  std::vector<int> bo_off((size_t)nb * (B->n_orbits + 1), 0), bo_cols;
  for (int b = 0; b < nb; ++b) {
    std::stable_sort(bo[b].begin(), bo[b].end(), [](const std::pair<int, int>& x, const std::pair<int, int>& y) { return x.first < y.first; });
    int* off = bo_off.data() + (size_t)b * (B->n_orbits + 1);
    for (auto& pr : bo[b]) off[pr.first + 1]++;
    for (int o = 0; o < B->n_orbits; ++o) off[o + 1] += off[o];
    for (auto& pr : bo[b]) bo_cols.push_back(pr.second);
    for (int o = 0; o <= B->n_orbits; ++o) off[o] += (int)bo_cols.size() - (int)bo[b].size();
  }
  B->block_off.assign(nb, 0);
  for (int b = 1; b < nb; ++b) B->block_off[b] = B->block_off[b - 1] + (long long)B->dims[b - 1] * B->dims[b - 1];
  BASIS_CUDA(upload(&B->d_col_block, col_block));
  BASIS_CUDA(upload(&B->d_col_index, col_index));
  BASIS_CUDA(upload(&B->d_col_orbit, B->col_orbit));
  BASIS_CUDA(upload(&B->d_col_vec, B->col_vec));
  BASIS_CUDA(upload(&B->d_bo_off, bo_off));
  BASIS_CUDA(upload(&B->d_bo_cols, bo_cols));
  BASIS_CUDA(upload(&B->d_block_dim, B->dims));
  BASIS_CUDA(upload(&B->d_block_off, B->block_off));
  return SQOC_OK;
}

extern "C" {

int sqoc_dn_basis_create(sqoc_basis** out, int device, int n) {
  if (!out) return report_error(SQOC_ERR_ARG, "out is NULL");
  *out = nullptr;
  if (n < 3 || n > kMaxBasisQubits) return report_error(SQOC_ERR_ARG, "D_n basis needs 3 <= n <= 16");
  sqoc_basis* B = new sqoc_basis();
  B->n = n;
  B->device = device;
  const int rc = build(B);
  if (rc != SQOC_OK) {
    basis_free(B);
    return rc;
  }
  *out = B;
  return SQOC_OK;
}

int sqoc_basis_info(const sqoc_basis* B, int* n_blocks, int* dims, int* irrep_rows) {
  if (!B || !n_blocks) return report_error(SQOC_ERR_ARG, "basis or n_blocks is NULL");
  *n_blocks = (int)B->dims.size();
  for (size_t b = 0; b < B->dims.size(); ++b) {
    if (dims) dims[b] = B->dims[b];
    if (irrep_rows) irrep_rows[b] = B->rows[b];
  }
  return SQOC_OK;
}

int sqoc_basis_columns(const sqoc_basis* B, int block, int* keys, int* col_nnz, int* rows, double* vals) {
  if (!B || block < 0 || block >= (int)B->dims.size()) return report_error(SQOC_ERR_ARG, "bad basis or block");
  int c0 = 0;
  for (int b = 0; b < block; ++b) c0 += B->dims[b];
  size_t w = 0;
  for (int i = 0; i < B->dims[block]; ++i) {
    const int c = c0 + i, o = B->col_orbit[c];
    const int beg = B->orb_off[o], s = B->orb_off[o + 1] - beg;
    if (keys) keys[i] = B->col_key[c];
    if (col_nnz) col_nnz[i] = s;
    for (int m = 0; m < s; ++m, ++w) {
      if (rows) rows[w] = B->members[beg + m];
      if (vals) vals[w] = B->vec_host[B->col_vec[c] + m];
    }
  }
  return SQOC_OK;
}

int sqoc_basis_nnz(const sqoc_basis* B, int block, long long* nnz) {
  if (!B || !nnz || block < 0 || block >= (int)B->dims.size()) return report_error(SQOC_ERR_ARG, "bad basis or block");
  int c0 = 0;
  for (int b = 0; b < block; ++b) c0 += B->dims[b];
  long long t = 0;
  for (int i = 0; i < B->dims[block]; ++i) {
    const int o = B->col_orbit[c0 + i];
    t += B->orb_off[o + 1] - B->orb_off[o];
  }
  *nnz = t;
  return SQOC_OK;
}

int sqoc_basis_compress(const sqoc_basis* B, int n_terms, const int* flip, const int* sign, const double* coef,
                        double* const* out) {
  if (!B || n_terms < 0 || (n_terms && (!flip || !sign || !coef)) || !out)
    return report_error(SQOC_ERR_ARG, "bad compress arguments");
  BASIS_CUDA(cudaSetDevice(B->device));
  const int nb = (int)B->dims.size();
  const long long total = B->block_off.back() + (long long)B->dims.back() * B->dims.back();
  double2* d_out = nullptr;
  int *d_flip = nullptr, *d_sign = nullptr;
  double2* d_coef = nullptr;
  BASIS_CUDA(cudaMalloc(&d_out, total * sizeof(double2)));
  BASIS_CUDA(cudaMemset(d_out, 0, total * sizeof(double2)));
  std::vector<int> vf(flip, flip + n_terms), vs(sign, sign + n_terms);
  std::vector<double2> vc(n_terms);
  for (int t = 0; t < n_terms; ++t) vc[t] = make_double2(coef[2 * t], coef[2 * t + 1]);
  BASIS_CUDA(upload(&d_flip, vf));
  BASIS_CUDA(upload(&d_sign, vs));
  BASIS_CUDA(upload(&d_coef, vc));
  CompressArgs a{B->n_cols, B->d_col_block, B->d_col_index, B->d_col_orbit, B->d_col_vec, B->d_vec,
                 B->d_orb_off, B->d_members, B->d_orbit_of, B->d_local, B->d_bo_off, B->d_bo_cols,
                 B->n_orbits, B->d_block_dim, B->d_block_off, n_terms, d_flip, d_sign, d_coef, d_out};
  compress_kernel<<<(B->n_cols + 127) / 128, 128>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  for (int b = 0; b < nb && e == cudaSuccess; ++b)
    e = cudaMemcpy(out[b], d_out + B->block_off[b], (size_t)B->dims[b] * B->dims[b] * sizeof(double2),
                   cudaMemcpyDeviceToHost);
  cudaFree(d_out);
  cudaFree(d_flip);
  cudaFree(d_sign);
  cudaFree(d_coef);
  if (e != cudaSuccess) return report_error(SQOC_ERR_CUDA, std::string("basis compress: ") + cudaGetErrorString(e));
  return SQOC_OK;
}

int sqoc_basis_destroy(sqoc_basis* B) {
  basis_free(B);
  return SQOC_OK;
}

}  // extern "C"
