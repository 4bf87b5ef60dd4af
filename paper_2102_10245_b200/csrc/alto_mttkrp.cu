// alto_mttkrp.cu — the deterministic reference-order MTTKRP engines.
//
//   out[i_n, r] = sum over elements x: x.value * prod_{m != n} F_m[x.coord_m, r]
//   (pkg/src/altotensor/mttkrp.py:1-14, contributions :80-105)
//
// 1. Exact-order engine (`alto_row_index` + `alto_mttkrp_exact`): per output
//    row, contributions are summed sequentially in element order, restarted
//    at partition boundaries, and the partition partials combined in
//    ascending order — the arithmetic order of _par_buffered
//    (mttkrp.py:148-172) and mttkrp_seq (:108-117), in float64 with
//    contraction disabled, hence bitwise equal to the reference on float64
//    inputs.
// 2. COO kernels over a coordinate list (mttkrp_oracle, mttkrp.py:64-77):
//    `alto_mttkrp_coo` (float64 atomics) and `alto_mttkrp_coo_ordered`
//    (stable row sort, each row summed in input order: bitwise = reference).
// The streaming kernels live in alto_mstream.cuh (mode stream), alto_pull.cuh
// (K8/K9 slice buffers + pull), alto_fast.cuh (ALTO-order planned kernel)
// and alto_stream.cuh (generic fallback).
#include <algorithm>
#include <climits>

#include "alto_common.cuh"

namespace alto {

struct ExactParams {
  const uint64_t* keys;
  const void* values;
  long long m;
  int mode;
  int rank;
  const void* factors[ALTO_MAX_ORDER];
  double* out;
};

// ---- exact-order engine ------------------------------------------------------

__global__ void row_ptr_kernel(const uint64_t* __restrict__ sorted_rows, long long m, long long dim,
                               long long* __restrict__ row_ptr) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i <= m; i += stride) {
    const long long prev = i > 0 ? static_cast<long long>(sorted_rows[i - 1]) : -1;
    const long long cur = i < m ? static_cast<long long>(sorted_rows[i]) : dim;
    for (long long r = prev + 1; r <= cur && r <= dim; ++r) row_ptr[r] = i;
  }
}

__global__ void iota_u32(unsigned* p, long long n) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n; i += stride)
    p[i] = static_cast<unsigned>(i);
}

template <int W, typename V, typename F>
__global__ void __launch_bounds__(256)
mttkrp_exact_kernel(const __grid_constant__ DevLayout L, const uint64_t* __restrict__ tab,
                    const __grid_constant__ ExactParams P, const int* __restrict__ row_perm,
                    const long long* __restrict__ row_ptr, const long long* __restrict__ part_off,
                    long long count, long long dim) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* s_dec = reinterpret_cast<uint64_t*>(smem);
  copy_to_smem(s_dec, tab + static_cast<long long>(L.dec_off) * W, L.dec_bytes * 256 * W);
  __syncthreads();
  const int N = L.order, R = P.rank, mode = P.mode;
  const int lane = threadIdx.x & 31;
  const long long gwarp = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5;
  const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
  const V* __restrict__ vals = static_cast<const V*>(P.values);
  for (long long row = gwarp; row < dim; row += nwarps) {
    const long long j0 = row_ptr[row], j1 = row_ptr[row + 1];
    for (int r0 = 0; r0 < R; r0 += 32) {
      const int r = r0 + lane;
      double total = 0.0, part = 0.0;
      long long l = 0;
      bool have_part = false;
      for (long long j = j0; j < j1; ++j) {
        const long long e = row_perm[j];
        while (l + 1 < count && part_off[l + 1] <= e) {  // crossed into a later partition
          if (have_part) { total = __dadd_rn(total, part); part = 0.0; have_part = false; }
          ++l;
        }
        const Key<W> p = decode_packed<W>(s_dec, L.dec_bytes, load_key<W>(P.keys, e));
        double x = static_cast<double>(vals[e]);
        if (r < R) {
          for (int n = 0; n < N; ++n) {
            if (n == mode) continue;
            const long long c = packed_field<W>(p, L.pack_off[n], L.bits[n]);
            const F* f = static_cast<const F*>(P.factors[n]);
            x = __dmul_rn(x, static_cast<double>(f[c * R + r]));
          }
        }
        part = __dadd_rn(part, x);
        have_part = true;
      }
      if (have_part) total = __dadd_rn(total, part);
      if (r < R) P.out[row * R + r] = total;
    }
  }
}

// ---- COO kernel (mttkrp_oracle) ------------------------------------------------

struct CooParams {
  const long long* coords;
  const double* values;
  long long m;
  int order, mode, rank;
  const double* factors[ALTO_MAX_ORDER];
  double* out;
};

__global__ void mttkrp_coo_kernel(const __grid_constant__ CooParams P) {
  const long long total = P.m * P.rank;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < total; t += stride) {
    const long long e = t / P.rank;
    const int r = static_cast<int>(t - e * P.rank);
    double x = P.values[e];
    for (int n = 0; n < P.order; ++n) {
      if (n == P.mode) continue;
      x = __dmul_rn(x, P.factors[n][P.coords[e * P.order + n] * P.rank + r]);
    }
    atomicAdd(P.out + P.coords[e * P.order + P.mode] * P.rank + r, x);
  }
}

// Input-order COO MTTKRP: rows sorted stably (element index as payload), one
// warp per output row sums its elements in input order — np.add.at's order in
// mttkrp_oracle (mttkrp.py:71-76), with contrib = ((v * F_a) * F_b) ... in
// ascending mode order, no contraction: bitwise equal to the reference.
__global__ void __launch_bounds__(256)
mttkrp_coo_ordered_kernel(const __grid_constant__ CooParams P, const unsigned* __restrict__ perm,
                          const long long* __restrict__ row_ptr, long long dim) {
  const int lane = threadIdx.x & 31;
  const long long gwarp = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5;
  const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
  for (long long row = gwarp; row < dim; row += nwarps) {
    const long long j0 = row_ptr[row], j1 = row_ptr[row + 1];
    for (int r0 = 0; r0 < P.rank; r0 += 32) {
      const int r = r0 + lane;
      double total = 0.0;
      if (r < P.rank) {
        for (long long j = j0; j < j1; ++j) {
          const long long e = perm[j];
          double x = P.values[e];
          for (int n = 0; n < P.order; ++n) {
            if (n == P.mode) continue;
            x = __dmul_rn(x, P.factors[n][P.coords[e * P.order + n] * P.rank + r]);
          }
          total = __dadd_rn(total, x);
        }
        P.out[row * P.rank + r] = total;
      }
    }
  }
}

__global__ void coo_rows_kernel(const long long* __restrict__ coords, long long m, int order, int mode,
                                uint64_t* __restrict__ rows, unsigned* __restrict__ idx) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < m; i += stride) {
    rows[i] = static_cast<uint64_t>(coords[i * order + mode]);
    idx[i] = static_cast<unsigned>(i);
  }
}

// ---- launch helpers ----------------------------------------------------------------

template <typename K>
static int prep_smem(K kernel, size_t smem) {
  ALTO_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  return ALTO_OK;
}

static int check_args(const alto_mttkrp_args* a) {
  ALTO_REQUIRE(a && a->lay && a->d_tables, "mttkrp args incomplete");
  ALTO_REQUIRE(a->lay->order >= 1 && a->lay->order <= ALTO_MAX_ORDER, "bad layout order");
  ALTO_REQUIRE(a->mode >= 0 && a->mode < a->lay->order, "mode out of range");
  ALTO_REQUIRE(a->rank >= 1, "rank must be positive");
  ALTO_REQUIRE((a->value_dtype == ALTO_F32 || a->value_dtype == ALTO_F64) &&
                   (a->factor_dtype == ALTO_F32 || a->factor_dtype == ALTO_F64),
               "unsupported dtype");
  ALTO_REQUIRE(a->out != nullptr, "out is NULL");
  ALTO_REQUIRE(a->out_dtype == ALTO_F32 || a->out_dtype == ALTO_F64, "unsupported output dtype");
  return ALTO_OK;
}

static ExactParams to_params(const alto_mttkrp_args* a) {
  ExactParams P{};
  P.keys = a->keys;
  P.values = a->values;
  P.m = a->m;
  P.mode = a->mode;
  P.rank = a->rank;
  for (int n = 0; n < ALTO_MAX_ORDER; ++n) P.factors[n] = n < a->lay->order ? a->factors[n] : nullptr;
  P.out = static_cast<double*>(a->out);
  return P;
}

}  // namespace alto

using namespace alto;

extern "C" {

size_t alto_row_index_workspace_bytes(int64_t m, int64_t dim) {
  (void)dim;
  if (m < 0) m = 0;
  const size_t a = ((static_cast<size_t>(m) * 8 + 255) & ~size_t(255));
  return a + alto_sort_workspace_bytes(m, 1, 4);
}

int alto_row_index(const alto_layout* lay, const void* d_tables, const uint64_t* keys, int64_t m, int32_t mode,
                   int32_t* row_perm, int64_t* row_ptr, void* workspace, size_t workspace_bytes, void* stream) {
  ALTO_REQUIRE(lay && mode >= 0 && mode < lay->order, "mode out of range");
  ALTO_REQUIRE(workspace_bytes >= alto_row_index_workspace_bytes(m, lay->dims[mode]), "row index workspace too small");
  cudaStream_t s = as_stream(stream);
  const long long dim = lay->dims[mode];
  if (m <= 0) {
    ALTO_CUDA_TRY(cudaMemsetAsync(row_ptr, 0, static_cast<size_t>(dim + 1) * 8, s));
    return ALTO_OK;
  }
  auto* rows = static_cast<uint64_t*>(workspace);
  const size_t a = ((static_cast<size_t>(m) * 8 + 255) & ~size_t(255));
  void* sort_ws = static_cast<char*>(workspace) + a;
  int st = alto_delinearize(lay, d_tables, keys, m, mode, reinterpret_cast<int64_t*>(rows), stream);
  if (st) return st;
  if (row_perm) {
    iota_u32<<<grid_for(m, 256), 256, 0, s>>>(reinterpret_cast<unsigned*>(row_perm), m);
    ALTO_LAUNCH_CHECK("alto_row_index/iota");
    st = alto_sort_pairs(rows, row_perm, m, 1, 4, lay->bits[mode], sort_ws, workspace_bytes - a, stream);
  } else {
    // row_ptr only (hot-row plans need the rows' element counts, not the permutation): keys-only sort
    st = alto_sort_pairs(rows, nullptr, m, 1, 0, lay->bits[mode], sort_ws, workspace_bytes - a, stream);
  }
  if (st) return st;
  row_ptr_kernel<<<grid_for(m + 1, 256), 256, 0, s>>>(rows, m, dim, reinterpret_cast<long long*>(row_ptr));
  ALTO_LAUNCH_CHECK("alto_row_index/row_ptr");
  return ALTO_OK;
}

int alto_mttkrp_exact(const alto_mttkrp_args* a, const int32_t* row_perm, const int64_t* row_ptr,
                      const int64_t* part_off, int64_t count, void* stream) {
  int st = check_args(a);
  if (st) return st;
  ALTO_REQUIRE(count >= 1 && part_off != nullptr, "partition offsets required");
  const DevLayout d = make_dev_layout(a->lay);
  cudaStream_t s = as_stream(stream);
  const long long dim = d.dims[a->mode];
  if (a->m <= 0 || dim <= 0) {
    ALTO_CUDA_TRY(cudaMemsetAsync(a->out, 0, static_cast<size_t>(dim) * a->rank * sizeof(double), s));
    return ALTO_OK;
  }
  ALTO_REQUIRE(a->out_dtype == ALTO_F64, "exact engine writes float64");
  ExactParams P = to_params(a);
  const auto* tab = static_cast<const uint64_t*>(a->d_tables);
  const size_t smem = static_cast<size_t>(d.dec_bytes) * 256 * d.n_words * 8;
  const int grid = grid_for(dim * 32, 256, kSMs * 8);
  auto go = [&](auto kern) -> int {
    if (prep_smem(kern, smem)) return ALTO_ECUDA;
    kern<<<grid, 256, smem, s>>>(d, tab, P, reinterpret_cast<const int*>(row_perm),
                                 reinterpret_cast<const long long*>(row_ptr),
                                 reinterpret_cast<const long long*>(part_off), count, dim);
    ALTO_LAUNCH_CHECK("alto_mttkrp_exact");
    return ALTO_OK;
  };
  const bool v32 = a->value_dtype == ALTO_F32, f32 = a->factor_dtype == ALTO_F32;
  if (d.n_words == 1) {
    if (v32 && f32) return go(mttkrp_exact_kernel<1, float, float>);
    if (!v32 && !f32) return go(mttkrp_exact_kernel<1, double, double>);
    if (v32) return go(mttkrp_exact_kernel<1, float, double>);
    return go(mttkrp_exact_kernel<1, double, float>);
  }
  if (v32 && f32) return go(mttkrp_exact_kernel<2, float, float>);
  if (!v32 && !f32) return go(mttkrp_exact_kernel<2, double, double>);
  if (v32) return go(mttkrp_exact_kernel<2, float, double>);
  return go(mttkrp_exact_kernel<2, double, float>);
}

size_t alto_mttkrp_coo_workspace_bytes(int64_t m, int64_t out_rows) {
  if (m < 0) m = 0;
  const size_t a = (static_cast<size_t>(m) * 8 + 255) & ~size_t(255);
  const size_t b = (static_cast<size_t>(m) * 4 + 255) & ~size_t(255);
  const size_t c = (static_cast<size_t>(out_rows + 1) * 8 + 255) & ~size_t(255);
  return a + b + c + alto_sort_workspace_bytes(m, 1, 4);
}

int alto_mttkrp_coo_ordered(const int64_t* coords, const double* values, int64_t m, int32_t order, int32_t mode,
                            int32_t rank, const double* const* factors_host_array, double* out, int64_t out_rows,
                            void* ws, size_t ws_bytes, void* stream) {
  ALTO_REQUIRE(order >= 1 && order <= ALTO_MAX_ORDER, "order out of range");
  ALTO_REQUIRE(mode >= 0 && mode < order, "mode out of range");
  ALTO_REQUIRE(rank >= 1, "rank must be positive");
  ALTO_REQUIRE(m < (1ll << 32) - 1, "ordered COO MTTKRP supports fewer than 2^32 elements");
  cudaStream_t s = as_stream(stream);
  if (m <= 0) {
    ALTO_CUDA_TRY(cudaMemsetAsync(out, 0, static_cast<size_t>(out_rows) * rank * sizeof(double), s));
    return ALTO_OK;
  }
  ALTO_REQUIRE(ws && ws_bytes >= alto_mttkrp_coo_workspace_bytes(m, out_rows), "COO workspace too small");
  const size_t a = (static_cast<size_t>(m) * 8 + 255) & ~size_t(255);
  const size_t b = (static_cast<size_t>(m) * 4 + 255) & ~size_t(255);
  const size_t c = (static_cast<size_t>(out_rows + 1) * 8 + 255) & ~size_t(255);
  auto* rows = static_cast<uint64_t*>(ws);
  auto* idx = reinterpret_cast<unsigned*>(static_cast<char*>(ws) + a);
  auto* row_ptr = reinterpret_cast<long long*>(static_cast<char*>(ws) + a + b);
  void* sws = static_cast<char*>(ws) + a + b + c;
  const auto* cc = reinterpret_cast<const long long*>(coords);
  coo_rows_kernel<<<grid_for(m, 256), 256, 0, s>>>(cc, m, order, mode, rows, idx);
  ALTO_LAUNCH_CHECK("alto_mttkrp_coo_ordered/rows");
  int bits = 1;
  while (bits < 63 && (1ll << bits) < out_rows) ++bits;
  const int st = alto_sort_pairs(rows, idx, m, 1, 4, bits, sws, ws_bytes - a - b - c, stream);
  if (st) return st;
  row_ptr_kernel<<<grid_for(m + 1, 256), 256, 0, s>>>(rows, m, out_rows, row_ptr);
  ALTO_LAUNCH_CHECK("alto_mttkrp_coo_ordered/row_ptr");
  CooParams P{};
  P.coords = cc;
  P.values = values;
  P.m = m;
  P.order = order;
  P.mode = mode;
  P.rank = rank;
  for (int n = 0; n < order; ++n) P.factors[n] = factors_host_array[n];
  P.out = out;
  mttkrp_coo_ordered_kernel<<<grid_for(out_rows * 32, 256, kSMs * 64), 256, 0, s>>>(P, idx, row_ptr, out_rows);
  ALTO_LAUNCH_CHECK("alto_mttkrp_coo_ordered");
  return ALTO_OK;
}

int alto_mttkrp_coo(const int64_t* coords, const double* values, int64_t m, int32_t order, int32_t mode,
                    int32_t rank, const double* const* factors_host_array, double* out, int64_t out_rows,
                    void* stream) {
  ALTO_REQUIRE(order >= 1 && order <= ALTO_MAX_ORDER, "order out of range");
  ALTO_REQUIRE(mode >= 0 && mode < order, "mode out of range");
  ALTO_REQUIRE(rank >= 1, "rank must be positive");
  cudaStream_t s = as_stream(stream);
  ALTO_CUDA_TRY(cudaMemsetAsync(out, 0, static_cast<size_t>(out_rows) * rank * sizeof(double), s));
  if (m <= 0) return ALTO_OK;
  CooParams P{};
  P.coords = reinterpret_cast<const long long*>(coords);
  P.values = values;
  P.m = m;
  P.order = order;
  P.mode = mode;
  P.rank = rank;
  for (int n = 0; n < order; ++n) P.factors[n] = factors_host_array[n];
  P.out = out;
  mttkrp_coo_kernel<<<grid_for(m * rank, 256), 256, 0, s>>>(P);
  ALTO_LAUNCH_CHECK("alto_mttkrp_coo");
  return ALTO_OK;
}

}  // extern "C"
