// alto_stream.cu — C ABI of the streaming ALTO MTTKRP (see alto_stream.cuh
// for the kernel design), the hot-row plan and the hot-copy reduction.
#include <type_traits>

#include "alto_mstream.cuh"

namespace alto {

// Sum the replicated hot-row partials into out and re-zero them.  A block
// covers 32 (hot row, rank) elements x 8 copy groups: thread (g, lane) sums
// copies g, g+8, ... of its element (coalesced across lanes), then group 0
// adds the 8 partials in a fixed order (deterministic).
template <typename O, typename B = O>
__global__ void __launch_bounds__(256) hot_reduce_kernel(B* __restrict__ buf, const int* __restrict__ hot_rows,
                                                         int n_hot, int copies, int R, O* __restrict__ out) {
  using S = typename std::conditional<std::is_same<O, long long>::value, long long, double>::type;
  __shared__ S s_part[8][33];
  const long long n = static_cast<long long>(n_hot) * R;
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const long long i = static_cast<long long>(blockIdx.x) * 32 + lane;
  S s = S(0);
  if (i < n) {
    // loads first, then the zeroing stores (no load-after-store chains)
    constexpr int UB = 8;
    for (int k0 = g; k0 < copies; k0 += 8 * UB) {
      B v[UB];
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        const int k = k0 + 8 * u;
        v[u] = k < copies ? buf[k * n + i] : B(0);
      }
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        const int k = k0 + 8 * u;
        s += static_cast<S>(v[u]);
        if (k < copies) buf[k * n + i] = B(0);
      }
    }
  }
  s_part[g][lane] = s;
  __syncthreads();
  if (g == 0 && i < n) {
    S t = S(0);
#pragma unroll
    for (int q = 0; q < 8; ++q) t += s_part[q][lane];
    const long long h = i / R;
    O* o = out + static_cast<long long>(hot_rows[h]) * R + (i - h * R);
    *o = static_cast<O>(static_cast<S>(*o) + t);
  }
}

// Hot-row copy plan: copies(r) = next power of two of (estimated merges of r)
// / bound, clamped to [1, 2^max_lg]; estimated merges = min(count, ntiles) +
// count / (tile/8) (one run per tile, plus one per slice the row spans).
__global__ void hot_copies_kernel(const long long* __restrict__ row_ptr, const int* __restrict__ hot_rows, int n_hot,
                                  long long ntiles, int tile, int row_major, int bound, int max_lg,
                                  int* __restrict__ hot_code, int* __restrict__ hot_base) {
  __shared__ int s_part[1024];
  const int per = (n_hot + blockDim.x - 1) / blockDim.x;
  const int s0 = threadIdx.x * per, s1 = min(n_hot, s0 + per);
  auto lg_of = [&](int s) {
    const long long r = hot_rows[s];
    const long long c = row_ptr[r + 1] - row_ptr[r];
    // merges of a row: row-major stream -> one per slice it spans (+ the two
    // partial ends); tile order -> up to one per tile plus one per slice
    const long long per_slice = c / max(1, tile / kMsSlices);
    const long long est = row_major ? per_slice + 2 : min(c, ntiles) + per_slice;
    const long long want = (est + bound - 1) / bound;
    int lg = 0;
    while (lg < max_lg && (1ll << lg) < want) ++lg;
    return lg;
  };
  int sum = 0;
  for (int s = s0; s < s1; ++s) sum += 1 << lg_of(s);
  s_part[threadIdx.x] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int i = 0; i < static_cast<int>(blockDim.x); ++i) {
      const int v = s_part[i];
      s_part[i] = run;
      run += v;
    }
    hot_base[n_hot] = run;
  }
  __syncthreads();
  int base = s_part[threadIdx.x];
  for (int s = s0; s < s1; ++s) {
    const int lg = lg_of(s);
    hot_base[s] = base;
    hot_code[hot_rows[s]] = (base << 5) | lg;
    base += 1 << lg;
  }
}

__global__ void hot_plan_kernel(const long long* __restrict__ row_ptr, long long dim, long long tau, int hmax,
                                int* __restrict__ hot_slot, int* __restrict__ hot_rows, int* __restrict__ nhot) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long r = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; r < dim; r += stride) {
    int slot = -1;
    if (row_ptr[r + 1] - row_ptr[r] > tau) {
      const int s = atomicAdd(nhot, 1);
      if (s < hmax) {
        slot = s;
        hot_rows[s] = static_cast<int>(r);
      }
    }
    hot_slot[r] = slot;
  }
}

__global__ void clamp_count(int* n, int hmax) {
  if (*n > hmax) *n = hmax;
}

}  // namespace alto

using namespace alto;


extern "C" {

int alto_mttkrp(const alto_mttkrp_args* a, void* stream) {
  ALTO_REQUIRE(a && a->lay && a->d_tables, "mttkrp args incomplete");
  ALTO_REQUIRE(a->lay->order >= 1 && a->lay->order <= ALTO_MAX_ORDER, "bad layout order");
  ALTO_REQUIRE(a->mode >= 0 && a->mode < a->lay->order, "mode out of range");
  ALTO_REQUIRE(a->rank >= 1, "rank must be positive");
  ALTO_REQUIRE((a->value_dtype == ALTO_F32 || a->value_dtype == ALTO_F64) &&
                   (a->factor_dtype == ALTO_F32 || a->factor_dtype == ALTO_F64) &&
                   (a->out_dtype == ALTO_F32 || a->out_dtype == ALTO_F64 || a->out_dtype == ALTO_I64),
               "unsupported dtype");
  ALTO_REQUIRE(a->out_dtype != ALTO_I64 || a->fixed_scale != nullptr, "fixed-point output needs fixed_scale");
  ALTO_REQUIRE(a->out_dtype != ALTO_F32 || (a->value_dtype == ALTO_F32 && a->factor_dtype == ALTO_F32),
               "float32 output needs float32 values and factors");
  ALTO_REQUIRE(a->out != nullptr, "out is NULL");
  ALTO_REQUIRE(a->n_hot <= 0 || (a->hot_rows && a->hot_slot && a->hot_buf && a->hot_copies > 0),
               "incomplete hot plan");
  for (int n = 0; n < a->lay->order; ++n)
    ALTO_REQUIRE(a->lay->dims[n] <= INT_MAX, "streaming kernel needs mode extents below 2^31");
  const DevLayout d = make_dev_layout(a->lay);
  cudaStream_t s = as_stream(stream);
  const long long dim = d.dims[a->mode];
  const size_t osz = a->out_dtype == ALTO_F32 ? 4 : 8;  // f64 and i64 are 8 bytes
  if (a->zero_out) ALTO_CUDA_TRY(cudaMemsetAsync(a->out, 0, static_cast<size_t>(dim) * a->rank * osz, s));
  if (a->m <= 0) return ALTO_OK;
  StreamParams P{};
  P.keys = a->keys;
  P.values = a->values;
  P.m = a->m;
  P.mode = a->mode;
  P.rank = a->rank;
  for (int n = 0; n < ALTO_MAX_ORDER; ++n) P.factors[n] = n < a->lay->order ? a->factors[n] : nullptr;
  P.out = a->out;
  P.tile = a->tile > 0 ? a->tile : 1024;
  ALTO_REQUIRE(P.tile >= kTileThreads && P.tile <= kEPT * kTileThreads && P.tile % kTileThreads == 0,
               "tile must be a multiple of 256 in [256, 1024]");
  P.ntiles = (a->m + P.tile - 1) / P.tile;
  P.n_hot = a->n_hot > 0 ? a->n_hot : 0;
  P.hot_slot = a->hot_slot;
  P.hot_copies = a->hot_copies > 0 ? a->hot_copies : 1;
  ALTO_REQUIRE((P.hot_copies & (P.hot_copies - 1)) == 0, "hot_copies must be a power of two");
  P.hot_buf = a->hot_buf;
  P.hot_adaptive = (a->hot_base != nullptr && P.n_hot > 0) ? 1 : 0;
  P.flags = a->flags;
  P.packed = a->packed;
  P.pos = a->pos;
  P.fixed_scale = a->out_dtype == ALTO_I64 ? a->fixed_scale : nullptr;
  P.mkeys = a->mkeys;
  P.mvals = a->mvals;
  P.mtile = a->mtile;
  P.mrr = a->mrr;
  P.mbase = a->mkeys ? a->mbase : nullptr;
  for (int n = 0; n < ALTO_MAX_ORDER; ++n) {
    const bool on = n < d.order && a->factor_dtype == ALTO_F32 && a->l2_hot_bytes[n] > 0;
    const unsigned long long tb = on ? static_cast<unsigned long long>(d.dims[n]) * a->rank * 4ull : 0ull;
    P.l2_tab[n] = static_cast<unsigned>(std::min<unsigned long long>(tb, 0xFFFFFFFFull));
    P.l2_hot[n] = on ? std::min(a->l2_hot_bytes[n], P.l2_tab[n]) : 0u;
  }
  P.n_pairs = ((a->mkeys || (a->packed && a->pos)) && a->out_dtype != ALTO_I64) ? std::max(0, std::min(a->n_pairs, 2))
                                                                                 : 0;
  ALTO_REQUIRE(a->n_pairs <= 2, "at most 2 paired input modes");
  for (int i = 0; i < 2; ++i) {
    P.pair_a[i] = a->pair_a[i];
    P.pair_b[i] = a->pair_b[i];
    P.pair_tab[i] = a->pair_tab[i];
  }
  ALTO_REQUIRE(!a->mkeys || (a->mvals && a->mtile >= 128 && a->mtile % 128 == 0),
               "mode stream needs values and a tile that is a multiple of 128");
  ALTO_REQUIRE(!a->mkeys || a->n_hot <= 0 || a->hot_base, "mode-stream hot plan needs hot_base");
  ALTO_REQUIRE(!a->mkeys || a->rank <= 32, "the mode-stream hot-row reduction supports ranks up to 32");
  const auto* tab = static_cast<const uint64_t*>(a->d_tables);
  const bool o32 = a->out_dtype == ALTO_F32;
  if (a->out_dtype == ALTO_I64) {
    int sti = d.n_words == 1 ? fast_w1_i64(d, tab, P, a->value_dtype, a->factor_dtype, s)
                             : fast_w2_i64(d, tab, P, a->value_dtype, a->factor_dtype, s);
    if (sti == ALTO_EUNSUPPORTED) {
      set_error("fixed-point (deterministic) MTTKRP supports orders 3-5 and ranks 16/32 with matching dtypes");
      return ALTO_EUNSUPPORTED;
    }
    if (sti) return sti;
    if (a->hot_base && P.n_hot > 0) {
      hot_reduce_rows_kernel<long long><<<(P.n_hot + 7) / 8, 256, 0, s>>>(
          static_cast<long long*>(P.hot_buf), a->hot_rows, a->hot_base, P.n_hot, a->rank,
          static_cast<long long*>(a->out));
      ALTO_LAUNCH_CHECK("alto_mttkrp/hot_reduce_rows");
    } else if (P.n_hot > 0) {
      const long long nh = static_cast<long long>(P.n_hot) * a->rank;
      hot_reduce_kernel<long long><<<static_cast<int>((nh + 31) / 32), 256, 0, s>>>(
          static_cast<long long*>(P.hot_buf), a->hot_rows, P.n_hot, P.hot_copies, a->rank,
          static_cast<long long*>(a->out));
      ALTO_LAUNCH_CHECK("alto_mttkrp/hot_reduce");
    }
    return ALTO_OK;
  }
  int st = d.n_words == 1 ? (o32 ? fast_w1_f32(d, tab, P, a->value_dtype, a->factor_dtype, s)
                                 : fast_w1_f64(d, tab, P, a->value_dtype, a->factor_dtype, s))
                          : (o32 ? fast_w2_f32(d, tab, P, a->value_dtype, a->factor_dtype, s)
                                 : fast_w2_f64(d, tab, P, a->value_dtype, a->factor_dtype, s));
  if (st == ALTO_EUNSUPPORTED && a->mkeys) return st;  // mode-stream arguments (hot plan) mean nothing to the generic kernel
  if (st == ALTO_EUNSUPPORTED)
    st = d.n_words == 1 ? (o32 ? stream_w1_f32(d, tab, P, a->value_dtype, a->factor_dtype, s)
                                 : stream_w1_f64(d, tab, P, a->value_dtype, a->factor_dtype, s))
                          : (o32 ? stream_w2_f32(d, tab, P, a->value_dtype, a->factor_dtype, s)
                                 : stream_w2_f64(d, tab, P, a->value_dtype, a->factor_dtype, s));
  if (st) return st;
  if (a->hot_base && P.n_hot > 0) {  // per-row copy counts (alto_hot_copies)
    if (a->out_dtype == ALTO_F32)
      hot_reduce_rows_kernel<float><<<(P.n_hot + 7) / 8, 256, 0, s>>>(static_cast<float*>(P.hot_buf), a->hot_rows,
                                                                      a->hot_base, P.n_hot, a->rank,
                                                                      static_cast<float*>(a->out));
    else
      hot_reduce_rows_kernel<double><<<(P.n_hot + 7) / 8, 256, 0, s>>>(static_cast<double*>(P.hot_buf), a->hot_rows,
                                                                       a->hot_base, P.n_hot, a->rank,
                                                                       static_cast<double*>(a->out));
    ALTO_LAUNCH_CHECK("alto_mttkrp/hot_reduce_rows");
  } else if (P.n_hot > 0) {
    const long long nh = static_cast<long long>(P.n_hot) * a->rank;
    const int grid = static_cast<int>((nh + 31) / 32);
    if (a->out_dtype == ALTO_F32)
      hot_reduce_kernel<float><<<grid, 256, 0, s>>>(static_cast<float*>(P.hot_buf), a->hot_rows, P.n_hot, P.hot_copies, a->rank,
                                                     static_cast<float*>(a->out));
    else
      hot_reduce_kernel<double><<<grid, 256, 0, s>>>(static_cast<double*>(P.hot_buf), a->hot_rows, P.n_hot, P.hot_copies, a->rank,
                                                      static_cast<double*>(a->out));
    ALTO_LAUNCH_CHECK("alto_mttkrp/hot_reduce");
  }
  return ALTO_OK;
}

int alto_mstream_block(int32_t order, int32_t rank, int32_t value_dtype, int32_t n_pairs, int32_t* u,
                       int32_t* groups) {
  ALTO_REQUIRE(u && groups, "null output");
  ALTO_REQUIRE(value_dtype == ALTO_F32 || value_dtype == ALTO_F64, "unsupported value dtype");
  if (order < 3 || order > 5 || (rank != 16 && rank != 32) || n_pairs < 0 || n_pairs > 2 ||
      order - 1 - n_pairs < 2 || value_dtype != ALTO_F32)
    return ALTO_EUNSUPPORTED;
  // same rule as ms_u<NV + 1, R, V, 32>() (alto_mstream.cuh): ~32 registers of
  // gathered factor data per lane, at most R/4 elements per group
  const int nv = order - 1 - n_pairs;
  const int vw = value_dtype == ALTO_F32 ? 1 : 2;
  *u = std::min(rank / 4, std::max(1, 32 / (nv * 4 * vw)));
  *groups = 128 / rank;
  return ALTO_OK;
}

int alto_hot_copies(const int64_t* row_ptr, const int32_t* hot_rows, int32_t n_hot, int64_t m, int32_t tile,
                    int32_t flags, int32_t bound, int32_t max_lg, int32_t* hot_code, int32_t* hot_base,
                    void* stream) {
  ALTO_REQUIRE(n_hot >= 0 && tile >= 128 && bound >= 1 && max_lg >= 0 && max_lg <= 20, "bad hot copy plan arguments");
  ALTO_REQUIRE(static_cast<long long>(n_hot) << max_lg < (1ll << 26), "too many hot-row copies");
  if (n_hot == 0) return ALTO_OK;
  cudaStream_t s = as_stream(stream);
  hot_copies_kernel<<<1, 1024, 0, s>>>(reinterpret_cast<const long long*>(row_ptr), hot_rows, n_hot,
                                       (m + tile - 1) / tile, tile, (flags & ALTO_MS_ROW_MAJOR) ? 1 : 0, bound,
                                       max_lg, hot_code, hot_base);
  ALTO_LAUNCH_CHECK("alto_hot_copies");
  return ALTO_OK;
}

int alto_hot_plan(const int64_t* row_ptr, int64_t dim, int64_t tau, int32_t hmax, int32_t* hot_slot,
                  int32_t* hot_rows, int32_t* d_nhot, void* stream) {
  ALTO_REQUIRE(dim >= 0 && dim <= INT_MAX, "hot plan needs mode extents below 2^31");
  ALTO_REQUIRE(hmax >= 0, "hmax must be nonnegative");
  cudaStream_t s = as_stream(stream);
  ALTO_CUDA_TRY(cudaMemsetAsync(d_nhot, 0, sizeof(int32_t), s));
  if (dim > 0)
    hot_plan_kernel<<<grid_for(dim, 256), 256, 0, s>>>(reinterpret_cast<const long long*>(row_ptr), dim, tau, hmax,
                                                        hot_slot, hot_rows, d_nhot);
  clamp_count<<<1, 1, 0, s>>>(d_nhot, hmax);
  ALTO_LAUNCH_CHECK("alto_hot_plan");
  return ALTO_OK;
}

}  // extern "C"

// ---- K14: shared-row pack/unpack for the multi-GPU exchange -----------------
namespace alto {
template <typename T>
__global__ void pack_rows_kernel(const T* __restrict__ src, const long long* __restrict__ rows, long long n, int R,
                                 T* __restrict__ dst, int unpack) {
  const long long total = n * R;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total; i += stride) {
    const long long k = i / R;
    const long long g = rows[k] * R + (i - k * R);
    if (unpack == 2)
      const_cast<T*>(src)[g] += dst[i];  // owner-side reduce of a received partial (rows unique per call)
    else if (unpack)
      const_cast<T*>(src)[g] = dst[i];
    else
      dst[i] = src[g];
  }
}
}  // namespace alto

extern "C" {
int alto_pack_rows(const void* src, int32_t dtype, const int64_t* rows, int64_t n, int32_t rank, void* buf,
                   void* stream) {
  if (n <= 0) return ALTO_OK;
  cudaStream_t s = as_stream(stream);
  const auto* r = reinterpret_cast<const long long*>(rows);
  if (dtype == ALTO_F32)
    pack_rows_kernel<float><<<grid_for(n * rank, 256), 256, 0, s>>>(static_cast<const float*>(src), r, n, rank,
                                                                     static_cast<float*>(buf), 0);
  else
    pack_rows_kernel<double><<<grid_for(n * rank, 256), 256, 0, s>>>(static_cast<const double*>(src), r, n, rank,
                                                                      static_cast<double*>(buf), 0);
  ALTO_LAUNCH_CHECK("alto_pack_rows");
  return ALTO_OK;
}

int alto_unpack_rows(void* dst, int32_t dtype, const int64_t* rows, int64_t n, int32_t rank, const void* buf,
                     void* stream) {
  if (n <= 0) return ALTO_OK;
  cudaStream_t s = as_stream(stream);
  const auto* r = reinterpret_cast<const long long*>(rows);
  if (dtype == ALTO_F32)
    pack_rows_kernel<float><<<grid_for(n * rank, 256), 256, 0, s>>>(static_cast<const float*>(dst), r, n, rank,
                                                                     const_cast<float*>(static_cast<const float*>(buf)),
                                                                     1);
  else
    pack_rows_kernel<double><<<grid_for(n * rank, 256), 256, 0, s>>>(
        static_cast<const double*>(dst), r, n, rank, const_cast<double*>(static_cast<const double*>(buf)), 1);
  ALTO_LAUNCH_CHECK("alto_unpack_rows");
  return ALTO_OK;
}

int alto_add_rows(void* dst, int32_t dtype, const int64_t* rows, int64_t n, int32_t rank, const void* buf,
                  void* stream) {
  if (n <= 0) return ALTO_OK;
  cudaStream_t s = as_stream(stream);
  const auto* r = reinterpret_cast<const long long*>(rows);
  if (dtype == ALTO_F32)
    pack_rows_kernel<float><<<grid_for(n * rank, 256), 256, 0, s>>>(static_cast<const float*>(dst), r, n, rank,
                                                                     const_cast<float*>(static_cast<const float*>(buf)),
                                                                     2);
  else
    pack_rows_kernel<double><<<grid_for(n * rank, 256), 256, 0, s>>>(
        static_cast<const double*>(dst), r, n, rank, const_cast<double*>(static_cast<const double*>(buf)), 2);
  ALTO_LAUNCH_CHECK("alto_add_rows");
  return ALTO_OK;
}
}  // extern "C"

// ---- paired input modes: row-wise product table (mode-stream gathers) --------
namespace alto {
// out[ia * rb + ib][r] = fa[ia][r] * fb[ib][r]; VEC elements per thread
// (float4 stores for float32 when rank % 4 == 0).
template <typename T, int VEC>
__global__ void krp_pair_kernel(const T* __restrict__ fa, const T* __restrict__ fb, long long rb, int R,
                                long long total, T* __restrict__ out) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i * VEC < total; i += stride) {
    const long long e = i * VEC;
    const long long row = e / R;
    const int r = static_cast<int>(e - row * R);
    const long long ia = row / rb, ib = row - ia * rb;
    if constexpr (VEC == 4) {
      const float4 a = __ldg(reinterpret_cast<const float4*>(fa + ia * R + r));
      const float4 b = __ldg(reinterpret_cast<const float4*>(fb + ib * R + r));
      reinterpret_cast<float4*>(out)[i] = make_float4(a.x * b.x, a.y * b.y, a.z * b.z, a.w * b.w);
    } else {
      out[e] = fa[ia * R + r] * fb[ib * R + r];
    }
  }
}
}  // namespace alto

extern "C" int alto_krp_pair(const void* fa, int64_t rows_a, const void* fb, int64_t rows_b, int32_t rank,
                             int32_t dtype, void* out, void* stream) {
  ALTO_REQUIRE(rank >= 1 && rows_a >= 0 && rows_b >= 0, "bad table shape");
  ALTO_REQUIRE(dtype == ALTO_F32 || dtype == ALTO_F64, "unsupported dtype");
  const long long total = static_cast<long long>(rows_a) * rows_b * rank;
  if (total <= 0) return ALTO_OK;
  cudaStream_t s = as_stream(stream);
  if (dtype == ALTO_F32 && rank % 4 == 0)
    krp_pair_kernel<float, 4><<<grid_for(total / 4, 256, kSMs * 8), 256, 0, s>>>(
        static_cast<const float*>(fa), static_cast<const float*>(fb), rows_b, rank, total, static_cast<float*>(out));
  else if (dtype == ALTO_F32)
    krp_pair_kernel<float, 1><<<grid_for(total, 256, kSMs * 8), 256, 0, s>>>(
        static_cast<const float*>(fa), static_cast<const float*>(fb), rows_b, rank, total, static_cast<float*>(out));
  else
    krp_pair_kernel<double, 1><<<grid_for(total, 256, kSMs * 8), 256, 0, s>>>(
        static_cast<const double*>(fa), static_cast<const double*>(fb), rows_b, rank, total,
        static_cast<double*>(out));
  ALTO_LAUNCH_CHECK("alto_krp_pair");
  return ALTO_OK;
}
