// alto_cpd.cu — CP-ALS step on device (K10-K13), replacing the NumPy/SciPy
// arithmetic of pkg/src/altotensor/cpd.py:66-146.
//
// Every reduction is two-stage over a FIXED number of blocks (kRedBlocks)
// with a fixed in-block order, so results are bitwise reproducible from run
// to run, which cpd_als's seed-determinism contract needs
// (pkg/tests/test_cpd.py:125-130).  All arithmetic is float64 (SURVEY §7.3
// item 9: fit parity needs float64 norms and Cholesky even for fp32 data).
#include <cmath>

#include "alto_common.cuh"

namespace alto {

constexpr int kRedBlocks = 256;
constexpr int kRedThreads = 256;
constexpr int kMaxRank = 64;

// ---- K10 gram ---------------------------------------------------------------

template <typename T>
__global__ void __launch_bounds__(kRedThreads) gram_partial(const T* __restrict__ f, long long rows, int R,
                                                            double* __restrict__ part) {
  __shared__ double s_f[32][kMaxRank + 1];
  const long long chunk = (rows + gridDim.x - 1) / gridDim.x;
  const long long r0 = blockIdx.x * chunk;
  const long long r1 = min(rows, r0 + chunk);
  const int RR = R * R;
  double acc[(kMaxRank * kMaxRank + kRedThreads - 1) / kRedThreads];
  const int per = (RR + kRedThreads - 1) / kRedThreads;
  for (int q = 0; q < per; ++q) acc[q] = 0.0;
  for (long long base = r0; base < r1; base += 32) {
    __syncthreads();
    for (int t = threadIdx.x; t < 32 * R; t += blockDim.x) {
      const int k = t / R, c = t - k * R;
      const long long row = base + k;
      s_f[k][c] = row < r1 ? static_cast<double>(f[row * R + c]) : 0.0;
    }
    __syncthreads();
    const int nk = static_cast<int>(min(32ll, r1 - base));
    for (int q = 0; q < per; ++q) {
      const int idx = threadIdx.x + q * kRedThreads;
      if (idx < RR) {
        const int i = idx / R, j = idx - (idx / R) * R;
        double a = acc[q];
        for (int k = 0; k < nk; ++k) a = fma(s_f[k][i], s_f[k][j], a);
        acc[q] = a;
      }
    }
  }
  for (int q = 0; q < per; ++q) {
    const int idx = threadIdx.x + q * kRedThreads;
    if (idx < RR) part[static_cast<long long>(blockIdx.x) * RR + idx] = acc[q];
  }
}

__global__ void sum_partials(const double* __restrict__ part, int nblocks, int width, double* __restrict__ out) {
  for (int idx = threadIdx.x; idx < width; idx += blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nblocks; ++b) s += part[static_cast<long long>(b) * width + idx];
    out[idx] = s;
  }
}

struct GramPtrs {
  const double* g[ALTO_MAX_ORDER];
};

__global__ void hadamard_kernel(const __grid_constant__ GramPtrs G, int order, int skip, int RR,
                                double* __restrict__ v) {
  for (int idx = threadIdx.x; idx < RR; idx += blockDim.x) {
    double x = 1.0;
    for (int n = 0; n < order; ++n)
      if (n != skip) x = __dmul_rn(x, G.g[n][idx]);
    v[idx] = x;
  }
}

// ---- K11 Cholesky + ridge retry ------------------------------------------------

__device__ bool cholesky_lower(double* a, int R) {
  // In place, lower triangle; a is R x R row-major in shared memory.
  for (int j = 0; j < R; ++j) {
    double d = a[j * R + j];
    for (int k = 0; k < j; ++k) d -= a[j * R + k] * a[j * R + k];
    if (!(d > 0.0) || !isfinite(d)) return false;
    const double l = sqrt(d);
    a[j * R + j] = l;
    for (int i = j + 1; i < R; ++i) {
      double s = a[i * R + j];
      for (int k = 0; k < j; ++k) s -= a[i * R + k] * a[j * R + k];
      a[i * R + j] = s / l;
    }
  }
  return true;
}

__global__ void cholesky_kernel(const double* __restrict__ v, int R, double* __restrict__ lout,
                                int* __restrict__ status) {
  __shared__ double s_a[kMaxRank * kMaxRank];
  if (threadIdx.x != 0) return;
  bool finite = true;
  double tr = 0.0;
  if (*status == 2) return;
  for (int i = 0; i < R * R; ++i) {
    s_a[i] = v[i];
    finite &= static_cast<bool>(isfinite(v[i]));
  }
  for (int i = 0; i < R; ++i) tr += v[i * R + i];
  int st = 0;
  if (!(finite && cholesky_lower(s_a, R))) {
    // ridge retry (cpd.py:87-91)
    const double ridge = 1e-12 * tr / R;
    for (int i = 0; i < R * R; ++i) s_a[i] = v[i];
    for (int i = 0; i < R; ++i) s_a[i * R + i] += ridge;
    st = (finite && isfinite(ridge) && cholesky_lower(s_a, R)) ? 1 : 2;
  }
  for (int i = 0; i < R * R; ++i) lout[i] = s_a[i];
  // sticky: a singular solve earlier in the stream stays visible until the
  // host checks (later solves on a poisoned stream are skipped)
  if (st > *status) *status = st;
}

// Row solve x V = m  <=>  L (L^T x^T) = m^T, plus per-block column sum of squares.
__global__ void __launch_bounds__(kRedThreads) solve_rows(const double* __restrict__ lmat,
                                                          const double* __restrict__ mt, long long rows, int R,
                                                          double* __restrict__ x64,
                                                          const int* __restrict__ status,
                                                          double* __restrict__ part) {
  __shared__ double s_l[kMaxRank * kMaxRank];
  __shared__ double s_sq[kRedThreads / 32][kMaxRank];
  if (*status == 2) return;
  for (int i = threadIdx.x; i < R * R; i += blockDim.x) s_l[i] = lmat[i];
  __syncthreads();
  const long long chunk = (rows + gridDim.x - 1) / gridDim.x;
  const long long r0 = blockIdx.x * chunk, r1 = min(rows, r0 + chunk);
  double sq[kMaxRank];
  for (int c = 0; c < R; ++c) sq[c] = 0.0;
  for (long long row = r0 + threadIdx.x; row < r1; row += blockDim.x) {
    double y[kMaxRank];
    for (int i = 0; i < R; ++i) {
      double s = mt[row * R + i];
      for (int k = 0; k < i; ++k) s -= s_l[i * R + k] * y[k];
      y[i] = s / s_l[i * R + i];
    }
    for (int i = R - 1; i >= 0; --i) {
      double s = y[i];
      for (int k = i + 1; k < R; ++k) s -= s_l[k * R + i] * y[k];
      y[i] = s / s_l[i * R + i];
    }
    for (int c = 0; c < R; ++c) {
      x64[row * R + c] = y[c];
      sq[c] += y[c] * y[c];
    }
  }
  // fixed-order block reduction of sq
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int c = 0; c < R; ++c) {
    double s = sq[c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) s_sq[warp][c] = s;
  }
  __syncthreads();
  if (threadIdx.x < R) {
    double s = 0.0;
    for (int w = 0; w < kRedThreads / 32; ++w) s += s_sq[w][threadIdx.x];
    part[static_cast<long long>(blockIdx.x) * R + threadIdx.x] = s;
  }
}

__global__ void lambda_kernel(const double* __restrict__ part, int nblocks, int R, double* __restrict__ lambda,
                              const int* __restrict__ status) {
  if (*status == 2) return;
  for (int c = threadIdx.x; c < R; c += blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nblocks; ++b) s += part[static_cast<long long>(b) * R + c];
    lambda[c] = sqrt(s);
  }
}

__global__ void sqrt_kernel(const double* __restrict__ sumsq, int R, double* __restrict__ lambda,
                            const int* __restrict__ status) {
  if (*status == 2) return;
  for (int c = threadIdx.x; c < R; c += blockDim.x) lambda[c] = sqrt(sumsq[c]);
}

__global__ void normalize_kernel(double* __restrict__ x64, float* __restrict__ x32, long long rows, int R,
                                 const double* __restrict__ lambda, const int* __restrict__ status) {
  if (*status == 2) return;
  const long long n = rows * R;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n; i += stride) {
    const int c = static_cast<int>(i % R);
    const double w = lambda[c];
    const double x = x64[i] / (w == 0.0 ? 1.0 : w);
    x64[i] = x;
    if (x32) x32[i] = static_cast<float>(x);
  }
}

// ---- K13 fit terms / norms ---------------------------------------------------------

__device__ __forceinline__ double block_sum_fixed(double v, double* s_tmp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if (lane == 0) s_tmp[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += s_tmp[w];
  return s;
}

__global__ void __launch_bounds__(kRedThreads) inner_partial(const double* __restrict__ mt,
                                                             const double* __restrict__ f,
                                                             const double* __restrict__ lambda, long long rows,
                                                             int R, double* __restrict__ part) {
  __shared__ double s_tmp[32];
  const long long n = rows * R;
  const long long chunk = (n + gridDim.x - 1) / gridDim.x;
  const long long i0 = blockIdx.x * chunk, i1 = min(n, i0 + chunk);
  double s = 0.0;
  for (long long i = i0 + threadIdx.x; i < i1; i += blockDim.x) s += (mt[i] * f[i]) * lambda[i % R];
  s = block_sum_fixed(s, s_tmp);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void fit_final(const double* __restrict__ part, int nblocks, const double* __restrict__ lambda,
                          const double* __restrict__ vall, int R, double* __restrict__ out2) {
  if (threadIdx.x != 0) return;
  double s = 0.0;
  for (int b = 0; b < nblocks; ++b) s += part[b];
  out2[0] = s;
  double q = 0.0;
  for (int j = 0; j < R; ++j) {
    double u = 0.0;
    for (int i = 0; i < R; ++i) u += lambda[i] * vall[i * R + j];
    q += u * lambda[j];
  }
  out2[1] = q;
}

template <typename T>
__global__ void __launch_bounds__(kRedThreads) sumsq_partial(const T* __restrict__ v, long long n,
                                                             double* __restrict__ part) {
  __shared__ double s_tmp[32];
  const long long chunk = (n + gridDim.x - 1) / gridDim.x;
  const long long i0 = blockIdx.x * chunk, i1 = min(n, i0 + chunk);
  double s = 0.0;
  for (long long i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    const double x = static_cast<double>(v[i]);
    s += x * x;
  }
  s = block_sum_fixed(s, s_tmp);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void sum_scalar(const double* __restrict__ part, int nblocks, double* __restrict__ out) {
  if (threadIdx.x != 0) return;
  double s = 0.0;
  for (int b = 0; b < nblocks; ++b) s += part[b];
  *out = s;
}

__global__ void cast_kernel(const double* __restrict__ in, float* __restrict__ out, long long n) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n; i += stride)
    out[i] = static_cast<float>(in[i]);
}

// ---- fused factor update (K11 + K12 + K10 for ranks 16 / 32) -------------------
// Two streaming passes over the rows of M (float32 or float64), each row
// solved in registers against the Cholesky factor in shared memory
// (forward + back substitution, reciprocal pivots):
//   pass 1: column sums of squares of X = M V^-1 (per-block, fixed order);
//   pass 2: X again, scaled by 1/lambda (zero-safe), written as float64 (and
//           float32 gather copy) through a shared-memory tile (coalesced),
//           plus the block's partial Gram X^T X from the same tile.
// Rows are staged through shared memory so every global access is coalesced.
constexpr int kUpdBlocks = 1024;

template <int R>
struct UpdCfg {
  static constexpr int THREADS = R <= 16 ? 256 : 96;  // static smem < 48 KB
  static constexpr int MINB = R <= 16 ? 3 : 2;
  static constexpr int LD = R + 1;  // padded row stride (doubles) of the tile
};

__device__ __forceinline__ double2 lds2(const double* p) {
  // volatile: re-loaded every use (broadcast LDS.128) rather than hoisted into registers
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y)
               : "r"(static_cast<unsigned>(__cvta_generic_to_shared(p))));
  return v;
}

template <int R, typename MT, bool PASS2>
__global__ void __launch_bounds__(UpdCfg<R>::THREADS, UpdCfg<R>::MINB) update_pass(const double* __restrict__ lmat,
                                                                 const MT* __restrict__ mt, long long rows,
                                                                 const double* __restrict__ lambda,
                                                                 double* __restrict__ x64, float* __restrict__ x32,
                                                                 const int* __restrict__ status,
                                                                 double* __restrict__ part) {
  constexpr int TH = UpdCfg<R>::THREADS;
  constexpr int NWARP = TH / 32;
  constexpr int LD = UpdCfg<R>::LD;
  constexpr int GL = R * R / 32;  // Gram entries per lane: row gi, columns gj0 .. gj0+GL-1
  __shared__ __align__(16) double s_l[R * R];   // L, row-major
  __shared__ __align__(16) double s_lt[R * R];  // L^T, row-major
  __shared__ double s_rd[R];
  __shared__ double s_scale[R];
  __shared__ double s_t[TH * LD];
  __shared__ double s_red[NWARP][R];
  if (*status == 2) return;
  for (int i = threadIdx.x; i < R * R; i += TH) {
    const double v = lmat[i];
    s_l[i] = v;
    s_lt[(i % R) * R + i / R] = v;
  }
  __syncthreads();
  if (threadIdx.x < R) {
    s_rd[threadIdx.x] = 1.0 / s_l[threadIdx.x * R + threadIdx.x];
    if constexpr (PASS2) {
      // reciprocal of lambda (zero-safe): one multiply per element instead of
      // a float64 division (within 1 ulp of x / lambda)
      const double w = lambda[threadIdx.x];
      s_scale[threadIdx.x] = 1.0 / (w == 0.0 ? 1.0 : w);
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gi = (lane * GL) / R, gj0 = (lane * GL) % R;
  const long long chunk = (rows + gridDim.x - 1) / gridDim.x;
  const long long r0 = blockIdx.x * chunk, r1 = min(rows, r0 + chunk);
  // pass 1: lane owns column (lane % R) of rows phase (lane / R) of its warp's
  // tile rows; pass 2: lane owns Gram entries (gi, gj0 .. gj0+GL-1)
  constexpr int RPW = 32 / R;  // rows per warp step (pass 1)
  double sq = 0.0;
  double g[PASS2 ? GL : 1];
#pragma unroll
  for (int q = 0; q < (PASS2 ? GL : 1); ++q) g[q] = 0.0;
  for (long long base = r0; base < r1; base += TH) {
    const int nr = static_cast<int>(min(static_cast<long long>(TH), r1 - base));
    __syncthreads();
    for (int e = threadIdx.x; e < nr * R; e += TH) {
      const int r = e / R, c = e - r * R;
      s_t[r * LD + c] = static_cast<double>(mt[base * R + e]);
    }
    __syncthreads();
    double y[R];
    if (threadIdx.x < nr) {
      // forward: L y = m (row i of L, pairs of k); back: L^T x = y (row i of L^T)
#pragma unroll
      for (int i = 0; i < R; ++i) {
        double v = s_t[threadIdx.x * LD + i];
#pragma unroll
        for (int k = 0; k + 1 < i; k += 2) {
          const double2 l = lds2(s_l + i * R + k);
          v -= l.x * y[k];
          v -= l.y * y[k + 1];
        }
        if (i & 1) v -= s_l[i * R + i - 1] * y[i - 1];
        y[i] = v * s_rd[i];
      }
#pragma unroll
      for (int i = R - 1; i >= 0; --i) {
        double v = y[i];
        int k = i + 1;
        if (k & 1) {
          if (k < R) v -= s_lt[i * R + k] * y[k];
          ++k;
        }
#pragma unroll
        for (; k + 1 < R + 1 && k < R; k += 2) {
          const double2 l = lds2(s_lt + i * R + k);
          v -= l.x * y[k];
          v -= l.y * y[k + 1];
        }
        y[i] = v * s_rd[i];
      }
    }
    if constexpr (!PASS2) {
      __syncthreads();
      if (threadIdx.x < nr) {
#pragma unroll
        for (int c = 0; c < R; ++c) s_t[threadIdx.x * LD + c] = y[c];
      }
      __syncthreads();
      for (int r = warp * RPW + lane / R; r < nr; r += NWARP * RPW) {
        const double v = s_t[r * LD + (lane % R)];
        sq = fma(v, v, sq);
      }
    }
    if constexpr (PASS2) {
      __syncthreads();
      if (threadIdx.x < nr) {
#pragma unroll
        for (int c = 0; c < R; ++c) s_t[threadIdx.x * LD + c] = y[c] * s_scale[c];
      }
      __syncthreads();
      for (int e = threadIdx.x; e < nr * R; e += TH) {
        const int r = e / R, c = e - r * R;
        const double v = s_t[r * LD + c];
        x64[base * R + e] = v;
        if (x32) x32[base * R + e] = static_cast<float>(v);
      }
      // Gram partial: warp w takes rows w, w+NWARP, ...; lane owns entries
      // (gi, gj0 .. gj0+GL-1) of the R x R block
      for (int r = warp; r < nr; r += NWARP) {
        const double xi = s_t[r * LD + gi];
#pragma unroll
        for (int q = 0; q < GL; ++q) g[q] = fma(xi, s_t[r * LD + gj0 + q], g[q]);
      }
    }
  }
  if constexpr (!PASS2) {
    // lanes c, c+R, ... of a warp hold column c: fixed-order fold, then warps in order
    double v = sq;
#pragma unroll
    for (int o = 16; o >= R; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane < R) s_red[warp][lane] = v;
    __syncthreads();
    if (threadIdx.x < R) {
      double t = 0.0;
      for (int w = 0; w < NWARP; ++w) t += s_red[w][threadIdx.x];
      part[static_cast<long long>(blockIdx.x) * R + threadIdx.x] = t;
    }
  } else {
    static_assert(NWARP * R * R <= TH * LD, "Gram reduction reuses the row tile");
    __syncthreads();
#pragma unroll
    for (int q = 0; q < GL; ++q) s_t[warp * R * R + gi * R + gj0 + q] = g[q];
    __syncthreads();
    for (int idx = threadIdx.x; idx < R * R; idx += TH) {
      double v = 0.0;
      for (int w = 0; w < NWARP; ++w) v += s_t[w * R * R + idx];
      part[static_cast<long long>(blockIdx.x) * R * R + idx] = v;
    }
  }
}

// out[idx] = sum over b of part[b * width + idx], a warp per entry: lane l sums
// blocks l, l+32, ... in order, then a fixed shuffle tree (deterministic).
__global__ void sum_partials_warp(const double* __restrict__ part, int nblocks, int width, double* __restrict__ out,
                                  int do_sqrt, const int* __restrict__ status) {
  if (status && *status == 2) return;
  const int idx = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (idx >= width) return;
  double s = 0.0;
  for (int b = lane; b < nblocks; b += 32) s += part[static_cast<long long>(b) * width + idx];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if (lane == 0) out[idx] = do_sqrt ? sqrt(s) : s;
}

// ---- rank-16 update on the float64 tensor cores (DMMA m8n8k4) ------------------
// X = M W (W = V^-1 from the Cholesky factor) and the Gram X^T X are
// GEMM-shaped, so rank 16 runs them as mma.sync m8n8k4 f64 (exact float64
// products and sums, like the scalar path up to summation order).  A warp
// takes 8 rows at a time: each lane loads 4 consecutive entries of its row
// (row = lane/4, columns 4*(lane%4) .. +3: one coalesced 16-byte load) and
// uses entry ks in k-step ks, so MMA k-index t stands for column 4t+ks; the
// W fragments are permuted the same way and stay in registers.  Pass 1 sums
// the squares of X per column; pass 2 scales by 1/lambda, writes X (float64
// + float32 copy) and accumulates X^T X from a per-warp 8x16 shared tile.

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

constexpr int kTcThreads = 256;

template <int R, typename MT, bool PASS2>
__global__ void __launch_bounds__(kTcThreads) update_tc(const double* __restrict__ w, const MT* __restrict__ mt,
                                                        long long rows, const double* __restrict__ lambda,
                                                        double* __restrict__ x64, float* __restrict__ x32,
                                                        const int* __restrict__ status, double* __restrict__ part) {
  constexpr int KS = R / 4;  // k-steps: a lane holds KS consecutive entries of its row
  constexpr int NT = R / 8;  // 8-column tiles
  constexpr int NW = kTcThreads / 32;
  constexpr int PER = R * R / kTcThreads;  // Gram entries summed per thread at the end
  __shared__ double s_x[NW][8][R + 1];
  __shared__ double s_red[R * R];
  if (*status == 2) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  // B fragments of W: k-step ks, n-tile nt: W[KS*tig + ks][8*nt + gid]
  double bw[KS][NT];
#pragma unroll
  for (int ks = 0; ks < KS; ++ks)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) bw[ks][nt] = w[(KS * tig + ks) * R + 8 * nt + gid];
  double rl[NT][2];  // 1/lambda of this lane's output columns 8*nt + 2*tig + {0,1}
  if constexpr (PASS2) {
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const double l = lambda[8 * nt + 2 * tig + q];
        rl[nt][q] = 1.0 / (l == 0.0 ? 1.0 : l);
      }
  }
  double sq[NT][2] = {};
  double g[PASS2 ? NT : 1][PASS2 ? NT : 1][2] = {};  // Gram tile (mt, nt), fragment entries
  const long long groups = (rows + 7) / 8;
  const long long gpb = (groups + gridDim.x - 1) / gridDim.x;  // 8-row groups per block (contiguous)
  const long long g0 = blockIdx.x * gpb, g1 = min(groups, g0 + gpb);
  for (long long grp = g0 + warp; grp < g1; grp += NW) {
    const long long row = grp * 8 + gid;
    double a[KS];
#pragma unroll
    for (int q = 0; q < KS; ++q) a[q] = 0.0;
    if (row < rows) {
      if constexpr (sizeof(MT) == 4) {
#pragma unroll
        for (int q = 0; q < KS; q += 4) {
          const float4 v = __ldg(reinterpret_cast<const float4*>(mt + row * R + KS * tig + q));
          a[q] = v.x; a[q + 1] = v.y; a[q + 2] = v.z; a[q + 3] = v.w;
        }
      } else {
#pragma unroll
        for (int q = 0; q < KS; q += 2) {
          const double2 v = __ldg(reinterpret_cast<const double2*>(mt + row * R + KS * tig + q));
          a[q] = v.x; a[q + 1] = v.y;
        }
      }
    }
    double c[NT][2] = {};  // X[gid][8*nt + 2*tig + q]
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) dmma(c[nt], a[ks], bw[ks][nt]);
    if constexpr (!PASS2) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int q = 0; q < 2; ++q) sq[nt][q] = fma(c[nt][q], c[nt][q], sq[nt][q]);
    } else {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int q = 0; q < 2; ++q) c[nt][q] = row < rows ? c[nt][q] * rl[nt][q] : 0.0;
      if (row < rows) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          *reinterpret_cast<double2*>(x64 + row * R + 8 * nt + 2 * tig) = make_double2(c[nt][0], c[nt][1]);
          if (x32)
            *reinterpret_cast<float2*>(x32 + row * R + 8 * nt + 2 * tig) =
                make_float2(static_cast<float>(c[nt][0]), static_cast<float>(c[nt][1]));
        }
      }
      __syncwarp();
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int q = 0; q < 2; ++q) s_x[warp][gid][8 * nt + 2 * tig + q] = c[nt][q];
      __syncwarp();
      // G(mt, nt) += X[:, 8mt..]^T X[:, 8nt..] over the 8 rows (2 k-steps of 4)
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        double fa[NT];
#pragma unroll
        for (int t = 0; t < NT; ++t) fa[t] = s_x[warp][4 * ks + tig][8 * t + gid];
#pragma unroll
        for (int mt2 = 0; mt2 < NT; ++mt2)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) dmma(g[mt2][nt], fa[mt2], fa[nt]);
      }
    }
  }
  if constexpr (!PASS2) {
    // column (8nt + 2tig + q) partials live in lanes with the same tig: fold gid
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        double v = sq[nt][q];
#pragma unroll
        for (int o = 16; o >= 4; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        if (gid == 0) s_x[warp][0][8 * nt + 2 * tig + q] = v;
      }
    __syncthreads();
    if (threadIdx.x < R) {
      double t = 0.0;
      for (int w2 = 0; w2 < NW; ++w2) t += s_x[w2][0][threadIdx.x];
      part[static_cast<long long>(blockIdx.x) * R + threadIdx.x] = t;
    }
  } else {
    // warps' Gram fragments summed in warp order through one R x R buffer
    double t[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) t[q] = 0.0;
    for (int w2 = 0; w2 < NW; ++w2) {
      __syncthreads();
      if (warp == w2) {
#pragma unroll
        for (int mt2 = 0; mt2 < NT; ++mt2)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int q = 0; q < 2; ++q) s_red[(8 * mt2 + gid) * R + 8 * nt + 2 * tig + q] = g[mt2][nt][q];
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < PER; ++q) t[q] += s_red[threadIdx.x + q * kTcThreads];
    }
#pragma unroll
    for (int q = 0; q < PER; ++q) part[static_cast<long long>(blockIdx.x) * R * R + threadIdx.x + q * kTcThreads] = t[q];
  }
}

// Cholesky of V with the ridge retry of cholesky_kernel (cpd.py:80-95) and
// W = V^-1 = L^-T L^-1, by one warp (rank <= 32): column j of L is one
// warp reduction for the pivot plus one lane per row below it; column j of
// L^-1 is lane j's forward substitution; W entries are spread over lanes.
template <int R>
__global__ void chol_inv_kernel(const double* __restrict__ v, double* __restrict__ w, int* __restrict__ status) {
  static_assert(R <= 32, "one lane per row");
  __shared__ double a[R][R + 1];
  __shared__ double z[R][R + 1];
  const int lane = threadIdx.x;
  if (*status == 2) return;
  bool finite = true;
  double tr = 0.0;
  for (int i = 0; i < R; ++i) {
    const double x = lane < R ? v[i * R + lane] : 0.0;
    finite &= static_cast<bool>(isfinite(x));
    if (lane == i) tr = x;
  }
  finite = __all_sync(0xffffffffu, finite);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) tr += __shfl_xor_sync(0xffffffffu, tr, o);  // trace (all lanes)
  auto factor = [&](double ridge) -> bool {
    if (lane < R)
      for (int i = 0; i < R; ++i) a[i][lane] = v[i * R + lane] + (i == lane ? ridge : 0.0);
    __syncwarp();
    for (int j = 0; j < R; ++j) {
      double t = lane < j ? a[j][lane] * a[j][lane] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      const double d = a[j][j] - t;
      if (!(d > 0.0) || !isfinite(d)) return false;  // warp-uniform
      const double l = sqrt(d);
      if (lane > j && lane < R) {
        double sum = a[lane][j];
        for (int k = 0; k < j; ++k) sum -= a[lane][k] * a[j][k];
        a[lane][j] = sum / l;
      }
      __syncwarp();
      if (lane == 0) a[j][j] = l;
      __syncwarp();
    }
    return true;
  };
  int st = 0;
  if (!(finite && factor(0.0))) {
    const double ridge = 1e-12 * tr / R;
    st = (finite && isfinite(ridge) && factor(ridge)) ? 1 : 2;
  }
  if (st == 2) {
    if (lane == 0 && st > *status) *status = st;
    return;
  }
  if (lane < R) {  // column `lane` of L^-1
    const int j = lane;
    for (int i = 0; i < R; ++i) {
      double x = i == j ? 1.0 : 0.0;
      for (int k = j; k < i; ++k) x -= a[i][k] * z[k][j];
      z[i][j] = i < j ? 0.0 : x / a[i][i];
    }
  }
  __syncwarp();
  for (int idx = lane; idx < R * R; idx += 32) {
    const int r = idx / R, c = idx % R;
    double x = 0.0;
    for (int k = (r > c ? r : c); k < R; ++k) x += z[k][r] * z[k][c];
    w[idx] = x;
  }
  if (lane == 0 && st > *status) *status = st;
}

template <int R, typename MT>
int update_tc_impl(const double* v, const MT* m, long long rows, double* x64, float* x32, double* lambda,
                   double* gram, int* d_status, double* ws, cudaStream_t s) {
  double* part = ws;
  double* lmat = ws + static_cast<size_t>(kUpdBlocks) * R * R;
  double* winv = lmat + R * R;
  chol_inv_kernel<R><<<1, 32, 0, s>>>(v, winv, d_status);
  (void)lmat;
  update_tc<R, MT, false><<<kUpdBlocks, kTcThreads, 0, s>>>(winv, m, rows, nullptr, x64, x32, d_status, part);
  sum_partials_warp<<<(R + 7) / 8, 256, 0, s>>>(part, kUpdBlocks, R, lambda, 1, d_status);
  update_tc<R, MT, true><<<kUpdBlocks, kTcThreads, 0, s>>>(winv, m, rows, lambda, x64, x32, d_status, part);
  sum_partials_warp<<<(R * R + 7) / 8, 256, 0, s>>>(part, kUpdBlocks, R * R, gram, 0, d_status);
  ALTO_LAUNCH_CHECK("alto_cpd_update(tc)");
  return ALTO_OK;
}

template <int R, typename MT>
int update_impl(const double* v, const MT* m, long long rows, double* x64, float* x32, double* lambda, double* gram,
                int* d_status, double* ws, cudaStream_t s) {
  double* part = ws;
  double* lmat = ws + static_cast<size_t>(kUpdBlocks) * R * R;
  cholesky_kernel<<<1, 32, 0, s>>>(v, R, lmat, d_status);
  update_pass<R, MT, false><<<kUpdBlocks, UpdCfg<R>::THREADS, 0, s>>>(lmat, m, rows, nullptr, x64, x32, d_status,
                                                                      part);
  sum_partials_warp<<<(R + 7) / 8, 256, 0, s>>>(part, kUpdBlocks, R, lambda, 1, d_status);
  update_pass<R, MT, true><<<kUpdBlocks, UpdCfg<R>::THREADS, 0, s>>>(lmat, m, rows, lambda, x64, x32, d_status,
                                                                     part);
  sum_partials_warp<<<(R * R + 7) / 8, 256, 0, s>>>(part, kUpdBlocks, R * R, gram, 0, d_status);
  ALTO_LAUNCH_CHECK("alto_cpd_update");
  return ALTO_OK;
}

static size_t cpd_ws_doubles(int R) {
  return static_cast<size_t>(kUpdBlocks) * R * R + 2 * static_cast<size_t>(R) * R + 64;
}

}  // namespace alto

using namespace alto;

extern "C" {

size_t alto_cpd_workspace_bytes(int32_t rank) {
  if (rank < 1) rank = 1;
  return cpd_ws_doubles(rank) * sizeof(double);
}

int alto_gram(const void* f, int32_t f_dtype, int64_t rows, int32_t rank, double* g, void* ws, size_t ws_bytes,
              void* stream) {
  ALTO_REQUIRE(rank >= 1 && rank <= kMaxRank, "rank must be in [1, 64]");
  ALTO_REQUIRE(ws && ws_bytes >= alto_cpd_workspace_bytes(rank), "cpd workspace too small");
  cudaStream_t s = as_stream(stream);
  auto* part = static_cast<double*>(ws);
  if (f_dtype == ALTO_F32)
    gram_partial<float><<<kRedBlocks, kRedThreads, 0, s>>>(static_cast<const float*>(f), rows, rank, part);
  else
    gram_partial<double><<<kRedBlocks, kRedThreads, 0, s>>>(static_cast<const double*>(f), rows, rank, part);
  sum_partials<<<1, 256, 0, s>>>(part, kRedBlocks, rank * rank, g);
  ALTO_LAUNCH_CHECK("alto_gram");
  return ALTO_OK;
}

int alto_hadamard_grams(const double* const* grams_host_array, int32_t order, int32_t skip, int32_t rank, double* v,
                        void* stream) {
  ALTO_REQUIRE(order >= 1 && order <= ALTO_MAX_ORDER, "order out of range");
  ALTO_REQUIRE(rank >= 1 && rank <= kMaxRank, "rank must be in [1, 64]");
  GramPtrs G{};
  for (int n = 0; n < order; ++n) G.g[n] = grams_host_array[n];
  hadamard_kernel<<<1, 256, 0, as_stream(stream)>>>(G, order, skip, rank * rank, v);
  ALTO_LAUNCH_CHECK("alto_hadamard_grams");
  return ALTO_OK;
}

int alto_solve_normalize(const double* v, const double* mttkrp, int64_t rows, int32_t rank, double* x64, float* x32,
                         double* lambda, int32_t* d_status, void* ws, size_t ws_bytes, void* stream) {
  ALTO_REQUIRE(rank >= 1 && rank <= kMaxRank, "rank must be in [1, 64]");
  ALTO_REQUIRE(ws && ws_bytes >= alto_cpd_workspace_bytes(rank), "cpd workspace too small");
  cudaStream_t s = as_stream(stream);
  auto* part = static_cast<double*>(ws);
  double* lmat = part + static_cast<size_t>(kRedBlocks) * rank * rank;
  cholesky_kernel<<<1, 32, 0, s>>>(v, rank, lmat, d_status);
  solve_rows<<<kRedBlocks, kRedThreads, 0, s>>>(lmat, mttkrp, rows, rank, x64, d_status, part);
  lambda_kernel<<<1, 64, 0, s>>>(part, kRedBlocks, rank, lambda, d_status);
  normalize_kernel<<<grid_for(rows * rank, 256), 256, 0, s>>>(x64, x32, rows, rank, lambda, d_status);
  ALTO_LAUNCH_CHECK("alto_solve_normalize");
  return ALTO_OK;
}

int alto_cpd_update(const double* v, const void* mttkrp, int32_t m_dtype, int64_t rows, int32_t rank, double* x64,
                    float* x32, double* lambda, double* gram, int32_t* d_status, int32_t flags, void* ws,
                    size_t ws_bytes, void* stream) {
  ALTO_REQUIRE(m_dtype == ALTO_F32 || m_dtype == ALTO_F64, "mttkrp dtype must be float32 or float64");
  ALTO_REQUIRE(ws && ws_bytes >= alto_cpd_workspace_bytes(rank), "cpd workspace too small");
  if (rank != 16 && rank != 32) {
    set_error("fused factor update supports ranks 16 and 32");
    return ALTO_EUNSUPPORTED;
  }
  cudaStream_t s = as_stream(stream);
  auto* w = static_cast<double*>(ws);
  const bool scalar = (flags & 1) != 0;  // ALTO_CPD_SCALAR: substitution kernels instead of DMMA
  if (rank == 16 && !scalar)
    return m_dtype == ALTO_F32 ? update_tc_impl<16>(v, static_cast<const float*>(mttkrp), rows, x64, x32, lambda,
                                                    gram, d_status, w, s)
                               : update_tc_impl<16>(v, static_cast<const double*>(mttkrp), rows, x64, x32, lambda,
                                                    gram, d_status, w, s);
  if (rank == 32 && !scalar)
    return m_dtype == ALTO_F32 ? update_tc_impl<32>(v, static_cast<const float*>(mttkrp), rows, x64, x32, lambda,
                                                    gram, d_status, w, s)
                               : update_tc_impl<32>(v, static_cast<const double*>(mttkrp), rows, x64, x32, lambda,
                                                    gram, d_status, w, s);
  if (rank == 16)
    return m_dtype == ALTO_F32 ? update_impl<16>(v, static_cast<const float*>(mttkrp), rows, x64, x32, lambda, gram,
                                                 d_status, w, s)
                               : update_impl<16>(v, static_cast<const double*>(mttkrp), rows, x64, x32, lambda,
                                                 gram, d_status, w, s);
  return m_dtype == ALTO_F32 ? update_impl<32>(v, static_cast<const float*>(mttkrp), rows, x64, x32, lambda, gram,
                                               d_status, w, s)
                             : update_impl<32>(v, static_cast<const double*>(mttkrp), rows, x64, x32, lambda, gram,
                                               d_status, w, s);
}

int alto_fit_terms(const double* mttkrp, const double* f, const double* lambda, const double* v_all, int64_t rows,
                   int32_t rank, double* out2, void* ws, size_t ws_bytes, void* stream) {
  ALTO_REQUIRE(rank >= 1 && rank <= kMaxRank, "rank must be in [1, 64]");
  ALTO_REQUIRE(ws && ws_bytes >= alto_cpd_workspace_bytes(rank), "cpd workspace too small");
  cudaStream_t s = as_stream(stream);
  auto* part = static_cast<double*>(ws);
  inner_partial<<<kRedBlocks, kRedThreads, 0, s>>>(mttkrp, f, lambda, rows, rank, part);
  fit_final<<<1, 32, 0, s>>>(part, kRedBlocks, lambda, v_all, rank, out2);
  ALTO_LAUNCH_CHECK("alto_fit_terms");
  return ALTO_OK;
}

int alto_sumsq(const void* values, int32_t dtype, int64_t m, double* out, void* ws, size_t ws_bytes, void* stream) {
  ALTO_REQUIRE(ws && ws_bytes >= kRedBlocks * sizeof(double), "workspace too small");
  cudaStream_t s = as_stream(stream);
  auto* part = static_cast<double*>(ws);
  if (dtype == ALTO_F32)
    sumsq_partial<float><<<kRedBlocks, kRedThreads, 0, s>>>(static_cast<const float*>(values), m, part);
  else
    sumsq_partial<double><<<kRedBlocks, kRedThreads, 0, s>>>(static_cast<const double*>(values), m, part);
  sum_scalar<<<1, 32, 0, s>>>(part, kRedBlocks, out);
  ALTO_LAUNCH_CHECK("alto_sumsq");
  return ALTO_OK;
}

int alto_cast_f64_f32(const double* in, float* out, int64_t n, void* stream) {
  if (n <= 0) return ALTO_OK;
  cast_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(in, out, n);
  ALTO_LAUNCH_CHECK("alto_cast_f64_f32");
  return ALTO_OK;
}

}  // extern "C"

// ---- distributed (key-range sharded) CP-ALS pieces --------------------------
// A shard owns a subset of output rows (rows only it touches, plus shared
// rows it is the designated owner of); sums over rows (Gram, column norms,
// fit inner product) take a 0/1 row mask so that every row is counted by
// exactly one shard before the cross-shard all-reduce.

namespace alto {

template <typename T>
__global__ void __launch_bounds__(kRedThreads) gram_partial_masked(const T* __restrict__ f, long long rows, int R,
                                                                   const unsigned char* __restrict__ mask,
                                                                   double* __restrict__ part) {
  __shared__ double s_f[32][kMaxRank + 1];
  const long long chunk = (rows + gridDim.x - 1) / gridDim.x;
  const long long r0 = blockIdx.x * chunk;
  const long long r1 = min(rows, r0 + chunk);
  const int RR = R * R;
  double acc[(kMaxRank * kMaxRank + kRedThreads - 1) / kRedThreads];
  const int per = (RR + kRedThreads - 1) / kRedThreads;
  for (int q = 0; q < per; ++q) acc[q] = 0.0;
  for (long long base = r0; base < r1; base += 32) {
    __syncthreads();
    for (int t = threadIdx.x; t < 32 * R; t += blockDim.x) {
      const int k = t / R, c = t - k * R;
      const long long row = base + k;
      const bool on = row < r1 && (mask == nullptr || mask[row]);
      s_f[k][c] = on ? static_cast<double>(f[row * R + c]) : 0.0;
    }
    __syncthreads();
    const int nk = static_cast<int>(min(32ll, r1 - base));
    for (int q = 0; q < per; ++q) {
      const int idx = threadIdx.x + q * kRedThreads;
      if (idx < RR) {
        const int i = idx / R, j = idx - (idx / R) * R;
        double a = acc[q];
        for (int k = 0; k < nk; ++k) a = fma(s_f[k][i], s_f[k][j], a);
        acc[q] = a;
      }
    }
  }
  for (int q = 0; q < per; ++q) {
    const int idx = threadIdx.x + q * kRedThreads;
    if (idx < RR) part[static_cast<long long>(blockIdx.x) * RR + idx] = acc[q];
  }
}

__global__ void __launch_bounds__(kRedThreads) colsumsq_partial(const double* __restrict__ x, long long rows, int R,
                                                                const unsigned char* __restrict__ mask,
                                                                double* __restrict__ part) {
  __shared__ double s_sq[kRedThreads / 32][kMaxRank];
  const long long chunk = (rows + gridDim.x - 1) / gridDim.x;
  const long long r0 = blockIdx.x * chunk, r1 = min(rows, r0 + chunk);
  double sq[kMaxRank];
  for (int c = 0; c < R; ++c) sq[c] = 0.0;
  for (long long row = r0 + threadIdx.x; row < r1; row += blockDim.x) {
    if (mask && !mask[row]) continue;
    for (int c = 0; c < R; ++c) {
      const double y = x[row * R + c];
      sq[c] += y * y;
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int c = 0; c < R; ++c) {
    double s = sq[c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) s_sq[warp][c] = s;
  }
  __syncthreads();
  if (threadIdx.x < R) {
    double s = 0.0;
    for (int w = 0; w < kRedThreads / 32; ++w) s += s_sq[w][threadIdx.x];
    part[static_cast<long long>(blockIdx.x) * R + threadIdx.x] = s;
  }
}

__global__ void __launch_bounds__(kRedThreads) inner_partial_masked(const double* __restrict__ mt,
                                                                    const double* __restrict__ f,
                                                                    const double* __restrict__ lambda,
                                                                    long long rows, int R,
                                                                    const unsigned char* __restrict__ mask,
                                                                    double* __restrict__ part) {
  __shared__ double s_tmp[32];
  const long long n = rows * R;
  const long long chunk = (n + gridDim.x - 1) / gridDim.x;
  const long long i0 = blockIdx.x * chunk, i1 = min(n, i0 + chunk);
  double s = 0.0;
  for (long long i = i0 + threadIdx.x; i < i1; i += blockDim.x)
    if (mask == nullptr || mask[i / R]) s += (mt[i] * f[i]) * lambda[i % R];
  s = block_sum_fixed(s, s_tmp);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

}  // namespace alto

extern "C" {

int alto_gram_masked(const void* f, int32_t f_dtype, int64_t rows, int32_t rank, const uint8_t* row_mask,
                     double* g_partial, void* ws, size_t ws_bytes, void* stream) {
  ALTO_REQUIRE(rank >= 1 && rank <= kMaxRank, "rank must be in [1, 64]");
  ALTO_REQUIRE(ws && ws_bytes >= alto_cpd_workspace_bytes(rank), "cpd workspace too small");
  cudaStream_t s = as_stream(stream);
  auto* part = static_cast<double*>(ws);
  if (f_dtype == ALTO_F32)
    gram_partial_masked<float><<<kRedBlocks, kRedThreads, 0, s>>>(static_cast<const float*>(f), rows, rank,
                                                                  row_mask, part);
  else
    gram_partial_masked<double><<<kRedBlocks, kRedThreads, 0, s>>>(static_cast<const double*>(f), rows, rank,
                                                                   row_mask, part);
  sum_partials<<<1, 256, 0, s>>>(part, kRedBlocks, rank * rank, g_partial);
  ALTO_LAUNCH_CHECK("alto_gram_masked");
  return ALTO_OK;
}

int alto_solve_rows(const double* v, const double* mttkrp, int64_t rows, int32_t rank, double* x64,
                    int32_t* d_status, void* ws, size_t ws_bytes, void* stream) {
  ALTO_REQUIRE(rank >= 1 && rank <= kMaxRank, "rank must be in [1, 64]");
  ALTO_REQUIRE(ws && ws_bytes >= alto_cpd_workspace_bytes(rank), "cpd workspace too small");
  cudaStream_t s = as_stream(stream);
  auto* part = static_cast<double*>(ws);
  double* lmat = part + static_cast<size_t>(kRedBlocks) * rank * rank;
  cholesky_kernel<<<1, 32, 0, s>>>(v, rank, lmat, d_status);
  solve_rows<<<kRedBlocks, kRedThreads, 0, s>>>(lmat, mttkrp, rows, rank, x64, d_status, part);
  ALTO_LAUNCH_CHECK("alto_solve_rows");
  return ALTO_OK;
}

int alto_colsumsq(const double* x, int64_t rows, int32_t rank, const uint8_t* row_mask, double* out,
                  void* ws, size_t ws_bytes, void* stream) {
  ALTO_REQUIRE(rank >= 1 && rank <= kMaxRank, "rank must be in [1, 64]");
  ALTO_REQUIRE(ws && ws_bytes >= alto_cpd_workspace_bytes(rank), "cpd workspace too small");
  cudaStream_t s = as_stream(stream);
  auto* part = static_cast<double*>(ws);
  colsumsq_partial<<<kRedBlocks, kRedThreads, 0, s>>>(x, rows, rank, row_mask, part);
  sum_partials<<<1, 64, 0, s>>>(part, kRedBlocks, rank, out);
  ALTO_LAUNCH_CHECK("alto_colsumsq");
  return ALTO_OK;
}

int alto_normalize(double* x64, float* x32, int64_t rows, int32_t rank, const double* colsumsq, double* lambda,
                   const int32_t* d_status, void* stream) {
  ALTO_REQUIRE(rank >= 1 && rank <= kMaxRank, "rank must be in [1, 64]");
  cudaStream_t s = as_stream(stream);
  sqrt_kernel<<<1, 64, 0, s>>>(colsumsq, rank, lambda, d_status);
  normalize_kernel<<<grid_for(rows * rank, 256), 256, 0, s>>>(x64, x32, rows, rank, lambda, d_status);
  ALTO_LAUNCH_CHECK("alto_normalize");
  return ALTO_OK;
}

int alto_fit_inner_masked(const double* mttkrp, const double* f, const double* lambda, int64_t rows, int32_t rank,
                          const uint8_t* row_mask, double* out, void* ws, size_t ws_bytes, void* stream) {
  ALTO_REQUIRE(rank >= 1 && rank <= kMaxRank, "rank must be in [1, 64]");
  ALTO_REQUIRE(ws && ws_bytes >= alto_cpd_workspace_bytes(rank), "cpd workspace too small");
  cudaStream_t s = as_stream(stream);
  auto* part = static_cast<double*>(ws);
  inner_partial_masked<<<kRedBlocks, kRedThreads, 0, s>>>(mttkrp, f, lambda, rows, rank, row_mask, part);
  sum_scalar<<<1, 32, 0, s>>>(part, kRedBlocks, out);
  ALTO_LAUNCH_CHECK("alto_fit_inner_masked");
  return ALTO_OK;
}

}  // extern "C"

namespace alto {
__global__ void cast_f32_f64_kernel(const float* __restrict__ in, double* __restrict__ out, long long n) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n; i += stride)
    out[i] = static_cast<double>(in[i]);
}
}  // namespace alto

extern "C" int alto_cast_f32_f64(const float* in, double* out, int64_t n, void* stream) {
  if (n <= 0) return ALTO_OK;
  alto::cast_f32_f64_kernel<<<alto::grid_for(n, 256), 256, 0, alto::as_stream(stream)>>>(in, out, n);
  ALTO_LAUNCH_CHECK("alto_cast_f32_f64");
  return ALTO_OK;
}

// ---- deterministic fixed-point MTTKRP support ---------------------------------
namespace alto {
template <typename T, bool MAX>
__global__ void __launch_bounds__(kRedThreads) abs_partial(const T* __restrict__ v, long long n,
                                                           double* __restrict__ part) {
  __shared__ double s_tmp[32];
  const long long chunk = (n + gridDim.x - 1) / gridDim.x;
  const long long i0 = blockIdx.x * chunk, i1 = min(n, i0 + chunk);
  double s = 0.0;
  for (long long i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    const double x = fabs(static_cast<double>(v[i]));
    s = MAX ? fmax(s, x) : s + x;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double y = __shfl_down_sync(0xffffffffu, s, o);
    s = MAX ? fmax(s, y) : s + y;
  }
  if (lane == 0) s_tmp[warp] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = MAX ? fmax(t, s_tmp[w]) : t + s_tmp[w];
    part[blockIdx.x] = t;
  }
}
template <bool MAX>
__global__ void abs_final(const double* __restrict__ part, int nb, double* __restrict__ out) {
  if (threadIdx.x) return;
  double t = 0.0;
  for (int b = 0; b < nb; ++b) t = MAX ? fmax(t, part[b]) : t + part[b];
  *out = t;
}
__global__ void fixed_scale_kernel(const double* __restrict__ terms, int nt, double* __restrict__ scale) {
  if (threadIdx.x) return;
  double b = 1.0;
  for (int i = 0; i < nt; ++i) b *= terms[i];
  if (!(b > 0.0) || !isfinite(b)) b = 1.0;
  int e = 0;
  frexp(b, &e);                  // b < 2^e
  *scale = ldexp(1.0, 61 - e);   // every partial sum < 2^61 in fixed point
}
__global__ void fixed_to_float_kernel(const long long* __restrict__ in, const double* __restrict__ scale,
                                      void* __restrict__ out, int o32, long long n) {
  const double inv = 1.0 / *scale;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n; i += stride) {
    const double x = static_cast<double>(in[i]) * inv;
    if (o32) static_cast<float*>(out)[i] = static_cast<float>(x);
    else static_cast<double*>(out)[i] = x;
  }
}
}  // namespace alto

extern "C" {
int alto_sumabs(const void* x, int32_t dtype, int64_t n, double* out, void* ws, size_t ws_bytes, void* stream) {
  ALTO_REQUIRE(ws && ws_bytes >= kRedBlocks * sizeof(double), "workspace too small");
  cudaStream_t s = as_stream(stream);
  auto* part = static_cast<double*>(ws);
  if (dtype == ALTO_F32)
    abs_partial<float, false><<<kRedBlocks, kRedThreads, 0, s>>>(static_cast<const float*>(x), n, part);
  else
    abs_partial<double, false><<<kRedBlocks, kRedThreads, 0, s>>>(static_cast<const double*>(x), n, part);
  abs_final<false><<<1, 32, 0, s>>>(part, kRedBlocks, out);
  ALTO_LAUNCH_CHECK("alto_sumabs");
  return ALTO_OK;
}
int alto_absmax(const void* x, int32_t dtype, int64_t n, double* out, void* ws, size_t ws_bytes, void* stream) {
  ALTO_REQUIRE(ws && ws_bytes >= kRedBlocks * sizeof(double), "workspace too small");
  cudaStream_t s = as_stream(stream);
  auto* part = static_cast<double*>(ws);
  if (dtype == ALTO_F32)
    abs_partial<float, true><<<kRedBlocks, kRedThreads, 0, s>>>(static_cast<const float*>(x), n, part);
  else
    abs_partial<double, true><<<kRedBlocks, kRedThreads, 0, s>>>(static_cast<const double*>(x), n, part);
  abs_final<true><<<1, 32, 0, s>>>(part, kRedBlocks, out);
  ALTO_LAUNCH_CHECK("alto_absmax");
  return ALTO_OK;
}
int alto_fixed_scale(const double* terms, int32_t nterms, double* scale, void* stream) {
  fixed_scale_kernel<<<1, 32, 0, as_stream(stream)>>>(terms, nterms, scale);
  ALTO_LAUNCH_CHECK("alto_fixed_scale");
  return ALTO_OK;
}
int alto_fixed_to_float(const int64_t* in, const double* scale, void* out, int32_t out_dtype, int64_t n,
                        void* stream) {
  if (n <= 0) return ALTO_OK;
  fixed_to_float_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const long long*>(in), scale, out, out_dtype == ALTO_F32, n);
  ALTO_LAUNCH_CHECK("alto_fixed_to_float");
  return ALTO_OK;
}
}  // extern "C"
