// alto_stream.cu — streaming ALTO MTTKRP (K7/K8), the fast path.
//
//   out[i_n, r] = sum over elements x: x.value * prod_{m != n} F_m[x.coord_m, r]
//   (pkg/src/altotensor/mttkrp.py:1-14; contributions :80-105)
//
// Generic fallback (runtime order and rank; the specialised order-3/4/5,
// rank-16/32 kernels live in alto_fast.cuh / alto_mstream.cuh / alto_pull.cuh).
// Each warp streams its own sub-tiles of kWarpTile consecutive elements of the
// sorted ALTO stream:
//  decode   coalesced key/value loads into registers, byte-table decode
//           (alto_common.cuh), and a mode-specific record {coords of the N-1
//           input modes, output target, value}.  The target is the output
//           row, or -(slot+1) for a row of the mode's hot plan.
//  sort     if the sub-tile's output interval spans <= kWarpBins rows it is
//           counting-sorted by output row in the warp's shared-memory slice
//           (the paper's per-partition Buffered scheme, Alg. 2 /
//           mttkrp.py:148-156, at warp granularity); wider sub-tiles keep
//           stream order (the Atomic scheme, mttkrp.py:178-224).
//  consume  G lanes per element, each lane owning 4 consecutive ranks; each
//           group walks a contiguous run of records with U elements' gathers
//           in flight, multiplies, and accumulates in registers while the
//           target row repeats; on a row change the partial is merged with
//           atomics (RED.F32x4, or float64 REDs after a 4x4 in-quad shuffle
//           transpose).  Hot rows go to one of hot_copies replicated buffers,
//           summed afterwards in a fixed order.
#include <algorithm>
#include <climits>
#include <type_traits>

#pragma once
#include "alto_common.cuh"

namespace alto {

constexpr int kTileThreads = 256;
constexpr int kTileWarps = kTileThreads / 32;
constexpr int kEPT = 4;  // tile argument: at most kEPT * kTileThreads elements (ABI check)

struct StreamParams {
  const uint64_t* keys;
  const void* values;
  long long m;
  int mode;
  int rank;
  const void* factors[ALTO_MAX_ORDER];
  void* out;
  int tile;
  int n_hot;
  long long ntiles;
  const int* hot_slot;
  int hot_copies;
  int hot_adaptive;  // hot_slot holds alto_hot_copies codes ((first copy << 5) | log2 copies), hot_buf the copies
  void* hot_buf;  // hot_copies x n_hot x R (adaptive: all rows' copies), element type = output type O
  int flags;
  const uint64_t* packed;     // mode-contiguous keys (optional, alto_pack_keys)
  const unsigned char* pos;   // per-mode sub-tile slots (optional, alto_subtile_order)
  const uint64_t* mkeys;      // per-mode stream (optional, alto_mode_stream): keys
  const void* mvals;          //   values
  int mtile;                  //   tile length T
  int mrr;                    //   round-robin slices (ALTO_MS_ROUND_ROBIN)
  const int* mbase;           //   delta stream (ALTO_MS_DELTA): base row per lane group, else null
  int n_pairs;                // paired input modes (mode stream): count,
  int pair_a[2], pair_b[2];   //   modes,
  const void* pair_tab[2];    //   row-wise product tables (alto_krp_pair)
  const double* fixed_scale;  // deterministic mode: device scalar, int64 output = round(x * scale)
  unsigned l2_hot[ALTO_MAX_ORDER];  // per mode: leading bytes of its factor gathered with L2 evict_last (0 = no policy)
  unsigned l2_tab[ALTO_MAX_ORDER];  //   and the factor's size in bytes
};

template <typename V, typename F>
struct AccOf { using type = double; };
template <>
struct AccOf<float, float> { using type = float; };

// Record: N-1 input-mode coordinates, target, value bits; padded to 16 B.
template <int N, typename V>
struct RecLayout {
  static constexpr int raw = (N - 1) + 1 + static_cast<int>(sizeof(V) / 4);
  static constexpr int NW = (raw + 3) & ~3;
  static constexpr int TGT = N - 1;
  static constexpr int VAL = N;
};

template <typename F>
struct V4 {
  F v[4];
};

template <typename F, bool VEC>
__device__ __forceinline__ V4<F> gather4(const F* __restrict__ row, int r, int R) {
  V4<F> o;
  if constexpr (VEC) {
    if constexpr (sizeof(F) == 4) {
      const float4 t = __ldg(reinterpret_cast<const float4*>(row + r));
      o.v[0] = t.x; o.v[1] = t.y; o.v[2] = t.z; o.v[3] = t.w;
    } else {
      const double2 a = __ldg(reinterpret_cast<const double2*>(row + r));
      const double2 b = __ldg(reinterpret_cast<const double2*>(row + r + 2));
      o.v[0] = a.x; o.v[1] = a.y; o.v[2] = b.x; o.v[3] = b.y;
    }
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q) o.v[q] = (r + q < R) ? __ldg(row + r + q) : F(0);
  }
  return o;
}

// FULLR gather: the record holds the row's byte offset, so the address is one add.
template <typename F>
__device__ __forceinline__ V4<F> gather_off(const char* base, unsigned off) {
  V4<F> o;
  if constexpr (sizeof(F) == 4) {
    const float4 t = __ldg(reinterpret_cast<const float4*>(base + off));
    o.v[0] = t.x; o.v[1] = t.y; o.v[2] = t.z; o.v[3] = t.w;
  } else {
    const double2 a = __ldg(reinterpret_cast<const double2*>(base + off));
    const double2 b = __ldg(reinterpret_cast<const double2*>(base + off) + 1);
    o.v[0] = a.x; o.v[1] = a.y; o.v[2] = b.x; o.v[3] = b.y;
  }
  return o;
}

// L2 policy per gathered table: the first `hot` bytes evict_last (the most
// referenced rows when rows are numbered by popularity), the rest evict_first.
__device__ __forceinline__ unsigned long long range_policy(const void* tab, unsigned hot, unsigned total) {
  unsigned long long p;
  asm volatile("createpolicy.range.global.L2::evict_last.L2::evict_first.b64 %0, [%1], %2, %3;"
               : "=l"(p)
               : "l"(tab), "r"(hot), "r"(total));
  return p;
}

__device__ __forceinline__ V4<float> gather_off_pol(const char* base, unsigned off, unsigned long long pol) {
  V4<float> o;
  asm("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
      : "=f"(o.v[0]), "=f"(o.v[1]), "=f"(o.v[2]), "=f"(o.v[3])
      : "l"(base + off), "l"(pol));
  return o;
}

__device__ __forceinline__ void red_f32x4_pol(float* p, const float (&acc)[4], unsigned long long pol) {
  asm volatile("red.global.add.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(acc[0]), "f"(acc[1]),
               "f"(acc[2]), "f"(acc[3]), "l"(pol)
               : "memory");
}

template <int NMAX>
__device__ __forceinline__ unsigned pick(const unsigned* w, int mode) {
  unsigned r = w[0];
#pragma unroll
  for (int n = 1; n < NMAX; ++n)
    if (n == mode) r = w[n];
  return r;
}

// 4x4 transpose across the aligned lane quad: on exit lane l (l = lane&3)
// holds, at index q, the value lane q held at index l.
template <typename A>
__device__ __forceinline__ void quad_transpose(A (&v)[4], unsigned qmask, int l) {
#pragma unroll
  for (int step = 1; step <= 2; step <<= 1) {
    A t[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) t[q] = __shfl_xor_sync(qmask, v[q ^ step], step);
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (((q & step) != 0) != ((l & step) != 0)) v[q] = t[q];
  }
}

template <typename A>
__device__ __forceinline__ void red_f64_sectors(double* __restrict__ rowbase, const A (&acc)[4], int r, int R,
                                                int G, unsigned qmask, int lane) {
  // rowbase points at rank 0 of the target row; this lane owns ranks r..r+3.
  if (G >= 4 && (R & 15) == 0) {
    A v[4] = {acc[0], acc[1], acc[2], acc[3]};
    const int l = lane & 3;
    quad_transpose(v, qmask, l);
    const int base = r - 4 * l;  // first rank of the quad's 16-rank block
#pragma unroll
    for (int q = 0; q < 4; ++q) atomicAdd(rowbase + base + 4 * q + l, static_cast<double>(v[q]));
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (r + q < R) atomicAdd(rowbase + r + q, static_cast<double>(acc[q]));
  }
}

template <typename A>
__device__ __forceinline__ void red_f32x4(float* __restrict__ p, const A (&acc)[4], int r, int R, bool vec) {
  if (vec) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p + r), "f"(static_cast<float>(acc[0])),
                 "f"(static_cast<float>(acc[1])), "f"(static_cast<float>(acc[2])), "f"(static_cast<float>(acc[3]))
                 : "memory");
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (r + q < R) atomicAdd(p + r + q, static_cast<float>(acc[q]));
  }
}

// ---- warp-autonomous kernel ---------------------------------------------------
// Only __syncwarp inside: a warp's decode/sort latency is hidden by the other
// warps instead of being serialised behind CTA barriers.
constexpr int kWarpTile = 128;   // elements per warp sub-tile (4 per lane)
constexpr int kWarpBins = 512;   // warp-private sort bins

template <int W, typename V, typename F, typename O, int NT, int G, bool VEC, bool FULLR>
__global__ void __launch_bounds__(kTileThreads, 2)
stream_warp_kernel(const __grid_constant__ DevLayout L, const uint64_t* __restrict__ tab,
                   const __grid_constant__ StreamParams P) {
  using A = typename AccOf<V, F>::type;
  constexpr int NMAX = NT > 0 ? NT : ALTO_MAX_ORDER;
  using RL = RecLayout<NMAX, V>;
  constexpr int NW = RL::NW;
  constexpr int NIN = NMAX - 1;
  constexpr int GPW = 32 / G;                    // element groups per warp
  constexpr int CH = kWarpTile / GPW;            // records per group chunk
  constexpr int U = 4;
  constexpr int EPL = kWarpTile / 32;            // elements per lane in the load/decode pass
  constexpr int REC_WORDS = kWarpTile * NW + GPW * 4;  // + swizzle headroom
  extern __shared__ __align__(16) unsigned char smem[];
  const int N = NT > 0 ? NT : L.order;
  const int R = P.rank;
  const int mode = P.mode;
  uint64_t* s_dec = reinterpret_cast<uint64_t*>(smem);
  size_t off = (static_cast<size_t>(L.dec_bytes) * 256 * W * 8 + 15) & ~size_t(15);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned* s_rec = reinterpret_cast<unsigned*>(smem + off) + warp * (REC_WORDS + kWarpBins);
  int* s_bin = reinterpret_cast<int*>(s_rec + REC_WORDS);

  copy_to_smem(s_dec, tab + static_cast<long long>(L.dec_off) * W, L.dec_bytes * 256 * W);
  __syncthreads();

  const int grp = lane / G;
  const int gl = lane % G;
  const int r_lane = 4 * gl;
  const unsigned qmask = (G >= 4) ? (0xFu << (lane & ~3)) : 0xffffffffu;
  const F* __restrict__ fin[NIN > 0 ? NIN : 1];
  const char* fin_lane[NIN > 0 ? NIN : 1];
#pragma unroll
  for (int k = 0; k < NIN; ++k) {
    const int n = k < mode ? k : k + 1;
    fin[k] = static_cast<const F*>(P.factors[n < ALTO_MAX_ORDER ? n : 0]);
    fin_lane[k] = reinterpret_cast<const char*>(fin[k] + r_lane);
  }
  const V* __restrict__ vals = static_cast<const V*>(P.values);
  O* __restrict__ out = static_cast<O*>(P.out);
  const int* __restrict__ hot_slot = P.n_hot > 0 ? P.hot_slot : nullptr;
  const int n_in = N - 1;
  auto rec_addr = [&](int j) { return j * NW + (j / CH) * 4; };
  const unsigned lt = (1u << lane) - 1u;
  (void)lt;

  const long long nsub = (P.m + kWarpTile - 1) / kWarpTile;
  const long long gwarp = static_cast<long long>(blockIdx.x) * (kTileThreads / 32) + warp;
  const long long nwarps = static_cast<long long>(gridDim.x) * (kTileThreads / 32);
  for (long long sub = gwarp; sub < nsub; sub += nwarps) {
    const long long e0 = sub * kWarpTile;
    const int cnt = static_cast<int>(min(static_cast<long long>(kWarpTile), P.m - e0));
    // ---- load + decode (lane per element) --------------------------------
    unsigned rec[EPL][NW];
    int myrow[EPL];
    Key<W> kk[EPL];
    V vv0[EPL];
#pragma unroll
    for (int k = 0; k < EPL; ++k) {
      const int e = lane + 32 * k;
      if (e < cnt) {
        kk[k] = load_key<W>(P.keys, e0 + e);
        vv0[k] = __ldg(vals + e0 + e);
      }
    }
    int lo = INT_MAX, hi = INT_MIN;
#pragma unroll
    for (int k = 0; k < EPL; ++k) {
      const int e = lane + 32 * k;
      myrow[k] = -1;
      if (e < cnt) {
        const Key<W> p = decode_packed<W>(s_dec, L.dec_bytes, kk[k]);
        unsigned c[NMAX];
#pragma unroll
        for (int n = 0; n < NMAX; ++n)
          c[n] = n < N ? static_cast<unsigned>(packed_field<W>(p, L.pack_off[n], L.bits[n])) : 0u;
        const int row = static_cast<int>(pick<NMAX>(c, mode));
#pragma unroll
        for (int q = 0; q < NIN; ++q) {
          const unsigned cq = (q < mode) ? c[q] : c[q + 1 < NMAX ? q + 1 : q];
          rec[k][q] = FULLR ? cq * static_cast<unsigned>(4 * G * sizeof(F)) : cq;
        }
        int tgt = row;
        if (hot_slot) {
          const int hs = __ldg(hot_slot + row);
          if (hs >= 0)  // adaptive plan: copy (sub-tile mod copies) of the row's own copies
            tgt = P.hot_adaptive ? -((hs >> 5) + static_cast<int>(static_cast<unsigned>(sub) & ((1u << (hs & 31)) - 1u)) + 1)
                                 : -(hs + 1);
        }
        rec[k][RL::TGT] = static_cast<unsigned>(tgt);
        if constexpr (sizeof(V) == 4) {
          rec[k][RL::VAL] = __float_as_uint(static_cast<float>(vv0[k]));
        } else {
          const unsigned long long u = __double_as_longlong(static_cast<double>(vv0[k]));
          rec[k][RL::VAL] = static_cast<unsigned>(u);
          rec[k][RL::VAL + 1] = static_cast<unsigned>(u >> 32);
        }
#pragma unroll
        for (int q = RL::raw; q < NW; ++q) rec[k][q] = 0u;
        myrow[k] = row;
        lo = min(lo, row);
        hi = max(hi, row);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    const int span = hi - lo + 1;
    // ---- warp-private counting sort by output row ------------------------
    if (span <= kWarpBins) {
      for (int i = lane; i < span; i += 32) s_bin[i] = 0;
      __syncwarp();
#pragma unroll
      for (int k = 0; k < EPL; ++k)
        if (myrow[k] >= 0) atomicAdd(&s_bin[myrow[k] - lo], 1);
      __syncwarp();
      const int per = (span + 31) / 32;
      const int b0 = min(span, lane * per), b1 = min(span, b0 + per);
      int sum = 0;
      for (int i = b0; i < b1; ++i) sum += s_bin[i];
      int x = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      int run = x - sum;
      for (int i = b0; i < b1; ++i) {
        const int c = s_bin[i];
        s_bin[i] = run;
        run += c;
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < EPL; ++k)
        if (myrow[k] >= 0) {
          const int slot = atomicAdd(&s_bin[myrow[k] - lo], 1);
#pragma unroll
          for (int q = 0; q < NW; q += 4)
            *reinterpret_cast<uint4*>(s_rec + rec_addr(slot) + q) =
                make_uint4(rec[k][q], rec[k][q + 1], rec[k][q + 2], rec[k][q + 3]);
        }
    } else {
#pragma unroll
      for (int k = 0; k < EPL; ++k)
        if (myrow[k] >= 0) {
          const int e = lane + 32 * k;
#pragma unroll
          for (int q = 0; q < NW; q += 4)
            *reinterpret_cast<uint4*>(s_rec + rec_addr(e) + q) =
                make_uint4(rec[k][q], rec[k][q + 1], rec[k][q + 2], rec[k][q + 3]);
        }
    }
    __syncwarp();
    // ---- consume: G lanes per element ------------------------------------
    O* hot_base = P.n_hot > 0
                      ? static_cast<O*>(P.hot_buf) +
                            (P.hot_adaptive
                                 ? 0ll
                                 : static_cast<long long>(static_cast<unsigned>(sub) & (P.hot_copies - 1)) * P.n_hot * R)
                      : nullptr;
    const int j0 = grp * CH;
    const int j1 = min(cnt, j0 + CH);
    for (int r0 = 0; r0 < (FULLR ? 4 * G : R); r0 += 4 * G) {
      const int r = r0 + r_lane;
      const bool rank_ok = FULLR || r < R;
      A acc[4] = {A(0), A(0), A(0), A(0)};
      int cur = INT_MIN;
      auto flush = [&](int target) {
        O* base = target >= 0 ? out + static_cast<long long>(target) * R
                              : hot_base + static_cast<long long>(-target - 1) * R;
        if constexpr (sizeof(O) == 4) {
          if (rank_ok) red_f32x4(reinterpret_cast<float*>(base), acc, r, R, VEC);
        } else {
          red_f64_sectors(reinterpret_cast<double*>(base), acc, r, R, G, qmask, lane);
        }
      };
      for (int jb = j0; jb < j1; jb += U) {
        int tg[U];
        A vv[U];
        V4<F> g[U][NIN > 0 ? NIN : 1];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int j = jb + u;
          tg[u] = INT_MIN;
          if (j < j1) {
            unsigned cw[NW];
#pragma unroll
            for (int q = 0; q < NW; q += 4) {
              const uint4 t = *reinterpret_cast<const uint4*>(s_rec + rec_addr(j) + q);
              cw[q] = t.x; cw[q + 1] = t.y; cw[q + 2] = t.z; cw[q + 3] = t.w;
            }
            tg[u] = static_cast<int>(cw[RL::TGT]);
            if constexpr (sizeof(V) == 4) {
              vv[u] = static_cast<A>(__uint_as_float(cw[RL::VAL]));
            } else {
              vv[u] = static_cast<A>(__longlong_as_double(static_cast<long long>(
                  (static_cast<unsigned long long>(cw[RL::VAL + 1]) << 32) | cw[RL::VAL])));
            }
#pragma unroll
            for (int k = 0; k < NIN; ++k)
              if ((NT > 0 || k < n_in) && rank_ok) {
                g[u][k] = FULLR ? gather_off<F>(fin_lane[k], cw[k])
                                : gather4<F, VEC>(fin[k] + static_cast<unsigned long long>(cw[k]) * R, r, R);
              }
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (tg[u] == INT_MIN) continue;
          A t[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) t[q] = vv[u];
          int last = -1;
          if (rank_ok) {
#pragma unroll
            for (int k = 0; k < NIN; ++k)
              if (NT > 0 || k < n_in) last = k;
#pragma unroll
            for (int k = 0; k < NIN; ++k)
              if ((NT > 0 || k < n_in) && k != last) {
#pragma unroll
                for (int q = 0; q < 4; ++q) t[q] *= static_cast<A>(g[u][k].v[q]);
              }
          }
          if (tg[u] == cur) {
            if (last >= 0) {
#pragma unroll
              for (int q = 0; q < 4; ++q) acc[q] = fma(t[q], static_cast<A>(g[u][last].v[q]), acc[q]);
            } else {
#pragma unroll
              for (int q = 0; q < 4; ++q) acc[q] += t[q];
            }
          } else {
            if (cur != INT_MIN) flush(cur);
            if (last >= 0) {
#pragma unroll
              for (int q = 0; q < 4; ++q) acc[q] = t[q] * static_cast<A>(g[u][last].v[q]);
            } else {
#pragma unroll
              for (int q = 0; q < 4; ++q) acc[q] = t[q];
            }
            cur = tg[u];
          }
        }
      }
      if (cur != INT_MIN) flush(cur);
    }
    __syncwarp();
  }
}

// ---- launch ---------------------------------------------------------------------

template <typename K>
inline int prep(K kernel, size_t smem) {
  ALTO_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  return ALTO_OK;
}

inline int device_sms() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) !=
                                                  cudaSuccess)
      sms = kSMs;
  }
  return sms;
}

template <int W, typename V, typename F, typename O, int NT, int G, bool VEC, bool FULLR>
int launch(const DevLayout& d, const uint64_t* tab, const StreamParams& P, cudaStream_t s) {
  constexpr int NMAX = NT > 0 ? NT : ALTO_MAX_ORDER;
  constexpr int NW = RecLayout<NMAX, V>::NW;
  const size_t dec = (static_cast<size_t>(d.dec_bytes) * 256 * W * 8 + 15) & ~size_t(15);
  constexpr int GPW = 32 / G;
  const size_t per_warp = (static_cast<size_t>(kWarpTile) * NW + GPW * 4 + kWarpBins) * 4;
  const size_t smem = dec + (kTileThreads / 32) * per_warp;
  auto kern = stream_warp_kernel<W, V, F, O, NT, G, VEC, FULLR>;
  if (prep(kern, smem)) return ALTO_ECUDA;
  int bps = 1;
  ALTO_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, kTileThreads, smem));
  const long long nsub = (P.m + kWarpTile - 1) / kWarpTile;
  const long long need = (nsub + kTileThreads / 32 - 1) / (kTileThreads / 32);
  const long long grid = std::min<long long>(need, static_cast<long long>(device_sms()) * std::max(bps, 1));
  kern<<<static_cast<unsigned>(grid), kTileThreads, smem, s>>>(d, tab, P);
  ALTO_LAUNCH_CHECK("alto_mttkrp");
  return ALTO_OK;
}

template <int W, typename V, typename F, typename O, int NT>
int by_rank(const DevLayout& d, const uint64_t* tab, const StreamParams& P, cudaStream_t s) {
  const int groups = (P.rank + 3) / 4;
  // FULLR kernels keep 32-bit row byte offsets in the records
  long long maxdim = 0;
  for (int n = 0; n < d.order; ++n) maxdim = std::max(maxdim, d.dims[n]);
  const bool off32 = maxdim * P.rank * static_cast<long long>(sizeof(F)) <= 0xFFFFFFFFll;
  (void)off32;
  if (P.rank % 4 == 0) {
    if (groups <= 1) return launch<W, V, F, O, NT, 1, true, false>(d, tab, P, s);
    if (groups <= 2) return launch<W, V, F, O, NT, 2, true, false>(d, tab, P, s);
    if (groups <= 4) return launch<W, V, F, O, NT, 4, true, false>(d, tab, P, s);
    return launch<W, V, F, O, NT, 8, true, false>(d, tab, P, s);
  }
  if (groups <= 1) return launch<W, V, F, O, NT, 1, false, false>(d, tab, P, s);
  if (groups <= 4) return launch<W, V, F, O, NT, 4, false, false>(d, tab, P, s);
  return launch<W, V, F, O, NT, 8, false, false>(d, tab, P, s);
}

template <int W, typename V, typename F, typename O>
int by_order(const DevLayout& d, const uint64_t* tab, const StreamParams& P, cudaStream_t s) {
  // Generic fallback: runtime order (the specialised order-3/4/5, rank-16/32
  // kernels live in alto_fast.cuh).
  return by_rank<W, V, F, O, 0>(d, tab, P, s);
}

// per-translation-unit entry points (alto_stream_w{1,2}_{f32,f64}.cu, and the
// specialised kernels of alto_fast_w{1,2}_{f32,f64}.cu, which return
// ALTO_EUNSUPPORTED without launching when the shape is not covered)
int fast_w1_f32(const DevLayout&, const uint64_t*, const StreamParams&, int vd, int fd, cudaStream_t);
int fast_w1_f64(const DevLayout&, const uint64_t*, const StreamParams&, int vd, int fd, cudaStream_t);
int fast_w2_f32(const DevLayout&, const uint64_t*, const StreamParams&, int vd, int fd, cudaStream_t);
int fast_w2_f64(const DevLayout&, const uint64_t*, const StreamParams&, int vd, int fd, cudaStream_t);
int fast_w1_i64(const DevLayout&, const uint64_t*, const StreamParams&, int vd, int fd, cudaStream_t);
int fast_w2_i64(const DevLayout&, const uint64_t*, const StreamParams&, int vd, int fd, cudaStream_t);
int stream_w1_f32(const DevLayout&, const uint64_t*, const StreamParams&, int vd, int fd, cudaStream_t);
int stream_w1_f64(const DevLayout&, const uint64_t*, const StreamParams&, int vd, int fd, cudaStream_t);
int stream_w2_f32(const DevLayout&, const uint64_t*, const StreamParams&, int vd, int fd, cudaStream_t);
int stream_w2_f64(const DevLayout&, const uint64_t*, const StreamParams&, int vd, int fd, cudaStream_t);

}  // namespace alto
