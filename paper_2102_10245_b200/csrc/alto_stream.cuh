// alto_stream.cu — streaming ALTO MTTKRP (K7/K8), the fast path.
//
//   out[i_n, r] = sum over elements x: x.value * prod_{m != n} F_m[x.coord_m, r]
//   (pkg/src/altotensor/mttkrp.py:1-14; contributions :80-105)
//
// A persistent CTA streams tiles of T (<= 1024) consecutive elements of the
// sorted ALTO stream:
//  Phase A  one thread per element: coalesced key/value loads, byte-table
//           decode in registers (alto_common.cuh), and a mode-specific
//           record {coords of the N-1 input modes, output target, value}.
//           The target is the output row, or -(slot+1) for a row of the
//           mode's hot plan.  The tile's output interval [lo, hi] is reduced.
//  Sort     if hi-lo+1 <= kSortBins the tile is counting-sorted by output row
//           in shared memory (the tile's interval buffer: the paper's
//           per-partition Buffered scheme, Alg. 2 / mttkrp.py:148-156, at CTA
//           granularity).  Wider tiles keep stream order (they are the
//           hypersparse tail where rows rarely repeat: the Atomic scheme,
//           mttkrp.py:178-224).
//  Phase B  G lanes per element, each lane owning 4 consecutive ranks, so a
//           factor row is gathered as one contiguous 16*G-byte request.
//           Each G-lane group walks a contiguous run of records with U
//           elements' gathers in flight, multiplies, and accumulates in
//           registers while the target row repeats; on a row change the
//           partial is merged with atomics: RED.F32x4 (float32 output, one
//           16-byte RED per lane) or float64 REDs after a 4x4 in-quad shuffle
//           transpose (each RED instruction then covers one 32-byte sector).
//           Hot rows — touched by nearly every tile — go to one of
//           hot_copies replicated float64 buffers instead, and a second
//           kernel sums the copies in a fixed order (same-address REDs from
//           every tile would otherwise serialise in one L2 slice).
#include <algorithm>
#include <climits>
#include <type_traits>

#pragma once
#include "alto_common.cuh"

namespace alto {

constexpr int kTileThreads = 256;
constexpr int kTileWarps = kTileThreads / 32;
constexpr int kSortBins = 2048;
constexpr int kEPT = 4;  // elements per thread in phase A -> tile <= 1024
constexpr int kRecPad = 4 * kTileThreads;  // words of swizzle headroom (4 per phase-B chunk)

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
  void* hot_buf;  // hot_copies x n_hot x R, element type = output type O
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
  const double* fixed_scale;  // deterministic mode: device scalar, int64 output = round(x * scale)  // tuning switches (ALTO_STREAM_* bits in alto_b200.h)
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

template <int W, typename V, typename F, typename O, int NT, int G, bool VEC, bool FULLR>
__global__ void __launch_bounds__(kTileThreads, 2)
stream_kernel(const __grid_constant__ DevLayout L, const uint64_t* __restrict__ tab,
              const __grid_constant__ StreamParams P) {
  using A = typename AccOf<V, F>::type;
  constexpr int NMAX = NT > 0 ? NT : ALTO_MAX_ORDER;
  using RL = RecLayout<NMAX, V>;
  constexpr int NW = RL::NW;
  constexpr int NIN = NMAX - 1;              // input modes per record
  constexpr int NGROUPS = kTileThreads / G;
  constexpr int U = 4;                       // elements in flight per group
  extern __shared__ __align__(16) unsigned char smem[];
  const int N = NT > 0 ? NT : L.order;
  const int T = P.tile;
  const int R = P.rank;
  const int mode = P.mode;
  uint64_t* s_dec = reinterpret_cast<uint64_t*>(smem);
  size_t off = (static_cast<size_t>(L.dec_bytes) * 256 * W * 8 + 15) & ~size_t(15);
  unsigned* s_rec = reinterpret_cast<unsigned*>(smem + off);  // [T][NW]
  off += static_cast<size_t>(T) * NW * 4 + kRecPad * 4;
  int* s_bin = reinterpret_cast<int*>(smem + off);            // [kSortBins + kTileWarps]
  off += (kSortBins + kTileWarps) * sizeof(int);
  off = (off + 15) & ~size_t(15);
  unsigned char* s_stage = smem + off;                        // 2 x (T keys + T values)
  const size_t stage_bytes = (static_cast<size_t>(T) * (W * 8 + sizeof(V)) + 15) & ~size_t(15);
  __shared__ int s_lo[kTileWarps], s_hi[kTileWarps];

  copy_to_smem(s_dec, tab + static_cast<long long>(L.dec_off) * W, L.dec_bytes * 256 * W);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int grp = tid / G;
  const int gl = tid % G;
  const int r_lane = 4 * gl;
  // Record swizzle: phase-B groups read chunks of T/NGROUPS consecutive
  // records; shifting chunk c by 16*c bytes puts the 8 groups of a warp on
  // distinct banks (unswizzled, equal strides make it an 8-way conflict).
  const int chunk_shift = 31 - __clz(max(T / NGROUPS, 1));
  auto rec_addr = [&](int j) { return j * NW + (j >> chunk_shift) * 4; };
  const unsigned qmask = (G >= 4) ? (0xFu << (lane & ~3)) : 0xffffffffu;
  // input-mode factor bases in record order (mode skipped)
  const F* __restrict__ fin[NIN > 0 ? NIN : 1];
  const char* fin_lane[NIN > 0 ? NIN : 1];  // fin[k] + this lane's first rank, as bytes
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

  // keys/values of the CTA's next tile are copied global->shared with
  // cp.async (double-buffered staging) while the current tile is consumed
  auto stage_keys = [&](int b) { return reinterpret_cast<uint64_t*>(s_stage + b * stage_bytes); };
  auto stage_vals = [&](int b) {
    return reinterpret_cast<V*>(s_stage + b * stage_bytes + static_cast<size_t>(T) * W * 8);
  };
  auto prefetch = [&](long long tl, int b) {
    if (tl >= P.ntiles) return;
    const long long b0 = tl * T;
    const int c = static_cast<int>(min(static_cast<long long>(T), P.m - b0));
    if (c == T) {
      const char* gk = reinterpret_cast<const char*>(P.keys + b0 * W);
      const char* gv = reinterpret_cast<const char*>(vals + b0);
      char* sk = reinterpret_cast<char*>(stage_keys(b));
      char* sv = reinterpret_cast<char*>(stage_vals(b));
      const int nk = T * W * 8 / 16, nv = T * static_cast<int>(sizeof(V)) / 16;
      for (int i = tid; i < nk + nv; i += kTileThreads) {
        const char* g = i < nk ? gk + 16 * i : gv + 16 * (i - nk);
        char* d = i < nk ? sk + 16 * i : sv + 16 * (i - nk);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(d))),
                     "l"(g)
                     : "memory");
      }
    } else {
      for (int e = tid; e < c; e += kTileThreads) {
        store_key<W>(stage_keys(b), e, load_key<W>(P.keys, b0 + e));
        stage_vals(b)[e] = __ldg(vals + b0 + e);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  int buf = 0;
  prefetch(blockIdx.x, 0);
  for (long long tile = blockIdx.x; tile < P.ntiles; tile += gridDim.x) {
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    const long long t0 = tile * T;
    const int cnt = static_cast<int>(min(static_cast<long long>(T), P.m - t0));
    const uint64_t* sk = stage_keys(buf);
    const V* sv = stage_vals(buf);
    // ---- phase A -----------------------------------------------------------
    unsigned rec[kEPT][NW];
    int myrow[kEPT];
    int lo = INT_MAX, hi = INT_MIN;
#pragma unroll
    for (int k = 0; k < kEPT; ++k) {
      const int e = tid + k * kTileThreads;
      myrow[k] = -1;
      if (e < cnt) {
        const Key<W> p = decode_packed<W>(s_dec, L.dec_bytes, load_key_smem<W>(sk, e));
        unsigned c[NMAX];
#pragma unroll
        for (int n = 0; n < NMAX; ++n)
          c[n] = n < N ? static_cast<unsigned>(packed_field<W>(p, L.pack_off[n], L.bits[n])) : 0u;
        const int row = static_cast<int>(pick<NMAX>(c, mode));
#pragma unroll
        for (int q = 0; q < NIN; ++q) {
          const unsigned cq = (q < mode) ? c[q] : c[q + 1 < NMAX ? q + 1 : q];
          // FULLR: byte offset of the factor row (fits in 32 bits, checked at launch)
          rec[k][q] = FULLR ? cq * static_cast<unsigned>(4 * G * sizeof(F)) : cq;
        }
        int tgt = row;
        if (hot_slot) {
          const int hs = __ldg(hot_slot + row);
          if (hs >= 0) tgt = -(hs + 1);
        }
        rec[k][RL::TGT] = static_cast<unsigned>(tgt);
        const V v = sv[e];
        if constexpr (sizeof(V) == 4) {
          rec[k][RL::VAL] = __float_as_uint(static_cast<float>(v));
        } else {
          const unsigned long long u = __double_as_longlong(static_cast<double>(v));
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
    buf ^= 1;
    prefetch(tile + gridDim.x, buf);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (lane == 0) { s_lo[warp] = lo; s_hi[warp] = hi; }
    __syncthreads();
    lo = s_lo[0]; hi = s_hi[0];
#pragma unroll
    for (int w = 1; w < kTileWarps; ++w) { lo = min(lo, s_lo[w]); hi = max(hi, s_hi[w]); }
    const int span = hi - lo + 1;
    // ---- in-tile counting sort by output row ----------------------------
    // Only the tile's span of bins is touched; equal bins inside a warp are
    // aggregated with __match_any_sync so hot rows cost one atomic per warp.
    if (span <= kSortBins) {
      const bool aggregate = (P.flags & ALTO_STREAM_WARP_AGG) != 0;
      const int nbins = (P.flags & ALTO_STREAM_FULL_BINS) ? kSortBins : span;
      for (int i = tid; i < nbins; i += kTileThreads) s_bin[i] = 0;
      __syncthreads();
      unsigned peers[kEPT];
      const unsigned lt = (1u << lane) - 1u;
      if (aggregate) {
#pragma unroll
        for (int k = 0; k < kEPT; ++k) {
          const bool ok = myrow[k] >= 0;
          const int bin = ok ? myrow[k] - lo : (1 << 30) + lane;
          peers[k] = __match_any_sync(0xffffffffu, bin);
          if (ok && (peers[k] & lt) == 0) atomicAdd(&s_bin[bin], __popc(peers[k]));
        }
      } else {
#pragma unroll
        for (int k = 0; k < kEPT; ++k)
          if (myrow[k] >= 0) atomicAdd(&s_bin[myrow[k] - lo], 1);
      }
      __syncthreads();
      const int per = (nbins + kTileThreads - 1) / kTileThreads;
      const int b0 = min(nbins, tid * per), b1 = min(nbins, b0 + per);
      int sum = 0;
      for (int i = b0; i < b1; ++i) sum += s_bin[i];
      int x = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) s_bin[kSortBins + warp] = x;
      __syncthreads();
      int run = x - sum;
#pragma unroll
      for (int w = 0; w < kTileWarps; ++w) run += (w < warp) ? s_bin[kSortBins + w] : 0;
      for (int i = b0; i < b1; ++i) {
        const int c = s_bin[i];
        s_bin[i] = run;
        run += c;
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < kEPT; ++k) {
        const bool ok = myrow[k] >= 0;
        int slot = 0;
        if (aggregate) {
          const int leader = __ffs(peers[k]) - 1;
          int base = 0;
          if (ok && leader == lane) base = atomicAdd(&s_bin[myrow[k] - lo], __popc(peers[k]));
          base = __shfl_sync(0xffffffffu, base, leader);
          slot = base + __popc(peers[k] & lt);
        } else if (ok) {
          slot = atomicAdd(&s_bin[myrow[k] - lo], 1);
        }
        if (ok) {
#pragma unroll
          for (int q = 0; q < NW; q += 4)
            *reinterpret_cast<uint4*>(s_rec + rec_addr(slot) + q) =
                make_uint4(rec[k][q], rec[k][q + 1], rec[k][q + 2], rec[k][q + 3]);
        }
      }
    } else {
#pragma unroll
      for (int k = 0; k < kEPT; ++k)
        if (myrow[k] >= 0) {
          const int e = tid + k * kTileThreads;
#pragma unroll
          for (int q = 0; q < NW; q += 4)
            *reinterpret_cast<uint4*>(s_rec + rec_addr(e) + q) =
                make_uint4(rec[k][q], rec[k][q + 1], rec[k][q + 2], rec[k][q + 3]);
        }
    }
    __syncthreads();
    // ---- phase B ------------------------------------------------------------
    O* hot_base = P.n_hot > 0
                      ? static_cast<O*>(P.hot_buf) +
                            static_cast<long long>(static_cast<unsigned>(tile) & (P.hot_copies - 1)) * P.n_hot * R
                      : nullptr;
    const int chunk = (cnt + NGROUPS - 1) / NGROUPS;
    const int j0 = grp * chunk;
    const int j1 = min(cnt, j0 + chunk);
    const bool full_chunk = (j1 - j0 == chunk) && (chunk % U == 0);
    for (int r0 = 0; r0 < (FULLR ? 4 * G : R); r0 += 4 * G) {
      const int r = r0 + r_lane;
      const bool rank_ok = FULLR || r < R;
      A acc[4] = {A(0), A(0), A(0), A(0)};
      int cur = INT_MIN;
      auto flush = [&](int target) {
        if (target >= 0) {
          if constexpr (sizeof(O) == 4) {
            if (rank_ok) red_f32x4(reinterpret_cast<float*>(out) + static_cast<long long>(target) * R, acc, r, R, VEC);
          } else {
            red_f64_sectors(reinterpret_cast<double*>(out) + static_cast<long long>(target) * R, acc, r, R, G,
                            qmask, lane);
          }
        } else {
          if constexpr (sizeof(O) == 4) {
            if (rank_ok) red_f32x4(reinterpret_cast<float*>(hot_base) + static_cast<long long>(-target - 1) * R, acc,
                                   r, R, VEC);
          } else {
            red_f64_sectors(reinterpret_cast<double*>(hot_base) + static_cast<long long>(-target - 1) * R, acc, r, R,
                            G, qmask, lane);
          }
        }
      };
      auto block = [&](auto check_tag, int jb) {
        constexpr bool CHECK = decltype(check_tag)::value;
        int tg[U];
        A vv[U];
        V4<F> g[U][NIN > 0 ? NIN : 1];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int j = jb + u;
          tg[u] = INT_MIN;
          if (!CHECK || j < j1) {
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
              if ((NT > 0 || k < n_in) && rank_ok)
                g[u][k] = FULLR ? gather_off<F>(fin_lane[k], cw[k])
                                : gather4<F, VEC>(fin[k] + static_cast<unsigned long long>(cw[k]) * R, r, R);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (CHECK && tg[u] == INT_MIN) continue;
          // t = v * prod of all but the last input row; the last multiply is
          // fused into the accumulate (FFMA) when the row repeats
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
      };
      if (full_chunk) {
        for (int jb = j0; jb < j1; jb += U) block(std::false_type{}, jb);
      } else {
        for (int jb = j0; jb < j1; jb += U) block(std::true_type{}, jb);
      }
      if (cur != INT_MIN) flush(cur);
    }
  }
}

// ---- warp-autonomous variant ------------------------------------------------
// Each warp streams its own sub-tiles of kWarpTile consecutive elements:
// coalesced key/value loads into registers, decode, a warp-private counting
// sort by output row (bins + records in the warp's own smem slice), and the
// same 4-lanes-per-element consumption as above — with only __syncwarp, so a
// warp's decode/sort latency is hidden by the other warps instead of being
// serialised behind CTA barriers.
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
        if (hot_slot && !(P.flags & ALTO_STREAM_DBG_NO_HOT)) {
          const int hs = __ldg(hot_slot + row);
          if (hs >= 0) tgt = -(hs + 1);
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
    if (span <= kWarpBins && !(P.flags & ALTO_STREAM_DBG_NO_SORT)) {
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
                            static_cast<long long>(static_cast<unsigned>(sub) & (P.hot_copies - 1)) * P.n_hot * R
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
        if (P.flags & ALTO_STREAM_DBG_NO_RED) {
          if (acc[0] == A(-12345.678)) out[0] = O(1);  // keep the math alive
          return;
        }
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
                if (P.flags & ALTO_STREAM_DBG_NO_GATHER) {
                  const float z = __uint_as_float(cw[k] & 0x3f800000u);
                  g[u][k].v[0] = g[u][k].v[1] = g[u][k].v[2] = g[u][k].v[3] = static_cast<F>(z);
                } else {
                  g[u][k] = FULLR ? gather_off<F>(fin_lane[k], cw[k])
                                  : gather4<F, VEC>(fin[k] + static_cast<unsigned long long>(cw[k]) * R, r, R);
                }
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
  if (P.flags & ALTO_STREAM_CTA_TILES) {
    const size_t stage_bytes = (static_cast<size_t>(P.tile) * (W * 8 + sizeof(V)) + 15) & ~size_t(15);
    const size_t smem = dec + static_cast<size_t>(P.tile) * NW * 4 + kRecPad * 4 +
                        (((kSortBins + kTileWarps) * sizeof(int) + 15) & ~size_t(15)) + 2 * stage_bytes;
    auto kern = stream_kernel<W, V, F, O, NT, G, VEC, FULLR>;
    if (prep(kern, smem)) return ALTO_ECUDA;
    int bps = 1;
    ALTO_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, kTileThreads, smem));
    const long long grid = std::min<long long>(P.ntiles, static_cast<long long>(device_sms()) * std::max(bps, 1));
    kern<<<static_cast<unsigned>(grid), kTileThreads, smem, s>>>(d, tab, P);
    ALTO_LAUNCH_CHECK("alto_mttkrp");
    return ALTO_OK;
  }
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
