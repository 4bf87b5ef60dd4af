// alto_fast.cuh — specialised streaming MTTKRP for the common shapes:
// order N in {3,4,5} and rank R in {16, 32} at compile time, 32-bit factor
// row byte offsets, warp-autonomous 128-element sub-tiles.
//
// Same algorithm as stream_warp_kernel (alto_stream.cuh) — decode, warp
// counting sort by output row, G = R/4 lanes per element, register
// accumulation of row runs, atomic merge, replicated hot rows — written for
// instruction economy: the per-element phase-B loop has no runtime order,
// rank or bounds checks (full sub-tiles), decode extracts key bytes with
// 32-bit funnel shifts and ORs table entries three at a time, and the merge
// address is formed only when a run ends.
#pragma once
#include <type_traits>

#include "alto_stream.cuh"

namespace alto {


// Row merge of one lane group's 4-rank partial (G lanes, ranks 4*gl..4*gl+3):
//  float  -> one RED.F32x4 per lane;
//  double -> 4x4 in-quad transpose, then fp64 REDs covering one sector each;
//  long long (deterministic mode) -> round to fixed point (x * scale, scale a
//            power of two chosen so no partial sum can overflow), transpose,
//            integer REDs: integer addition is associative, so the merged
//            result does not depend on the order in which tiles arrive.
template <typename O, typename A, int G, int R>
__device__ __forceinline__ void merge_row(O* base, const A (&acc)[4], int gl, unsigned qmask, int lane,
                                          double scale) {
  if constexpr (std::is_same<O, float>::value) {
    red_f32x4(reinterpret_cast<float*>(base), acc, 4 * gl, R, true);
  } else if constexpr (std::is_same<O, double>::value) {
    red_f64_sectors(reinterpret_cast<double*>(base), acc, 4 * gl, R, G, qmask, lane);
  } else {
    static_assert(G >= 4 && R % 16 == 0, "fixed-point merge needs full lane quads");
    long long v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] = __double2ll_rn(static_cast<double>(acc[q]) * scale);
    const int l = lane & 3;
    quad_transpose(v, qmask, l);
    const int b0 = 4 * gl - 4 * l;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      atomicAdd(reinterpret_cast<unsigned long long*>(base + b0 + 4 * q + l), static_cast<unsigned long long>(v[q]));
  }
}

constexpr int kFastTile = 128;  // elements per warp sub-tile
constexpr int kFastBins = 512;

// Packed-coordinate decode of one key (W words) with DB key bytes.
template <int W>
__device__ __forceinline__ void fast_decode(const uint64_t* __restrict__ tab, int db, const Key<W>& k,
                                            unsigned (&p)[2 * W]) {
#pragma unroll
  for (int i = 0; i < 2 * W; ++i) p[i] = 0u;
#pragma unroll
  for (int j = 0; j < 8 * W; ++j) {
    if (j < db) {
      const unsigned word = static_cast<unsigned>(k.w[j >> 3] >> (32 * ((j >> 2) & 1)));
      const unsigned b = (word >> (8 * (j & 3))) & 0xffu;
      if constexpr (W == 1) {
        const uint2 e = *reinterpret_cast<const uint2*>(tab + j * 256 + b);
        p[0] |= e.x;
        p[1] |= e.y;
      } else {
        const uint4 e = *reinterpret_cast<const uint4*>(tab + (j * 256 + b) * 2);
        p[0] |= e.x;
        p[1] |= e.y;
        p[2] |= e.z;
        p[3] |= e.w;
      }
    }
  }
}

// Field [off, off + nb) (nb <= 31) of the packed coordinate words.
template <int W>
__device__ __forceinline__ unsigned fast_field(const unsigned (&p)[2 * W], int off, int nb) {
  const int wi = off >> 5, sh = off & 31;
  unsigned lo = p[0], hi = p[1 < 2 * W ? 1 : 0];
#pragma unroll
  for (int i = 1; i < 2 * W; ++i)
    if (i == wi) { lo = p[i]; hi = (i + 1 < 2 * W) ? p[i + 1] : 0u; }
  const unsigned v = __funnelshift_r(lo, hi, sh);
  return nb >= 32 ? v : (v & ((1u << nb) - 1u));
}

template <int W, typename V, typename O, int N, int R, int MINB = 3, int UF = 2>
__global__ void __launch_bounds__(kTileThreads, MINB)
fast_kernel(const __grid_constant__ DevLayout L, const uint64_t* __restrict__ tab,
            const __grid_constant__ StreamParams P) {
  using F = V;
  using A = V;
  constexpr int G = R / 4;                  // lanes per element
  constexpr int GPW = 32 / G;               // element groups per warp
  constexpr int CH = kFastTile / GPW;       // records per group
  constexpr int NIN = N - 1;
  using RL = RecLayout<N, V>;
  constexpr int NW = RL::NW;
  constexpr int EPL = kFastTile / 32;
  constexpr int U = UF;
  constexpr int REC_WORDS = kFastTile * NW + GPW * 4;
  extern __shared__ __align__(16) unsigned char smem[];
  const int mode = P.mode;
  uint64_t* s_dec = reinterpret_cast<uint64_t*>(smem);
  const size_t off0 = (static_cast<size_t>(L.dec_bytes) * 256 * W * 8 + 15) & ~size_t(15);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned* s_rec = reinterpret_cast<unsigned*>(smem + off0) + warp * (REC_WORDS + kFastBins);
  int* s_bin = reinterpret_cast<int*>(s_rec + REC_WORDS);
  copy_to_smem(s_dec, tab + static_cast<long long>(L.dec_off) * W, L.dec_bytes * 256 * W);
  __syncthreads();

  const int grp = lane / G;
  const int gl = lane % G;
  const unsigned qmask = (G >= 4) ? (0xFu << (lane & ~3)) : 0xffffffffu;
  const char* fin_lane[NIN];
#pragma unroll
  for (int k = 0; k < NIN; ++k) {
    const int n = k < mode ? k : k + 1;
    fin_lane[k] = reinterpret_cast<const char*>(static_cast<const F*>(P.factors[n]) + 4 * gl);
  }
  int pack_off[N], bits[N];
#pragma unroll
  for (int n = 0; n < N; ++n) { pack_off[n] = L.pack_off[n]; bits[n] = L.bits[n]; }
  const int db = L.dec_bytes;
  const V* __restrict__ vals = static_cast<const V*>(P.values);
  O* __restrict__ out = static_cast<O*>(P.out);
  const double fixed_scale = P.fixed_scale ? *P.fixed_scale : 1.0;
  const int* __restrict__ hot_slot = P.n_hot > 0 ? P.hot_slot : nullptr;
  constexpr unsigned ROWB = static_cast<unsigned>(R * sizeof(F));  // factor row bytes
  // swizzled record address (words): chunk c shifted by 16*c bytes
  auto rec_addr = [](int j) { return j * NW + (j / CH) * 4; };

  const long long nsub = (P.m + kFastTile - 1) / kFastTile;
  const long long gw0 = static_cast<long long>(blockIdx.x) * (kTileThreads / 32) + warp;
  (void)0;
  const long long nwarps = static_cast<long long>(gridDim.x) * (kTileThreads / 32);
  // keys/values of the warp's next sub-tile are loaded into registers while
  // the current one is sorted and consumed (hides the DRAM latency)
  Key<W> nk[EPL];
  V nv[EPL];
  auto prefetch = [&](long long sb) {
    if (sb >= nsub) return;
    const long long b0 = sb * kFastTile;
    const int c = static_cast<int>(min(static_cast<long long>(kFastTile), P.m - b0));
#pragma unroll
    for (int k = 0; k < EPL; ++k) {
      const int e = lane + 32 * k;
      if (e < c) {
        nk[k] = load_key<W>(P.keys, b0 + e);
        nv[k] = __ldg(vals + b0 + e);
      }
    }
  };
  prefetch(gw0);
  for (long long sub = gw0; sub < nsub; sub += nwarps) {
    const long long e0 = sub * kFastTile;
    const int cnt = static_cast<int>(min(static_cast<long long>(kFastTile), P.m - e0));
    // ---- load + decode (lane per element) ----------------------------------
    Key<W> kk[EPL];
    V vv0[EPL];
#pragma unroll
    for (int k = 0; k < EPL; ++k) {
      kk[k] = nk[k];
      vv0[k] = nv[k];
    }
    prefetch(sub + nwarps);
    unsigned rec[EPL][NW];
    int myrow[EPL];
    int lo = INT_MAX, hi = INT_MIN;
#pragma unroll
    for (int k = 0; k < EPL; ++k) {
      const int e = lane + 32 * k;
      myrow[k] = -1;
      if (e < cnt) {
        unsigned p[2 * W];
        fast_decode<W>(s_dec, db, kk[k], p);
        unsigned c[N];
#pragma unroll
        for (int n = 0; n < N; ++n) c[n] = fast_field<W>(p, pack_off[n], bits[n]);
        unsigned row = c[0];
#pragma unroll
        for (int n = 1; n < N; ++n)
          if (n == mode) row = c[n];
#pragma unroll
        for (int q = 0; q < NIN; ++q) rec[k][q] = ((q < mode) ? c[q] : c[q + 1]) * ROWB;
        int tgt = static_cast<int>(row);
        if (hot_slot) {
          const int hs = __ldg(hot_slot + row);
          if (hs >= 0)  // adaptive plan: copy (sub-tile mod copies) of the row's own copies
            tgt = P.hot_adaptive ? -((hs >> 5) + static_cast<int>(static_cast<unsigned>(sub) & ((1u << (hs & 31)) - 1u)) + 1)
                                 : -(hs + 1);
        }
        rec[k][RL::TGT] = static_cast<unsigned>(tgt);
        if constexpr (sizeof(V) == 4) {
          rec[k][RL::VAL] = __float_as_uint(vv0[k]);
        } else {
          const unsigned long long u = __double_as_longlong(vv0[k]);
          rec[k][RL::VAL] = static_cast<unsigned>(u);
          rec[k][RL::VAL + 1] = static_cast<unsigned>(u >> 32);
        }
#pragma unroll
        for (int q = RL::raw; q < NW; ++q) rec[k][q] = 0u;
        myrow[k] = static_cast<int>(row);
        lo = min(lo, myrow[k]);
        hi = max(hi, myrow[k]);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    const int span = hi - lo + 1;
    // ---- warp counting sort by output row ----------------------------------
    if (span <= kFastBins) {
      for (int i = lane; i < span; i += 32) s_bin[i] = 0;
      __syncwarp();
      // histogram: one atomic per group of equal rows (hot rows repeat a lot)
      unsigned peers[EPL];
      const unsigned ltm = (1u << lane) - 1u;
#pragma unroll
      for (int k = 0; k < EPL; ++k) {
        const bool ok = myrow[k] >= 0;
        peers[k] = __match_any_sync(0xffffffffu, ok ? myrow[k] : -1 - lane);
        if (ok && (peers[k] & ltm) == 0) atomicAdd(&s_bin[myrow[k] - lo], __popc(peers[k]));
      }
      __syncwarp();
      // exclusive scan over the span in conflict-free 32-bin rounds
      int carry = 0;
      for (int base = 0; base < span; base += 32) {
        const int i = base + lane;
        const int v = i < span ? s_bin[i] : 0;
        int x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        if (i < span) s_bin[i] = carry + x - v;
        carry += __shfl_sync(0xffffffffu, x, 31);
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < EPL; ++k) {
        const bool ok = myrow[k] >= 0;
        const int leader = __ffs(peers[k]) - 1;
        int basev = 0;
        if (ok && leader == lane) basev = atomicAdd(&s_bin[myrow[k] - lo], __popc(peers[k]));
        basev = __shfl_sync(0xffffffffu, basev, leader);
        if (ok) {
          const int slot = basev + __popc(peers[k] & ltm);
#pragma unroll
          for (int q = 0; q < NW; q += 4)
            *reinterpret_cast<uint4*>(s_rec + rec_addr(slot) + q) =
                make_uint4(rec[k][q], rec[k][q + 1], rec[k][q + 2], rec[k][q + 3]);
        }
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
    // ---- consume: G lanes per element, 4 ranks per lane ---------------------
    O* hot_base = hot_slot ? static_cast<O*>(P.hot_buf) +
                                 (P.hot_adaptive ? 0ll
                                                 : static_cast<long long>(static_cast<unsigned>(sub) & (P.hot_copies - 1)) *
                                                       P.n_hot * R)
                           : nullptr;
    A acc[4] = {A(0), A(0), A(0), A(0)};
    int cur = INT_MIN;
    auto flush = [&]() {
      O* base = cur >= 0 ? out + static_cast<long long>(cur) * R : hot_base + static_cast<long long>(-cur - 1) * R;
      merge_row<O, A, G, R>(base, acc, gl, qmask, lane, fixed_scale);
    };
    auto consume = [&](const unsigned (&cw)[NW], const V4<F> (&g)[NIN]) {
      const int tg = static_cast<int>(cw[RL::TGT]);
      A v;
      if constexpr (sizeof(V) == 4) {
        v = __uint_as_float(cw[RL::VAL]);
      } else {
        v = __longlong_as_double(
            static_cast<long long>((static_cast<unsigned long long>(cw[RL::VAL + 1]) << 32) | cw[RL::VAL]));
      }
      A t[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) t[q] = v * static_cast<A>(g[0].v[q]);
#pragma unroll
      for (int k = 1; k < NIN - 1; ++k)
#pragma unroll
        for (int q = 0; q < 4; ++q) t[q] *= static_cast<A>(g[k].v[q]);
      if (tg == cur) {
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[q] = fma(t[q], static_cast<A>(g[NIN - 1].v[q]), acc[q]);
      } else {
        if (cur != INT_MIN) flush();
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[q] = t[q] * static_cast<A>(g[NIN - 1].v[q]);
        cur = tg;
      }
    };
    const int j0 = grp * CH;
    if (cnt == kFastTile) {
#pragma unroll 1
      for (int jb = j0; jb < j0 + CH; jb += U) {
        unsigned cw[U][NW];
        V4<F> g[U][NIN];
#pragma unroll
        for (int u = 0; u < U; ++u) {
#pragma unroll
          for (int q = 0; q < NW; q += 4) {
            const uint4 t = *reinterpret_cast<const uint4*>(s_rec + rec_addr(jb + u) + q);
            cw[u][q] = t.x; cw[u][q + 1] = t.y; cw[u][q + 2] = t.z; cw[u][q + 3] = t.w;
          }
#pragma unroll
          for (int k = 0; k < NIN; ++k) g[u][k] = gather_off<F>(fin_lane[k], cw[u][k]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) consume(cw[u], g[u]);
      }
    } else {
      const int j1 = min(cnt, j0 + CH);
#pragma unroll 1
      for (int j = j0; j < j1; ++j) {
        unsigned cw[NW];
        V4<F> g[NIN];
#pragma unroll
        for (int q = 0; q < NW; q += 4) {
          const uint4 t = *reinterpret_cast<const uint4*>(s_rec + rec_addr(j) + q);
          cw[q] = t.x; cw[q + 1] = t.y; cw[q + 2] = t.z; cw[q + 3] = t.w;
        }
#pragma unroll
        for (int k = 0; k < NIN; ++k) g[k] = gather_off<F>(fin_lane[k], cw[k]);
        consume(cw, g);
      }
    }
    if (cur != INT_MIN) flush();
    __syncwarp();
  }
}

template <int W, typename V, typename O, int N, int R, int MINB = 3, int UF = 2>
int launch_fast(const DevLayout& d, const uint64_t* tab, const StreamParams& P, cudaStream_t s) {
  constexpr int NW = RecLayout<N, V>::NW;
  constexpr int GPW = 32 / (R / 4);
  const size_t dec = (static_cast<size_t>(d.dec_bytes) * 256 * W * 8 + 15) & ~size_t(15);
  const size_t smem = dec + (kTileThreads / 32) * (static_cast<size_t>(kFastTile) * NW + GPW * 4 + kFastBins) * 4;
  auto kern = fast_kernel<W, V, O, N, R, MINB, UF>;
  // launch configuration cached per instantiation and shared-memory size
  static size_t cached_smem = 0;
  static int cached_bps = 0;
  if (cached_smem != smem) {
    if (prep(kern, smem)) return ALTO_ECUDA;
    int b = 1;
    ALTO_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, kTileThreads, smem));
    cached_bps = b;
    cached_smem = smem;
  }
  const int bps = cached_bps;
  const long long nsub = (P.m + kFastTile - 1) / kFastTile;
  const long long need = (nsub + kTileThreads / 32 - 1) / (kTileThreads / 32);
  const long long grid = std::min<long long>(need, static_cast<long long>(device_sms()) * std::max(bps, 1));
  kern<<<static_cast<unsigned>(grid), kTileThreads, smem, s>>>(d, tab, P);
  ALTO_LAUNCH_CHECK("alto_mttkrp(fast)");
  return ALTO_OK;
}

// Returns ALTO_EUNSUPPORTED (without launching) when the shape is not covered.
template <int W, typename V, typename O>
int try_planned(const DevLayout& d, const StreamParams& P, const uint64_t* packed, const unsigned char* pos,
                cudaStream_t s);
template <int W, typename V, typename O>
int try_mstream(const DevLayout& d, const StreamParams& P, cudaStream_t s);

template <int W, typename V, typename O>
int try_fast(const DevLayout& d, const uint64_t* tab, const StreamParams& P, cudaStream_t s) {
  if (P.flags & ALTO_STREAM_GENERIC) return ALTO_EUNSUPPORTED;
  if (P.mkeys) {
    // a mode stream pins the kernel (its hot copies are float64 for float32 output)
    const int st = try_mstream<W, V, O>(d, P, s);
    if (st == ALTO_EUNSUPPORTED) set_error("shape not covered by the mode-stream kernel");
    return st;
  }
  if (P.packed && P.pos) {
    const int st = try_planned<W, V, O>(d, P, P.packed, P.pos, s);
    if (st != ALTO_EUNSUPPORTED) return st;
  }
  long long maxdim = 0;
  for (int n = 0; n < d.order; ++n) maxdim = std::max(maxdim, d.dims[n]);
  if (maxdim * P.rank * static_cast<long long>(sizeof(V)) > 0xFFFFFFFFll) return ALTO_EUNSUPPORTED;
  for (int n = 0; n < d.order; ++n)
    if (d.bits[n] > 31) return ALTO_EUNSUPPORTED;
  if (P.rank == 16) {
    if (d.order == 3) return launch_fast<W, V, O, 3, 16>(d, tab, P, s);
    if (d.order == 4) return launch_fast<W, V, O, 4, 16>(d, tab, P, s);
    if (d.order == 5) return launch_fast<W, V, O, 5, 16>(d, tab, P, s);
  }
  if (P.rank == 32) {
    if (d.order == 3) return launch_fast<W, V, O, 3, 32>(d, tab, P, s);
    if (d.order == 4) return launch_fast<W, V, O, 4, 32>(d, tab, P, s);
    if (d.order == 5) return launch_fast<W, V, O, 5, 32>(d, tab, P, s);
  }
  return ALTO_EUNSUPPORTED;
}


// ---- planned variant: mode-contiguous keys + precomputed sub-tile order --------
// Built once per tensor (packed keys) and per mode (positions) — see
// alto_pack_keys / alto_subtile_order.  The packed key is the ALTO key with
// its bits permuted so that mode n occupies bits [pack_off[n], +bits[n]):
// same bits, same element order, decode = one funnel shift + mask per mode.
// pos[e] is element e's slot in its 128-element sub-tile after a stable
// counting sort by output row (identity when the sub-tile's rows span more
// than kFastBins), so phase A scatters records without any sorting work.

template <int W>
__device__ __forceinline__ unsigned packed_field32(const Key<W>& k, int off, int nb) {
  unsigned w[2 * W];
#pragma unroll
  for (int i = 0; i < W; ++i) {
    w[2 * i] = static_cast<unsigned>(k.w[i]);
    w[2 * i + 1] = static_cast<unsigned>(k.w[i] >> 32);
  }
  return fast_field<W>(w, off, nb);
}

// Gathered inputs of the planned kernel when input modes are paired (float32,
// rank 16, orders 4-5; alto_krp_pair tables): input k is the table `tab` with
// row c[na] * db + c[nb] (nb < 0: a plain factor, row c[na]).
struct PlanIn {
  const void* tab[ALTO_MAX_ORDER];
  int na[ALTO_MAX_ORDER], nb[ALTO_MAX_ORDER];
  unsigned db[ALTO_MAX_ORDER];
};

template <int W, typename V, typename O, int N, int R, int MINB = 3, int UF = 2, int NV = N - 1>
__global__ void __launch_bounds__(kTileThreads, MINB)
planned_kernel(const __grid_constant__ DevLayout L, const uint64_t* __restrict__ packed,
               const unsigned char* __restrict__ pos, const __grid_constant__ StreamParams P,
               const __grid_constant__ PlanIn Q) {
  using F = V;
  using A = V;
  constexpr int G = R / 4;
  constexpr int GPW = 32 / G;
  constexpr int CH = kFastTile / GPW;
  constexpr int NIN = NV;
  constexpr bool PAIR = NV < N - 1;
  using RL = RecLayout<NV + 1, V>;
  constexpr int NW = RL::NW;
  constexpr int EPL = kFastTile / 32;
  constexpr int U = UF;
  constexpr int REC_WORDS = kFastTile * NW + GPW * 4;
  extern __shared__ __align__(16) unsigned char smem[];
  const int mode = P.mode;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned* s_rec = reinterpret_cast<unsigned*>(smem) + warp * REC_WORDS;
  const int grp = lane / G;
  const int gl = lane % G;
  const unsigned qmask = (G >= 4) ? (0xFu << (lane & ~3)) : 0xffffffffu;
  const char* fin_lane[NIN];
#pragma unroll
  for (int k = 0; k < NIN; ++k) {
    if constexpr (PAIR) {
      fin_lane[k] = reinterpret_cast<const char*>(static_cast<const F*>(Q.tab[k]) + 4 * gl);
    } else {
      const int n = k < mode ? k : k + 1;
      fin_lane[k] = reinterpret_cast<const char*>(static_cast<const F*>(P.factors[n]) + 4 * gl);
    }
  }
  int pack_off[N], bits[N];
#pragma unroll
  for (int n = 0; n < N; ++n) { pack_off[n] = L.pack_off[n]; bits[n] = L.bits[n]; }
  const V* __restrict__ vals = static_cast<const V*>(P.values);
  O* __restrict__ out = static_cast<O*>(P.out);
  const double fixed_scale = P.fixed_scale ? *P.fixed_scale : 1.0;
  const int* __restrict__ hot_slot = P.n_hot > 0 ? P.hot_slot : nullptr;
  constexpr unsigned ROWB = static_cast<unsigned>(R * sizeof(F));
  auto rec_addr = [](int j) { return j * NW + (j / CH) * 4; };

  const long long nsub = (P.m + kFastTile - 1) / kFastTile;
  const long long gw0 = static_cast<long long>(blockIdx.x) * (kTileThreads / 32) + warp;
  const long long nwarps = static_cast<long long>(gridDim.x) * (kTileThreads / 32);
  Key<W> nk[EPL];
  V nv[EPL];
  unsigned char np[EPL];
  auto prefetch = [&](long long sb) {
    if (sb >= nsub) return;
    const long long b0 = sb * kFastTile;
    const int c = static_cast<int>(min(static_cast<long long>(kFastTile), P.m - b0));
#pragma unroll
    for (int k = 0; k < EPL; ++k) {
      const int e = lane + 32 * k;
      if (e < c) {
        nk[k] = load_key<W>(packed, b0 + e);
        nv[k] = __ldg(vals + b0 + e);
        np[k] = __ldg(pos + b0 + e);
      }
    }
  };
  prefetch(gw0);
  for (long long sub = gw0; sub < nsub; sub += nwarps) {
    const long long e0 = sub * kFastTile;
    const int cnt = static_cast<int>(min(static_cast<long long>(kFastTile), P.m - e0));
    Key<W> kk[EPL];
    V vv0[EPL];
    unsigned char pp[EPL];
#pragma unroll
    for (int k = 0; k < EPL; ++k) { kk[k] = nk[k]; vv0[k] = nv[k]; pp[k] = np[k]; }
    prefetch(sub + nwarps);
    // ---- records straight to their sorted slots ------------------------------
#pragma unroll
    for (int k = 0; k < EPL; ++k) {
      const int e = lane + 32 * k;
      if (e < cnt) {
        unsigned c[N];
#pragma unroll
        for (int n = 0; n < N; ++n) c[n] = packed_field32<W>(kk[k], pack_off[n], bits[n]);
        unsigned row = c[0];
#pragma unroll
        for (int n = 1; n < N; ++n)
          if (n == mode) row = c[n];
        unsigned rec[NW];
#pragma unroll
        for (int q = 0; q < NIN; ++q) {
          if constexpr (PAIR) {
            // decoded again with the pair's run-time modes (indexing c[] by them would spill it)
            const unsigned ca = packed_field32<W>(kk[k], L.pack_off[Q.na[q]], L.bits[Q.na[q]]);
            const unsigned cb = Q.nb[q] >= 0 ? packed_field32<W>(kk[k], L.pack_off[Q.nb[q]], L.bits[Q.nb[q]]) : 0u;
            rec[q] = (ca * Q.db[q] + cb) * ROWB;
          } else {
            rec[q] = ((q < mode) ? c[q] : c[q + 1]) * ROWB;
          }
        }
        int tgt = static_cast<int>(row);
        if (hot_slot) {
          const int hs = __ldg(hot_slot + row);
          if (hs >= 0)  // adaptive plan: copy (sub-tile mod copies) of the row's own copies
            tgt = P.hot_adaptive ? -((hs >> 5) + static_cast<int>(static_cast<unsigned>(sub) & ((1u << (hs & 31)) - 1u)) + 1)
                                 : -(hs + 1);
        }
        rec[RL::TGT] = static_cast<unsigned>(tgt);
        if constexpr (sizeof(V) == 4) {
          rec[RL::VAL] = __float_as_uint(vv0[k]);
        } else {
          const unsigned long long u = __double_as_longlong(vv0[k]);
          rec[RL::VAL] = static_cast<unsigned>(u);
          rec[RL::VAL + 1] = static_cast<unsigned>(u >> 32);
        }
#pragma unroll
        for (int q = RL::raw; q < NW; ++q) rec[q] = 0u;
        const int slot = pp[k];
#pragma unroll
        for (int q = 0; q < NW; q += 4)
          *reinterpret_cast<uint4*>(s_rec + rec_addr(slot) + q) = make_uint4(rec[q], rec[q + 1], rec[q + 2], rec[q + 3]);
      }
    }
    __syncwarp();
    // ---- consume (identical to fast_kernel) -------------------------------------
    O* hot_base = hot_slot ? static_cast<O*>(P.hot_buf) +
                                 (P.hot_adaptive ? 0ll
                                                 : static_cast<long long>(static_cast<unsigned>(sub) & (P.hot_copies - 1)) *
                                                       P.n_hot * R)
                           : nullptr;
    A acc[4] = {A(0), A(0), A(0), A(0)};
    int cur = INT_MIN;
    auto flush = [&]() {
      O* base = cur >= 0 ? out + static_cast<long long>(cur) * R : hot_base + static_cast<long long>(-cur - 1) * R;
      merge_row<O, A, G, R>(base, acc, gl, qmask, lane, fixed_scale);
    };
    auto consume = [&](const unsigned (&cw)[NW], const V4<F> (&g)[NIN]) {
      const int tg = static_cast<int>(cw[RL::TGT]);
      A v;
      if constexpr (sizeof(V) == 4) {
        v = __uint_as_float(cw[RL::VAL]);
      } else {
        v = __longlong_as_double(
            static_cast<long long>((static_cast<unsigned long long>(cw[RL::VAL + 1]) << 32) | cw[RL::VAL]));
      }
      A t[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) t[q] = v * static_cast<A>(g[0].v[q]);
#pragma unroll
      for (int k = 1; k < NIN - 1; ++k)
#pragma unroll
        for (int q = 0; q < 4; ++q) t[q] *= static_cast<A>(g[k].v[q]);
      if (tg == cur) {
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[q] = fma(t[q], static_cast<A>(g[NIN - 1].v[q]), acc[q]);
      } else {
        if (cur != INT_MIN) flush();
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[q] = t[q] * static_cast<A>(g[NIN - 1].v[q]);
        cur = tg;
      }
    };
    const int j0 = grp * CH;
    if (cnt == kFastTile) {
#pragma unroll 1
      for (int jb = j0; jb < j0 + CH; jb += U) {
        unsigned cw[U][NW];
        V4<F> g[U][NIN];
#pragma unroll
        for (int u = 0; u < U; ++u) {
#pragma unroll
          for (int q = 0; q < NW; q += 4) {
            const uint4 t = *reinterpret_cast<const uint4*>(s_rec + rec_addr(jb + u) + q);
            cw[u][q] = t.x; cw[u][q + 1] = t.y; cw[u][q + 2] = t.z; cw[u][q + 3] = t.w;
          }
#pragma unroll
          for (int k = 0; k < NIN; ++k) g[u][k] = gather_off<F>(fin_lane[k], cw[u][k]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) consume(cw[u], g[u]);
      }
    } else {
      const int j1 = min(cnt, j0 + CH);
#pragma unroll 1
      for (int j = j0; j < j1; ++j) {
        unsigned cw[NW];
        V4<F> g[NIN];
#pragma unroll
        for (int q = 0; q < NW; q += 4) {
          const uint4 t = *reinterpret_cast<const uint4*>(s_rec + rec_addr(j) + q);
          cw[q] = t.x; cw[q + 1] = t.y; cw[q + 2] = t.z; cw[q + 3] = t.w;
        }
#pragma unroll
        for (int k = 0; k < NIN; ++k) g[k] = gather_off<F>(fin_lane[k], cw[k]);
        consume(cw, g);
      }
    }
    if (cur != INT_MIN) flush();
    __syncwarp();
  }
}

template <int W, typename V, typename O, int N, int R, int NV = N - 1>
int launch_planned(const DevLayout& d, const StreamParams& P, const uint64_t* packed, const unsigned char* pos,
                   cudaStream_t s, const PlanIn& Q = PlanIn{}) {
  constexpr int NW = RecLayout<NV + 1, V>::NW;
  constexpr int GPW = 32 / (R / 4);
  const size_t smem = (kTileThreads / 32) * (static_cast<size_t>(kFastTile) * NW + GPW * 4) * 4;
  auto kern = planned_kernel<W, V, O, N, R, 3, 2, NV>;
  static size_t cached_smem = 0;
  static int cached_bps = 0;
  if (cached_smem != smem) {
    if (prep(kern, smem)) return ALTO_ECUDA;
    int b = 1;
    ALTO_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, kTileThreads, smem));
    cached_bps = b;
    cached_smem = smem;
  }
  const long long nsub = (P.m + kFastTile - 1) / kFastTile;
  const long long need = (nsub + kTileThreads / 32 - 1) / (kTileThreads / 32);
  const long long grid = std::min<long long>(need, static_cast<long long>(device_sms()) * std::max(cached_bps, 1));
  kern<<<static_cast<unsigned>(grid), kTileThreads, smem, s>>>(d, packed, pos, P, Q);
  ALTO_LAUNCH_CHECK("alto_mttkrp(planned)");
  return ALTO_OK;
}

template <int W, typename V, typename O>
int try_planned(const DevLayout& d, const StreamParams& P, const uint64_t* packed, const unsigned char* pos,
                cudaStream_t s) {
  if (!packed || !pos || (P.flags & ALTO_STREAM_GENERIC)) return ALTO_EUNSUPPORTED;
  long long maxdim = 0;
  for (int n = 0; n < d.order; ++n) maxdim = std::max(maxdim, d.dims[n]);
  if (maxdim * P.rank * static_cast<long long>(sizeof(V)) > 0xFFFFFFFFll) return ALTO_EUNSUPPORTED;
  for (int n = 0; n < d.order; ++n)
    if (d.bits[n] > 31) return ALTO_EUNSUPPORTED;
  if (P.n_pairs > 0) {
    // paired input modes (alto_krp_pair tables): float32 data, rank 16, orders 4-5
    if constexpr (sizeof(V) == 4 && !std::is_same<O, long long>::value) {
      if (P.rank != 16 || d.order < 4) return ALTO_EUNSUPPORTED;
      PlanIn Q{};
      int nv = 0;
      unsigned used = 1u << P.mode;
      for (int i = 0; i < P.n_pairs; ++i) {
        const int a = P.pair_a[i], b = P.pair_b[i];
        if (a < 0 || b < 0 || a >= d.order || b >= d.order || a == b || ((used >> a) & 1u) || ((used >> b) & 1u) ||
            !P.pair_tab[i] || d.dims[a] * d.dims[b] * P.rank * static_cast<long long>(sizeof(V)) > 0xFFFFFFFFll)
          return ALTO_EUNSUPPORTED;
        used |= (1u << a) | (1u << b);
        Q.tab[nv] = P.pair_tab[i];
        Q.na[nv] = a;
        Q.nb[nv] = b;
        Q.db[nv] = static_cast<unsigned>(d.dims[b]);
        ++nv;
      }
      for (int n = 0; n < d.order; ++n)
        if (!((used >> n) & 1u)) {
          Q.tab[nv] = P.factors[n];
          Q.na[nv] = n;
          Q.nb[nv] = -1;
          Q.db[nv] = 1u;
          ++nv;
        }
      if (d.order == 4 && nv == 2) return launch_planned<W, V, O, 4, 16, 2>(d, P, packed, pos, s, Q);
      if (d.order == 5 && nv == 3) return launch_planned<W, V, O, 5, 16, 3>(d, P, packed, pos, s, Q);
      if (d.order == 5 && nv == 2) return launch_planned<W, V, O, 5, 16, 2>(d, P, packed, pos, s, Q);
    }
    return ALTO_EUNSUPPORTED;
  }
  if (P.rank == 16) {
    if (d.order == 3) return launch_planned<W, V, O, 3, 16>(d, P, packed, pos, s);
    if (d.order == 4) return launch_planned<W, V, O, 4, 16>(d, P, packed, pos, s);
    if (d.order == 5) return launch_planned<W, V, O, 5, 16>(d, P, packed, pos, s);
  }
  if (P.rank == 32) {
    if (d.order == 3) return launch_planned<W, V, O, 3, 32>(d, P, packed, pos, s);
    if (d.order == 4) return launch_planned<W, V, O, 4, 32>(d, P, packed, pos, s);
    if (d.order == 5) return launch_planned<W, V, O, 5, 32>(d, P, packed, pos, s);
  }
  return ALTO_EUNSUPPORTED;
}

}  // namespace alto
