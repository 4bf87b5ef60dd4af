// alto_mstream.cuh — mode-stream MTTKRP: the streaming ALTO MTTKRP over a
// per-mode copy of the ALTO stream that is already in the order the kernel
// consumes it.
//
// The per-mode stream (built once per tensor and mode by alto_mode_stream,
// like the reference's per-mode plans and flagged key copies in
// _make_backend, pkg/src/altotensor/cpd.py:149-181) holds the same elements,
// keys (mode-contiguous bit order, alto_pack_keys) and values as the sorted
// ALTO stream, cut into tiles of T consecutive elements — contiguous
// linearized-key ranges, i.e. ALTO partitions (format.py:127-154) — and, inside
// each tile, stably sorted by the output-mode coordinate (the per-partition
// interval buffer of the paper's Buffered scheme, Alg. 2 / mttkrp.py:148-156,
// at tile granularity) and split into 8 slices of T/8 elements stored
// interleaved: sorted position p of tile t lives at t*T + (p % CH)*8 + p / CH
// (CH = T/8).  Rows of the mode's hot plan carry a flag in the key's top bit.
//
// Kernel: a warp owns a tile; G = R/4 lanes own one slice each (4 consecutive
// ranks per lane, a factor row is one contiguous 16*G-byte request); the 8
// slices of instruction j are 8 consecutive keys/values (one coalesced
// request each).  Every lane decodes its slice's element with shifts,
// gathers the N-1 input rows with U elements in flight, forms the Hadamard
// product and accumulates in registers while the output row repeats; on a
// row change the partial row is merged with one RED.F32x4 per lane (float32),
// sector-covering float64 REDs, or int64 fixed-point REDs (deterministic).
// Hot rows (a Zipf head row is touched by nearly every tile) merge into one of
// that row's replicated partial rows (tile mod copies; copies per row sized by
// alto_hot_copies so each receives a bounded number of merges), summed
// afterwards in a fixed order by hot_reduce_rows_kernel.
//
// Compared with planned_kernel (alto_fast.cuh) this removes the in-kernel
// record pass through shared memory (phase A), the per-element plan byte and
// hot-slot lookups, and lets tiles be long (1024-4096 elements: fewer row
// runs, hence fewer merges) because no per-tile state lives on chip.
#pragma once
#include "alto_fast.cuh"

namespace alto {

constexpr int kMsSlices = 8;  // slices per tile (lane groups of a rank-16 warp)

// Stream loads bypass L1 and carry an L2 eviction policy (evict_first by
// default: the stream is read once, the factor rows and output rows it
// touches should keep the L2).
__device__ __forceinline__ unsigned long long stream_policy(bool evict_first) {
  unsigned long long p;
  if (evict_first)
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  else
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}

template <int W>
__device__ __forceinline__ Key<W> load_key_stream(const uint64_t* __restrict__ keys, long long i,
                                                  unsigned long long pol) {
  Key<W> k;
  if constexpr (W == 1) {
    unsigned long long v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(keys + i), "l"(pol));
    k.w[0] = v;
  } else {
    unsigned long long a, b;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u64 {%0, %1}, [%2], %3;"
        : "=l"(a), "=l"(b)
        : "l"(keys + 2 * i), "l"(pol));
    k.w[0] = a;
    k.w[1] = b;
  }
  return k;
}

template <typename V>
__device__ __forceinline__ V load_val_stream(const V* __restrict__ p, unsigned long long pol) {
  if constexpr (sizeof(V) == 4) {
    float v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    return v;
  } else {
    double v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
  }
}

// Field layout of a per-mode stream key: the coordinates of the input modes
// (ascending) and then of the output mode, packed from bit 0 without any
// field straddling a 64-bit word; bit 64W-1 is the hot-row flag.
struct MsFields {
  int word[ALTO_MAX_ORDER];
  int sh[ALTO_MAX_ORDER];
  unsigned mask[ALTO_MAX_ORDER];
  int ok;  // layout fits below the flag bit
};

inline MsFields ms_fields(const DevLayout& d, int mode) {
  MsFields f{};
  int cur = 0;
  for (int i = 0; i < d.order; ++i) {
    const int n = i < d.order - 1 ? (i < mode ? i : i + 1) : mode;
    const int b = d.bits[n];
    if ((cur & 63) + b > 64) cur = (cur + 63) & ~63;
    f.word[n] = cur >> 6;
    f.sh[n] = cur & 63;
    f.mask[n] = b >= 32 ? 0xffffffffu : ((1u << b) - 1u);
    cur += b;
  }
  f.ok = cur <= 64 * d.n_words - 1;
  return f;
}

// Delta stream layout (ALTO_MS_DELTA, 128-bit layouts): one 64-bit word per
// element holding the input-mode coordinates (ascending, no field straddling
// bit 63) and, in place of the output coordinate, the row increment from the
// previous element of the same lane group (its base row is stored per group,
// alto_mode_stream base_rows); bit 63 = hot-row flag.  `ok` needs at least 8
// increment bits.
inline MsFields ms_fields_delta(const DevLayout& d, int mode) {
  MsFields f{};
  int cur = 0;
  for (int n = 0; n < d.order; ++n) {
    if (n == mode) continue;
    f.word[n] = 0;
    f.sh[n] = cur;
    f.mask[n] = d.bits[n] >= 32 ? 0xffffffffu : ((1u << d.bits[n]) - 1u);
    cur += d.bits[n];
  }
  const int db = std::min(31, 63 - cur);
  f.word[mode] = 0;
  f.sh[mode] = cur;
  f.mask[mode] = db >= 1 ? ((1u << db) - 1u) : 0u;
  f.ok = db >= 8;
  return f;
}

// One field selector held in registers (hoisted out of the element loops).
struct FSel {
  unsigned sh, mask;
  bool hi;
};

__device__ __forceinline__ FSel fsel_of(const MsFields& f, int n) { return FSel{static_cast<unsigned>(f.sh[n]), f.mask[n], f.word[n] != 0}; }

template <int W>
__device__ __forceinline__ unsigned ms_field(const Key<W>& k, const FSel& f) {
  const uint64_t w = (W == 1 || !f.hi) ? k.w[0] : k.w[W - 1];
  return static_cast<unsigned>(w >> f.sh) & f.mask;
}

// One gathered input of the mode-stream kernel: a factor (nb < 0) or, for a
// pair of input modes (na, nb), the row-wise product table of their factors
// with row ia * db + ib (alto_krp_pair), so one gather serves both modes.
struct VIn {
  const void* tab;
  int na, nb;
  unsigned db;
};

struct MStream {
  const uint64_t* keys;  // (ntiles*T, W) stream keys (MsFields layout), hot flag in bit 64W-1
  const void* vals;      // (ntiles*T,) values
  int tile;              // T (multiple of 128)
  MsFields f;
  int rr;                // round-robin slices: group s takes sorted positions s, s+8, ...
  VIn vin[ALTO_MAX_ORDER];  // gathered inputs when input modes are paired (P.n_pairs > 0)
  const int* base;       // delta stream: row of every lane group's first element (ntiles x 8)
};

// L2P: factor rows are gathered with a per-table L2 range policy (the
// table's first l2_hot bytes evict_last, the rest evict_first) and output
// rows merged with evict_first (alto_mttkrp_args.l2_hot_bytes).
template <int W, typename V, typename O, int N, int R, int MINB = 3, int U = 4, int NV = N - 1, bool DELTA = false,
          bool L2P = false>
__global__ void __launch_bounds__(kTileThreads, MINB)
mstream_kernel(const __grid_constant__ DevLayout L, const __grid_constant__ MStream S,
               const __grid_constant__ StreamParams P) {
  using F = V;
  using A = V;
  constexpr int G = R / 4;          // lanes per element
  constexpr int GPW = 32 / G;       // slices processed at once by a warp
  constexpr int PASSES = kMsSlices / GPW;
  constexpr int NIN = NV;            // gathered inputs (N-1, or fewer with paired modes)
  constexpr bool PAIR = NV < N - 1;
  constexpr unsigned ROWB = static_cast<unsigned>(R * sizeof(F));
  constexpr unsigned HOTF = 0x80000000u;
  static_assert(U >= 1 && U <= G, "one decoding lane per element of a block");
  constexpr int VW = static_cast<int>(sizeof(V) / 4);
  constexpr int NWREC = (NIN + 1 + VW + 3) & ~3;  // record words (16-byte multiple)
  const int mode = P.mode;
  const int T = S.tile;
  const int CH = T / kMsSlices;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane / G;
  const int gl = lane % G;
  const unsigned qmask = (G >= 4) ? (0xFu << (lane & ~3)) : 0xffffffffu;
  const char* fin_lane[NIN];
  FSel fin[NIN];
  FSel finb[PAIR ? NIN : 1];
  unsigned vdb[PAIR ? NIN : 1];
#pragma unroll
  for (int k = 0; k < NIN; ++k) {
    if constexpr (PAIR) {
      const VIn& vi = S.vin[k];
      fin_lane[k] = reinterpret_cast<const char*>(static_cast<const F*>(vi.tab) + 4 * gl);
      fin[k] = fsel_of(S.f, vi.na);
      finb[k] = vi.nb >= 0 ? fsel_of(S.f, vi.nb) : FSel{0u, 0u, false};  // empty field reads 0
      vdb[k] = vi.nb >= 0 ? vi.db : 1u;
    } else {
      const int n = k < mode ? k : k + 1;
      fin_lane[k] = reinterpret_cast<const char*>(static_cast<const F*>(P.factors[n]) + 4 * gl);
      fin[k] = fsel_of(S.f, n);
    }
  }
  // byte offset of input k's gathered row for key kk
  auto voff = [&](const Key<W>& kk, int k) -> unsigned {
    if constexpr (PAIR)
      return (ms_field<W>(kk, fin[k]) * vdb[k] + ms_field<W>(kk, finb[k])) * ROWB;
    else
      return ms_field<W>(kk, fin[k]) * ROWB;
  };
  const FSel fout = fsel_of(S.f, mode);
  const V* __restrict__ vals = static_cast<const V*>(S.vals);
  O* __restrict__ out = static_cast<O*>(P.out);
  const double fixed_scale = P.fixed_scale ? *P.fixed_scale : 1.0;
  // hot plan of the mode stream (alto_hot_copies): hot_code[row] = (first copy
  // << 5) | log2(copies); each hot row has its own power-of-two number of
  // replicated partial rows, sized so that no copy receives more than a
  // bounded number of merges (contention and float32 rounding stay bounded)
  const int* __restrict__ hot_code = P.n_hot > 0 ? P.hot_slot : nullptr;
  O* __restrict__ hot_buf = static_cast<O*>(P.hot_buf);
  const unsigned hotmask = hot_code ? HOTF : 0u;  // stream flags are ignored without a hot plan
  const unsigned long long pol = stream_policy(!(P.flags & ALTO_STREAM_MS_L2_NORMAL));
  unsigned long long gpol[L2P ? NIN : 1];
  if constexpr (L2P) {
    static_assert(!PAIR && sizeof(F) == 4 && std::is_same<O, float>::value, "L2 policies: unpaired float32 kernels");
#pragma unroll
    for (int k = 0; k < NIN; ++k) {
      const int n = k < mode ? k : k + 1;
      gpol[k] = range_policy(P.factors[n], P.l2_hot[n], P.l2_tab[n]);
    }
  }

  const long long ntiles = (P.m + T - 1) / T;
  const long long gw0 = static_cast<long long>(blockIdx.x) * (kTileThreads / 32) + warp;
  const long long nwarps = static_cast<long long>(gridDim.x) * (kTileThreads / 32);
  for (long long t = gw0; t < ntiles; t += nwarps) {
    const long long tb = t * T;
    const int cnt = static_cast<int>(min(static_cast<long long>(T), P.m - tb));
#pragma unroll 1
    for (int pass = 0; pass < PASSES; ++pass) {
      const int s = pass * GPW + grp;
      const int len = S.rr ? max(0, (cnt - s + kMsSlices - 1) / kMsSlices) : max(0, min(CH, cnt - s * CH));
      const uint64_t* kp = S.keys + (tb + s) * W;
      const V* vp = vals + tb + s;
      A acc[4] = {A(0), A(0), A(0), A(0)};
      unsigned cur = 0xffffffffu;  // no run yet (never a valid target: rows < 2^31)
      auto flush = [&]() {
        O* base;
        if (cur & HOTF) {
          // hot row: copy (tile mod copies) of the row's replicated partials
          const int hc = __ldg(hot_code + (cur & ~HOTF));
          base = hot_buf + (static_cast<long long>(hc >> 5) + (static_cast<unsigned>(t) & ((1u << (hc & 31)) - 1u))) * R;
        } else {
          base = out + static_cast<long long>(cur) * R;
        }
        if constexpr (L2P)
          red_f32x4_pol(reinterpret_cast<float*>(base) + 4 * gl, acc, pol);  // output rows pass through the L2
        else
          merge_row<O, A, G, R>(base, acc, gl, qmask, lane, fixed_scale);
      };
      // loop trip count is uniform across the warp's groups except in the
      // final partial tile; inactive groups keep their lanes converged
      const int jmax = __reduce_max_sync(0xffffffffu, len);
      // consume one decoded element (gathered rows g, value v, target t)
      auto consume = [&](unsigned t, V v, const V4<F> (&gg)[NIN]) {
        A tv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) tv[q] = static_cast<A>(v) * static_cast<A>(gg[0].v[q]);
#pragma unroll
        for (int k = 1; k < NIN - 1; ++k)
#pragma unroll
          for (int q = 0; q < 4; ++q) tv[q] *= static_cast<A>(gg[k].v[q]);
        if (t == cur) {
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[q] = fma(tv[q], static_cast<A>(gg[NIN - 1].v[q]), acc[q]);
        } else {
          if (cur != 0xffffffffu) flush();
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[q] = tv[q] * static_cast<A>(gg[NIN - 1].v[q]);
          cur = t;
        }
      };
      auto target = [&](const Key<W>& k) {
        return ms_field<W>(k, fout) | (static_cast<unsigned>(k.w[W - 1] >> 32) & hotmask);
      };
      {
        // Cooperative decode: lane gl < U of a group loads and decodes element
        // j0+gl of the group's slice; the U decoded records {input row byte
        // offsets, target, value} are broadcast within the group by shuffles.
        Key<W> nk{};
        V nv = V(0);
        auto prefetch = [&](int jb) {
          const int j = jb + gl;
          if (gl < U && j < len) {
            nk = load_key_stream<W>(kp, static_cast<long long>(j) * kMsSlices, pol);
            nv = load_val_stream<V>(vp + static_cast<long long>(j) * kMsSlices, pol);
          }
        };
        prefetch(0);
        const int gbase = lane & ~(G - 1);
        // delta stream: running row of the group (its first element's row)
        unsigned carry = 0;
        if constexpr (DELTA) carry = len > 0 ? static_cast<unsigned>(__ldg(S.base + t * kMsSlices + s)) : 0u;
#pragma unroll 1
        for (int j0 = 0; j0 < jmax; j0 += U) {
          const Key<W> kk = nk;
          const V vv = nv;
          prefetch(j0 + U);
          unsigned moff[NIN];
#pragma unroll
          for (int k = 0; k < NIN; ++k) moff[k] = voff(kk, k);
          unsigned mtg;
          if constexpr (DELTA) {
            // rows = carry + inclusive prefix of the U decoded increments (lanes gl < U)
            const bool ok = gl < U && j0 + gl < len;
            unsigned dlt = ok ? ms_field<W>(kk, fout) : 0u;
#pragma unroll
            for (int o = 1; o < U; o <<= 1) {
              const unsigned y = __shfl_up_sync(0xffffffffu, dlt, o, G);
              if (gl >= o) dlt += y;
            }
            const unsigned row = carry + dlt;
            carry = __shfl_sync(0xffffffffu, row, gbase + U - 1);
            mtg = ok ? (row | (static_cast<unsigned>(kk.w[W - 1] >> 32) & hotmask)) : 0xffffffffu;
          } else {
            mtg = (gl < U && j0 + gl < len) ? target(kk) : 0xffffffffu;
          }
          V4<F> g[U][NIN];
          unsigned tg[U];
          V vu[U];
          {
#pragma unroll
            for (int u = 0; u < U; ++u) {
              tg[u] = __shfl_sync(0xffffffffu, mtg, gbase + u);
              vu[u] = __shfl_sync(0xffffffffu, vv, gbase + u);
#pragma unroll
              for (int k = 0; k < NIN; ++k) {
                const unsigned off = __shfl_sync(0xffffffffu, moff[k], gbase + u);
                if (tg[u] != 0xffffffffu) {
                  if constexpr (L2P)
                    g[u][k] = gather_off_pol(fin_lane[k], off, gpol[k]);
                  else
                    g[u][k] = gather_off<F>(fin_lane[k], off);
                }
              }
            }
          }
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (tg[u] != 0xffffffffu) consume(tg[u], vu[u], g[u]);
        }
      }
      if (cur != 0xffffffffu) flush();
    }
  }
}

// Stream loads of NB bytes (16-byte pieces) that all lanes of a group issue
// on the same address (one broadcast request for the warp's GPW groups).
template <int NB>
__device__ __forceinline__ void load_stream_bytes(unsigned (&dst)[NB / 4], const void* p, unsigned long long pol) {
  static_assert(NB == 4 || NB == 8 || NB % 16 == 0, "4, 8 or a multiple of 16 bytes");
  if constexpr (NB == 4) {
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(dst[0]) : "l"(p), "l"(pol));
  } else if constexpr (NB == 8) {
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0, %1}, [%2], %3;"
        : "=r"(dst[0]), "=r"(dst[1])
        : "l"(p), "l"(pol));
  } else {
#pragma unroll
    for (int i = 0; i < NB / 16; ++i)
      asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
          : "=r"(dst[4 * i]), "=r"(dst[4 * i + 1]), "=r"(dst[4 * i + 2]), "=r"(dst[4 * i + 3])
          : "l"(static_cast<const char*>(p) + 16 * i), "l"(pol));
  }
}

// Field selectors of the blocked kernel's gathered inputs, resolved on the
// host in gather order so the kernel reads them from the parameter bank with
// compile-time indices (a selector indexed by `mode` at run time costs
// SEL/LEA/LDC per field per element once registers are short).
struct MsSel {
  unsigned sh, mask, hi;  // hi: field lives in the key's last word
};
struct MsBlk {
  MsSel in[ALTO_MAX_ORDER];   // gathered input k: row field (pairs: the a field)
  MsSel inb[ALTO_MAX_ORDER];  //   pairs: the b field (mask 0 when unpaired)
  unsigned vdb[ALTO_MAX_ORDER];  // pairs: I_b (1 when unpaired)
  const void* tab[ALTO_MAX_ORDER];  // factor or product table of input k
  MsSel out;                  // output row (or row increment) field
};

template <int W>
__device__ __forceinline__ unsigned ms_sel(const Key<W>& k, const MsSel& f) {
  if constexpr (W == 1) {
    return static_cast<unsigned>(k.w[0] >> f.sh) & f.mask;
  } else {
    const uint64_t w = f.hi ? k.w[W - 1] : k.w[0];
    return static_cast<unsigned>(w >> f.sh) & f.mask;
  }
}

// Blocked mode-stream kernel (ALTO_MS_BLOCKED).  A warp step covers B = GPW*U
// consecutive sorted elements; lane group s takes elements s, s+GPW, ... of
// the step (round robin: the GPW elements of one gather instruction are
// consecutive, so their ALTO-ordered input rows share lines) and the stream
// stores those U elements contiguously (element u*GPW+s of a step at s*U+u).
// Every lane of a group reads the group's U keys and U values itself with
// 16-byte accesses on group-uniform addresses (broadcast) and decodes them
// redundantly, so no shuffle is left in the element loop (the cooperative
// decode above spends 19 shuffles per 32 elements, ~20 % of the load/store
// pipe's wavefronts on cfg5).  Delta streams: the increment is taken from the
// group's previous element (GPW positions earlier); base[tile * GPW + s]
// holds the row of the group's first element.
// The next step's keys and values are prefetched into registers.  Measured
// (profiles/r02e_ab_blocked.jsonl): faster than the cooperative kernel at
// rank 32 (cfg3 2.64-2.77 -> 2.32-2.38 ms per mode) and for orders 4-5 (cfg4
// 0.265 -> 0.239 ms), slower at order 3 / rank 16 (cfg2 0.46 -> 0.50 ms:
// a broadcast 16-byte load still costs 4 data-pipe wavefronts, 512 bytes of
// register writeback, so the load/store pipe total does not drop there while
// the redundant decode adds instructions) — the host picks per shape.  A
// variant staging the stream through shared memory with cp.async (no
// prefetch registers) was slower everywhere (cfg2 0.53, cfg3 3.0-3.4 ms), and
// 2 instead of 4 elements per group for the paired order-5 shape (62-72
// registers, no spill, also at 4 CTAs/SM) ran cfg4 at 0.259-0.280 vs 0.240.
template <int W, typename V, typename O, int N, int R, int MINB, int U, int NV, bool DELTA>
__global__ void __launch_bounds__(kTileThreads, MINB)
mstream_blk_kernel(const __grid_constant__ MStream S, const __grid_constant__ MsBlk Q,
                   const __grid_constant__ StreamParams P) {
  using F = V;
  using A = V;
  constexpr int G = R / 4;
  constexpr int GPW = 32 / G;
  constexpr int B = GPW * U;
  constexpr int NIN = NV;
  constexpr bool PAIR = NV < N - 1;
  constexpr unsigned ROWB = static_cast<unsigned>(R * sizeof(F));
  constexpr unsigned HOTF = 0x80000000u;
  constexpr int KB = U * W * 8;                           // key bytes of a group per step
  constexpr int VB = U * static_cast<int>(sizeof(V));     // value bytes of a group per step
  constexpr int KSTEP = B * W * 8;                        // key bytes of a warp step
  constexpr int VSTEP = B * static_cast<int>(sizeof(V));  // value bytes of a warp step
  const int T = S.tile;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane / G;
  const int gl = lane % G;
  const unsigned qmask = (G >= 4) ? (0xFu << (lane & ~3)) : 0xffffffffu;
  // byte offset of input k's gathered row for key kk
  auto voff = [&](const Key<W>& kk, int k) -> unsigned {
    if constexpr (PAIR)
      return (ms_sel<W>(kk, Q.in[k]) * Q.vdb[k] + ms_sel<W>(kk, Q.inb[k])) * ROWB;
    else
      return ms_sel<W>(kk, Q.in[k]) * ROWB;
  };
  O* __restrict__ out = static_cast<O*>(P.out);
  const double fixed_scale = P.fixed_scale ? *P.fixed_scale : 1.0;
  const int* __restrict__ hot_code = P.n_hot > 0 ? P.hot_slot : nullptr;
  O* __restrict__ hot_buf = static_cast<O*>(P.hot_buf);
  const unsigned hotmask = hot_code ? HOTF : 0u;
  const unsigned long long pol = stream_policy(!(P.flags & ALTO_STREAM_MS_L2_NORMAL));

  const long long ntiles = (P.m + T - 1) / T;
  const long long gw0 = static_cast<long long>(blockIdx.x) * (kTileThreads / 32) + warp;
  const long long nwarps = static_cast<long long>(gridDim.x) * (kTileThreads / 32);
  if (gw0 >= ntiles) return;
  unsigned next_base = 0;
  if constexpr (DELTA) next_base = static_cast<unsigned>(__ldg(S.base + gw0 * GPW + grp));
  for (long long t = gw0; t < ntiles; t += nwarps) {
    const long long tb = t * T;
    const int cnt = static_cast<int>(min(static_cast<long long>(T), P.m - tb));
    A acc[4] = {A(0), A(0), A(0), A(0)};
    unsigned cur = 0xffffffffu;
    auto flush = [&]() {
      O* base;
      if (cur & HOTF) {
        const int hc = __ldg(hot_code + (cur & ~HOTF));
        base = hot_buf + (static_cast<long long>(hc >> 5) + (static_cast<unsigned>(t) & ((1u << (hc & 31)) - 1u))) * R;
      } else {
        base = out + static_cast<long long>(cur) * R;
      }
      merge_row<O, A, G, R>(base, acc, gl, qmask, lane, fixed_scale);
    };
    auto consume = [&](unsigned tgt, V v, const V4<F> (&gg)[NIN]) {
      A tv[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) tv[q] = static_cast<A>(v) * static_cast<A>(gg[0].v[q]);
#pragma unroll
      for (int k = 1; k < NIN - 1; ++k)
#pragma unroll
        for (int q = 0; q < 4; ++q) tv[q] *= static_cast<A>(gg[k].v[q]);
      if (tgt == cur) {
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[q] = fma(tv[q], static_cast<A>(gg[NIN - 1].v[q]), acc[q]);
      } else {
        if (cur != 0xffffffffu) flush();
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[q] = tv[q] * static_cast<A>(gg[NIN - 1].v[q]);
        cur = tgt;
      }
    };
    unsigned carry = 0;
    if constexpr (DELTA) {
      carry = next_base;
      if (t + nwarps < ntiles) next_base = static_cast<unsigned>(__ldg(S.base + (t + nwarps) * GPW + grp));
    }
    const char* kp = reinterpret_cast<const char*>(S.keys) + (tb + grp * U) * (W * 8);
    const char* vp = static_cast<const char*>(S.vals) + (tb + grp * U) * static_cast<long long>(sizeof(V));
    unsigned nkw[KB / 4], nvw[VB / 4];  // next step's keys / values
    load_stream_bytes<KB>(nkw, kp, pol);
    load_stream_bytes<VB>(nvw, vp, pol);
    const int nsteps = (cnt + B - 1) / B;
#pragma unroll 1
    for (int jb = 0; jb < nsteps; ++jb) {
      unsigned kw[KB / 4], vw[VB / 4];  // keys / values of the step being consumed
#pragma unroll
      for (int i = 0; i < KB / 4; ++i) kw[i] = nkw[i];
#pragma unroll
      for (int i = 0; i < VB / 4; ++i) vw[i] = nvw[i];
      if (jb + 1 < nsteps) {
        load_stream_bytes<KB>(nkw, kp + static_cast<long long>(jb + 1) * KSTEP, pol);
        load_stream_bytes<VB>(nvw, vp + static_cast<long long>(jb + 1) * VSTEP, pol);
      }
      const int e0 = jb * B + grp;  // sorted position of the group's first element of the step
      unsigned tg[U];
      V4<F> g[U][NIN];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        Key<W> kk;
#pragma unroll
        for (int w = 0; w < W; ++w)
          kk.w[w] = (static_cast<uint64_t>(kw[(u * W + w) * 2 + 1]) << 32) | kw[(u * W + w) * 2];
        const bool ok = e0 + u * GPW < cnt;
        unsigned row;
        if constexpr (DELTA) {
          carry += ok ? ms_sel<W>(kk, Q.out) : 0u;
          row = carry;
        } else {
          row = ms_sel<W>(kk, Q.out);
        }
        tg[u] = ok ? (row | (kw[(u * W + W - 1) * 2 + 1] & hotmask)) : 0xffffffffu;
        if (ok) {
#pragma unroll
          for (int k = 0; k < NIN; ++k)
            g[u][k] = gather_off<F>(static_cast<const char*>(Q.tab[k]) + 4 * sizeof(F) * gl, voff(kk, k));
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (tg[u] != 0xffffffffu) {
          V v;
          if constexpr (sizeof(V) == 4)
            v = __uint_as_float(vw[u]);
          else
            v = __hiloint2double(static_cast<int>(vw[2 * u + 1]), static_cast<int>(vw[2 * u]));
          consume(tg[u], v, g[u]);
        }
    }
    if (cur != 0xffffffffu) flush();
  }
}

// Elements in flight per group: ~UREG registers of gathered factor data per
// lane, at most one decoding lane per element (U <= G).
template <int N, int R, typename V, int UREG>
constexpr int ms_u() {
  constexpr int ub = std::max(1, UREG / ((N - 1) * 4 * static_cast<int>(sizeof(V) / 4)));
  return std::min(R / 4, ub);
}

template <int W, typename V, typename O, int N, int R, int MINB = 3, int U = ms_u<N, R, V, 32>(), int NV = N - 1,
          bool DELTA = false, bool L2P = false>
int launch_mstream(const DevLayout& d, const MStream& S, const StreamParams& P, cudaStream_t s) {
  if constexpr (!L2P && N == 3 && R == 16 && NV == 2 && sizeof(V) == 4 && std::is_same<O, float>::value) {
    // L2 residency policies requested for an input factor (order 3, rank 16, float32)
    bool want = false;
    for (int n = 0; n < 3; ++n) want = want || (n != P.mode && P.l2_hot[n] > 0);
    if (want && S.rr != 2) return launch_mstream<W, V, O, N, R, MINB, U, NV, DELTA, true>(d, S, P, s);
  }
  if (S.rr == 2) {
    // blocked stream (ALTO_MS_BLOCKED): broadcast vector loads, redundant decode, no shuffles
    // (float32 data only: alto_mstream_block reports no blocked kernel for float64)
    if constexpr (sizeof(V) != 4) {
      return ALTO_EUNSUPPORTED;
    } else {
    constexpr int GPW = 32 / (R / 4);
    if (S.tile % (GPW * U)) return ALTO_EUNSUPPORTED;
    MsBlk Q{};
    constexpr bool PAIR = NV < N - 1;
    for (int k = 0; k < NV; ++k) {
      int na, nb = -1;
      if (PAIR) {
        na = S.vin[k].na;
        nb = S.vin[k].nb;
        Q.tab[k] = S.vin[k].tab;
        Q.vdb[k] = nb >= 0 ? S.vin[k].db : 1u;
      } else {
        na = k < P.mode ? k : k + 1;
        Q.tab[k] = P.factors[na];
        Q.vdb[k] = 1u;
      }
      Q.in[k] = MsSel{static_cast<unsigned>(S.f.sh[na]), S.f.mask[na], S.f.word[na] != 0 ? 1u : 0u};
      Q.inb[k] = nb >= 0 ? MsSel{static_cast<unsigned>(S.f.sh[nb]), S.f.mask[nb], S.f.word[nb] != 0 ? 1u : 0u}
                         : MsSel{0u, 0u, 0u};
    }
    Q.out = MsSel{static_cast<unsigned>(S.f.sh[P.mode]), S.f.mask[P.mode], S.f.word[P.mode] != 0 ? 1u : 0u};
    auto kern = mstream_blk_kernel<W, V, O, N, R, MINB, U, NV, DELTA>;
    static int blk_bps = 0;
    if (!blk_bps) {
      int b = 1;
      ALTO_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, kTileThreads, 0));
      blk_bps = std::max(b, 1);
    }
    const long long ntiles = (P.m + S.tile - 1) / S.tile;
    const long long need = (ntiles + kTileThreads / 32 - 1) / (kTileThreads / 32);
    const long long grid = std::min<long long>(need, static_cast<long long>(device_sms()) * blk_bps);
    kern<<<static_cast<unsigned>(grid), kTileThreads, 0, s>>>(S, Q, P);
    ALTO_LAUNCH_CHECK("alto_mttkrp(blocked mode stream)");
    return ALTO_OK;
    }
  }
  auto kern = mstream_kernel<W, V, O, N, R, MINB, U, NV, DELTA, L2P>;
  static int cached_bps = 0;
  if (!cached_bps) {
    int b = 1;
    ALTO_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, kTileThreads, 0));
    cached_bps = std::max(b, 1);
  }
  const long long ntiles = (P.m + S.tile - 1) / S.tile;
  const long long need = (ntiles + kTileThreads / 32 - 1) / (kTileThreads / 32);
  const long long grid = std::min<long long>(need, static_cast<long long>(device_sms()) * cached_bps);
  kern<<<static_cast<unsigned>(grid), kTileThreads, 0, s>>>(d, S, P);
  ALTO_LAUNCH_CHECK("alto_mttkrp(mode stream)");
  return ALTO_OK;
}

// Dispatch of one stream layout (DELTA: one-word delta keys, W = 1).
template <int W, typename V, typename O, bool DELTA>
int mstream_dispatch(const DevLayout& d, MStream S, const StreamParams& P, cudaStream_t s) {
  if (P.n_pairs > 0) {
    // paired input modes (alto_krp_pair tables): float32 data, rank 16, orders 4-5
    if constexpr (sizeof(V) == 4 && !std::is_same<O, long long>::value) {
      if (P.rank != 16 || d.order < 4) return ALTO_EUNSUPPORTED;
      int nv = 0;
      unsigned used = 1u << P.mode;
      for (int i = 0; i < P.n_pairs; ++i) {
        const int a = P.pair_a[i], b = P.pair_b[i];
        if (a < 0 || b < 0 || a >= d.order || b >= d.order || a == b || ((used >> a) & 1u) || ((used >> b) & 1u) ||
            !P.pair_tab[i] || d.dims[a] * d.dims[b] * P.rank * static_cast<long long>(sizeof(V)) > 0xFFFFFFFFll)
          return ALTO_EUNSUPPORTED;
        used |= (1u << a) | (1u << b);
        S.vin[nv++] = VIn{P.pair_tab[i], a, b, static_cast<unsigned>(d.dims[b])};
      }
      for (int n = 0; n < d.order; ++n)
        if (!((used >> n) & 1u)) S.vin[nv++] = VIn{P.factors[n], n, -1, 1u};
      if (d.order == 4 && nv == 2)
        return launch_mstream<W, V, O, 4, 16, 3, ms_u<3, 16, V, 32>(), 2, DELTA>(d, S, P, s);
      if (d.order == 5 && nv == 3)
        return launch_mstream<W, V, O, 5, 16, 3, ms_u<4, 16, V, 32>(), 3, DELTA>(d, S, P, s);
      if (d.order == 5 && nv == 2)
        return launch_mstream<W, V, O, 5, 16, 3, ms_u<3, 16, V, 32>(), 2, DELTA>(d, S, P, s);
    }
    return ALTO_EUNSUPPORTED;
  }
  // (round 2, same kernel with raw key words + value shuffled, 3 per element instead of 4 decoded words plus
  // the increment scan, every lane decoding for itself: cfg2 0.476 vs 0.459, cfg5 6.4-7.0 vs 5.9-6.7 ms: dropped)
  // (measured and dropped on cfg2, ms/mode: broadcast key loads 0.70-0.72,
  // 4 CTAs/SM 0.64-0.68, a two-stage pipeline 0.65-0.88, a shared-memory
  // record exchange 0.66-0.68, raw-key shuffles 0.69-0.73 — against 0.45-0.46
  // for this cooperative-decode + shuffle kernel with round-robin groups)
  if (P.rank == 16) {
    if (d.order == 3) return launch_mstream<W, V, O, 3, 16, 3, ms_u<3, 16, V, 32>(), 2, DELTA>(d, S, P, s);
    if (d.order == 4) return launch_mstream<W, V, O, 4, 16, 3, ms_u<4, 16, V, 32>(), 3, DELTA>(d, S, P, s);
    if (d.order == 5) return launch_mstream<W, V, O, 5, 16, 3, ms_u<5, 16, V, 32>(), 4, DELTA>(d, S, P, s);
  }
  if (P.rank == 32) {
    if (d.order == 3) return launch_mstream<W, V, O, 3, 32, 3, ms_u<3, 32, V, 32>(), 2, DELTA>(d, S, P, s);
    if (d.order == 4) return launch_mstream<W, V, O, 4, 32, 3, ms_u<4, 32, V, 32>(), 3, DELTA>(d, S, P, s);
    if (d.order == 5) return launch_mstream<W, V, O, 5, 32, 3, ms_u<5, 32, V, 32>(), 4, DELTA>(d, S, P, s);
  }
  return ALTO_EUNSUPPORTED;
}

// Returns ALTO_EUNSUPPORTED (without launching) when the shape is not covered.
template <int W, typename V, typename O>
int try_mstream(const DevLayout& d, const StreamParams& P, cudaStream_t s) {
  if (!P.mkeys || !P.mvals || P.mtile <= 0) return ALTO_EUNSUPPORTED;
  long long maxdim = 0;
  for (int n = 0; n < d.order; ++n) maxdim = std::max(maxdim, d.dims[n]);
  if (maxdim * P.rank * static_cast<long long>(sizeof(V)) > 0xFFFFFFFFll) return ALTO_EUNSUPPORTED;
  for (int n = 0; n < d.order; ++n)
    if (d.bits[n] > 31) return ALTO_EUNSUPPORTED;
  if (P.mbase) {
    // delta stream: one key word whatever the layout width (ALTO_MS_DELTA)
    if constexpr (W != 1) {
      return try_mstream<1, V, O>(d, P, s);
    } else {
      const MStream S{P.mkeys, P.mvals, P.mtile, ms_fields_delta(d, P.mode), P.mrr, {}, P.mbase};
      if (!S.f.ok) return ALTO_EUNSUPPORTED;
      return mstream_dispatch<1, V, O, true>(d, S, P, s);
    }
  }
  const MStream S{P.mkeys, P.mvals, P.mtile, ms_fields(d, P.mode), P.mrr, {}, nullptr};
  if (!S.f.ok) return ALTO_EUNSUPPORTED;
  return mstream_dispatch<W, V, O, false>(d, S, P, s);
}

// out[row(s)] += sum of the row's copies (float64, fixed order), copies re-zeroed.
// One warp per hot row; lane (j, r): rank r of copies j, j + 32/R, ... with
// 8 independent accumulators (copy j + (8q + a)·32/R goes to accumulator a),
// then a fixed-order combine across accumulators and lanes.
template <typename O>
__global__ void __launch_bounds__(256) hot_reduce_rows_kernel(O* __restrict__ buf, const int* __restrict__ hot_rows,
                                                              const int* __restrict__ hot_base, int n_hot, int R,
                                                              O* __restrict__ out) {
  using S = typename std::conditional<std::is_same<O, long long>::value, long long, double>::type;
  const int slot = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (slot >= n_hot) return;
  const int lane = threadIdx.x & 31;
  if (R > 32 || (R & (R - 1)) != 0) {
    // generic kernel's ranks (above 32, or not a power of two): lane r, r+32, ... sums its rank over the
    // copies in order
    for (int r = lane; r < R; r += 32) {
      S acc = S(0);
      for (int k = hot_base[slot]; k < hot_base[slot + 1]; ++k) {
        O* p = buf + static_cast<long long>(k) * R + r;
        acc += static_cast<S>(*p);
        *p = O(0);
      }
      O* o = out + static_cast<long long>(hot_rows[slot]) * R + r;
      *o = static_cast<O>(static_cast<S>(*o) + acc);
    }
    return;
  }
  const int per = R >= 32 ? 1 : 32 / R;
  const int r = lane % R, j = lane / R;
  const bool active = R >= 32 ? (lane < R) : (j < per);
  const int b0 = hot_base[slot], b1 = hot_base[slot + 1];
  constexpr int NA = 8;  // independent accumulators = loads in flight per lane
  S acc[NA];
#pragma unroll
  for (int q = 0; q < NA; ++q) acc[q] = S(0);
  if (active) {
    const long long st = static_cast<long long>(per) * R;
    int k = b0 + j;
    for (; k + (NA - 1) * per < b1; k += NA * per) {
      O* p = buf + static_cast<long long>(k) * R + r;
      O v[NA];
#pragma unroll
      for (int q = 0; q < NA; ++q) v[q] = p[q * st];
#pragma unroll
      for (int q = 0; q < NA; ++q) {
        acc[q] += static_cast<S>(v[q]);
        p[q * st] = O(0);
      }
    }
    for (int q = 0; k < b1; k += per, ++q) {
      O* p = buf + static_cast<long long>(k) * R + r;
      acc[q] += static_cast<S>(*p);
      *p = O(0);
    }
  }
  S t = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
  // lanes r, r+R, ... hold rank r: fold in a fixed order
  for (int o = 16; o >= R && o > 0; o >>= 1) {
    const S u = __shfl_down_sync(0xffffffffu, t, o);
    t += u;
  }
  if (lane < R) {
    O* o = out + static_cast<long long>(hot_rows[slot]) * R + lane;
    *o = static_cast<O>(static_cast<S>(*o) + t);
  }
}

}  // namespace alto
