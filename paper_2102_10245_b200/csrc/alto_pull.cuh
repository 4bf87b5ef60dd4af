// alto_pull.cuh — K8/K9: the paper's Buffered scheme (Alg. 2; reference
// pkg/src/altotensor/mttkrp.py:132-175) as slice interval buffers plus a
// deterministic pull reduction, and its Atomic scheme (mttkrp.py:178-224)
// with boundary flags resolved on the fly.
//
// Input: the mode's row-major stream (alto_mode_stream with ALTO_MS_ROW_MAJOR,
// contiguous slices): the ALTO elements stably sorted by the output-mode
// coordinate (ALTO order inside a row), cut into slices of CH = T/8
// consecutive sorted positions — slice g holds sorted positions [g*CH,
// (g+1)*CH) and its j-th element is stored at (g/8)*T + j*8 + g%8, so the
// j-th elements of 8 consecutive slices are one coalesced request.
//
// A slice is a partition in the reference's sense: its output interval
// [first row, last row] is contiguous (the stream is row-sorted), every row
// strictly inside it is touched by this slice only, and only its first and
// last row can be shared with the neighbouring slices — the paper's "overlap"
// rows, i.e. exactly the elements apply_boundary_flags (format.py:257-285)
// would flag, decided here from the neighbours' rows instead of a key bit.
//
// Stage (pull_stage_kernel): G = R/4 lanes own a slice (4 consecutive ranks
// per lane); lane gl < U of a group loads and decodes element j0+gl and the
// U records {input row offsets, target row, value} are broadcast in the
// group by shuffles; the N-1 factor rows are gathered as 16-byte vectors
// (float) / 2x16 bytes (double), multiplied, and accumulated in registers
// while the output row repeats, in element order.  At each row end:
//   * owned row       -> one plain vector store of the final row (no atomic);
//   * shared row      -> Buffered: the partial goes to the slice's record slot
//                        (per-slice interval buffer, only the overlap rows);
//                        Atomic: RED into the output (rows pre-zeroed);
//   * rows with no element between two runs (and before the first / after the
//     last element) are zero-filled by the slice that discovers the gap, so
//     every output row is written exactly once and no memset is needed
//     (Buffered).
// Pull (pull_chunk_kernel, pull_seg_kernel): each shared row's records are
// contiguous in slot order; they are summed in float64 in slot (= element)
// order with a fixed two-level shape (chunks of kPullChunk records, then the
// chunk partials), so the result is bitwise reproducible and independent of
// scheduling, like the reference's ascending-partition pull (mttkrp.py:160-174).
#pragma once
#include "alto_mstream.cuh"

namespace alto {

constexpr int kPullChunk = 64;  // records per level-1 pull chunk

struct PullStage {
  const uint64_t* keys;   // mode stream keys (MsFields layout)
  const void* vals;       // mode stream values
  long long m;            // elements
  int tile;               // T (slices of T/8)
  int mode;
  long long dim;          // output rows
  MsFields f;
  const void* factors[ALTO_MAX_ORDER];
  void* out;              // (dim, R) O
  void* rec;              // (n_rec, R) A: shared-row partials (Buffered)
  const int2* slice_rec;  // (nslices) record slot of the slice's first / last run, -1 if owned
  const int2* slice_rows; // (nslices) first / last output row of every slice (alto_pull_slice_rows)
  VIn vin[ALTO_MAX_ORDER]; // gathered inputs when input modes are paired (alto_krp_pair tables), as in MStream
};

template <typename O, typename A>
__device__ __forceinline__ void store_row4(O* p, const A (&a)[4]) {
  if constexpr (sizeof(O) == 4) {
    *reinterpret_cast<float4*>(p) = make_float4(static_cast<float>(a[0]), static_cast<float>(a[1]),
                                                static_cast<float>(a[2]), static_cast<float>(a[3]));
  } else {
    reinterpret_cast<double2*>(p)[0] = make_double2(static_cast<double>(a[0]), static_cast<double>(a[1]));
    reinterpret_cast<double2*>(p)[1] = make_double2(static_cast<double>(a[2]), static_cast<double>(a[3]));
  }
}

template <typename O>
__device__ __forceinline__ void zero_row4(O* p) {
  if constexpr (sizeof(O) == 4) {
    *reinterpret_cast<float4*>(p) = make_float4(0.f, 0.f, 0.f, 0.f);
  } else {
    reinterpret_cast<double2*>(p)[0] = make_double2(0.0, 0.0);
    reinterpret_cast<double2*>(p)[1] = make_double2(0.0, 0.0);
  }
}

template <typename O, typename A>
__device__ __forceinline__ void red_row4(O* p, const A (&a)[4]) {
  if constexpr (sizeof(O) == 4) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(static_cast<float>(a[0])),
                 "f"(static_cast<float>(a[1])), "f"(static_cast<float>(a[2])), "f"(static_cast<float>(a[3]))
                 : "memory");
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q) atomicAdd(reinterpret_cast<double*>(p) + q, static_cast<double>(a[q]));
  }
}

// V: stored value type, F: factor type (= accumulation type A), O: output.
// DELTA: one-word delta stream keys (ALTO_MS_DELTA): the output field holds the
// row increment from the previous element of the slice; the slice's first row
// comes from slice_rows.
// NV < N - 1: paired input modes — one gather from a row-wise product table
// replaces two (S.vin, float32 factors, rank 16, orders 4-5).
template <int W, typename V, typename F, typename O, int N, int R, int U, bool ATOMIC, bool DELTA = false,
          int NV = N - 1>
__global__ void __launch_bounds__(256, (sizeof(F) == 4 ? 3 : 2))
pull_stage_kernel(const __grid_constant__ PullStage S) {
  using A = F;
  constexpr int G = R / 4;     // lanes per slice
  constexpr int GPW = 32 / G;  // slices per warp
  constexpr int NIN = NV;
  constexpr bool PAIR = NV < N - 1;
  constexpr unsigned ROWB = static_cast<unsigned>(R * sizeof(F));
  static_assert(R % 4 == 0 && G >= 1 && G <= 32 && 32 % G == 0, "rank must be 4 * a power of two <= 128");
  static_assert(U >= 1 && U <= G, "one decoding lane per element of a block");
  const int T = S.tile;
  const int CH = T >> 3;
  const int lane = threadIdx.x & 31;
  const int grp = lane / G, gl = lane % G;
  const int gbase = lane & ~(G - 1);
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
      const int n = k < S.mode ? k : k + 1;
      fin_lane[k] = reinterpret_cast<const char*>(static_cast<const F*>(S.factors[n]) + 4 * gl);
      fin[k] = fsel_of(S.f, n);
    }
  }
  const FSel fout = fsel_of(S.f, S.mode);
  const V* __restrict__ vals = static_cast<const V*>(S.vals);
  O* __restrict__ out = static_cast<O*>(S.out) + 4 * gl;
  A* __restrict__ rec = static_cast<A*>(S.rec) + 4 * gl;
  const unsigned long long pol = stream_policy(true);
  const long long nslices = (S.m + CH - 1) / CH;
  const long long nblocks = (nslices + GPW - 1) / GPW;
  const long long w0 = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long long nw = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
  for (long long sb = w0; sb < nblocks; sb += nw) {
    const long long g = sb * GPW + grp;
    const long long q0 = g * CH;
    const int len = g < nslices ? static_cast<int>(min(static_cast<long long>(CH), S.m - q0)) : 0;
    const long long sbase = (g >> 3) * T + (g & 7);  // storage index of element 0 of slice g
    // neighbours' rows: the last element of slice g-1 and the first of g+1
    // (rows < 2^31; -1 = none)
    int prev_row = -1, next_row = -1;
    unsigned carry = 0;  // DELTA: running row of the slice
    int2 slots = make_int2(-1, -1);
    if (len > 0) {
      if (q0 > 0) prev_row = __ldg(S.slice_rows + g - 1).y;
      if (q0 + len < S.m) next_row = __ldg(S.slice_rows + g + 1).x;
      if constexpr (DELTA) carry = static_cast<unsigned>(__ldg(S.slice_rows + g).x);
      if constexpr (!ATOMIC) slots = __ldg(S.slice_rec + g);
    }
    int lw = prev_row;  // last output row written by or before this slice
    A acc[4] = {A(0), A(0), A(0), A(0)};
    int cur = -1;
    bool first_run = true;
    auto flush = [&](bool last_run) {
      const int r = cur;
      for (int z = lw + 1; z < r; ++z) zero_row4<O>(out + static_cast<long long>(z) * R);  // empty rows of the gap
      lw = r;
      const bool sh_first = first_run && r == prev_row;
      const bool sh_last = last_run && r == next_row;
      if (sh_first || sh_last) {
        if constexpr (ATOMIC) {
          red_row4<O, A>(out + static_cast<long long>(r) * R, acc);
        } else {
          const int slot = sh_first ? slots.x : slots.y;
          store_row4<A, A>(rec + static_cast<long long>(slot) * R, acc);
        }
      } else {
        store_row4<O, A>(out + static_cast<long long>(r) * R, acc);
      }
      first_run = false;
    };
    auto consume = [&](int t, A v, const V4<F> (&gg)[NIN]) {
      A tv[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) tv[q] = v * gg[0].v[q];
#pragma unroll
      for (int k = 1; k < NIN - 1; ++k)
#pragma unroll
        for (int q = 0; q < 4; ++q) tv[q] *= gg[k].v[q];
      if (t == cur) {
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[q] = fma(tv[q], gg[NIN - 1].v[q], acc[q]);
      } else {
        if (cur >= 0) flush(false);
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[q] = tv[q] * gg[NIN - 1].v[q];
        cur = t;
      }
    };
    const int jmax = __reduce_max_sync(0xffffffffu, len);
    Key<W> nk{};
    V nv = V(0);
    auto prefetch = [&](int jb) {
      const int j = jb + gl;
      if (gl < U && j < len) {
        nk = load_key_stream<W>(S.keys, sbase + static_cast<long long>(j) * 8, pol);
        nv = load_val_stream<V>(vals + sbase + static_cast<long long>(j) * 8, pol);
      }
    };
    prefetch(0);
#pragma unroll 1
    for (int j0 = 0; j0 < jmax; j0 += U) {
      const Key<W> kk = nk;
      const V vv = nv;
      prefetch(j0 + U);
      unsigned mrow[NIN];
#pragma unroll
      for (int k = 0; k < NIN; ++k) {
        if constexpr (PAIR)
          mrow[k] = ms_field<W>(kk, fin[k]) * vdb[k] + ms_field<W>(kk, finb[k]);
        else
          mrow[k] = ms_field<W>(kk, fin[k]);
      }
      int mtg;
      if constexpr (DELTA) {
        // rows = carry + inclusive prefix of the U decoded increments
        const bool ok = gl < U && j0 + gl < len;
        unsigned dlt = ok ? ms_field<W>(kk, fout) : 0u;
#pragma unroll
        for (int o = 1; o < U; o <<= 1) {
          const unsigned y = __shfl_up_sync(0xffffffffu, dlt, o, G);
          if (gl >= o) dlt += y;
        }
        const unsigned row = carry + dlt;
        carry = __shfl_sync(0xffffffffu, row, gbase + U - 1);
        mtg = ok ? static_cast<int>(row) : -1;
      } else {
        mtg = (gl < U && j0 + gl < len) ? static_cast<int>(ms_field<W>(kk, fout)) : -1;
      }
      V4<F> gv[U][NIN];
      int tg[U];
      A vu[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        tg[u] = __shfl_sync(0xffffffffu, mtg, gbase + u);
        vu[u] = static_cast<A>(__shfl_sync(0xffffffffu, vv, gbase + u));
#pragma unroll
        for (int k = 0; k < NIN; ++k) {
          const unsigned row = __shfl_sync(0xffffffffu, mrow[k], gbase + u);
          // 64-bit row address (one IMAD.WIDE.U32): factors may exceed 4 GB
          if (tg[u] >= 0) gv[u][k] = gather_off<F>(fin_lane[k] + static_cast<unsigned long long>(row) * ROWB, 0u);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (tg[u] >= 0) consume(tg[u], vu[u], gv[u]);
    }
    if (cur >= 0) flush(true);
    if (len > 0 && q0 + len == S.m)  // the last slice: rows after the last element
      for (long long z = static_cast<long long>(lw) + 1; z < S.dim; ++z) zero_row4<O>(out + z * R);
  }
}

// Level 1 of the pull: chunk c = records [chunk_off[c], chunk_off[c+1]) of
// segment chunk_seg[c] (one shared row).  A warp sums them in float64 in
// record order — lane L takes rank L % R of records k = L / R (mod P),
// P = 32 / R interleaved accumulators combined in a fixed order — and
// writes the row (single-chunk segment) or the chunk partial.
template <typename A, typename O, int R>
__global__ void __launch_bounds__(256) pull_chunk_kernel(const A* __restrict__ rec, long long n_chunks,
                                                         const int64_t* __restrict__ chunk_off,
                                                         const int* __restrict__ chunk_seg,
                                                         const int64_t* __restrict__ seg_chunk_off,
                                                         const int* __restrict__ seg_row, O* __restrict__ out,
                                                         double* __restrict__ part) {
  constexpr int P = R >= 32 ? 1 : 32 / R;
  constexpr int E = R > 32 ? R / 32 : 1;  // ranks per lane
  const long long c = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (c >= n_chunks) return;
  const int lane = threadIdx.x & 31;
  const int r0 = R >= 32 ? lane : lane % R, k0 = R >= 32 ? 0 : lane / R;
  const long long b = chunk_off[c], e = chunk_off[c + 1];
  double acc[E];
#pragma unroll
  for (int i = 0; i < E; ++i) acc[i] = 0.0;
  for (long long k = b + k0; k < e; k += P)
#pragma unroll
    for (int i = 0; i < E; ++i) acc[i] += static_cast<double>(rec[k * R + r0 + 32 * i]);
  // fixed-order fold of the P interleaved accumulators (lanes r, r+R, ...)
#pragma unroll
  for (int i = 0; i < E; ++i)
    for (int o = 16; o >= R && o > 0; o >>= 1) acc[i] += __shfl_down_sync(0xffffffffu, acc[i], o);
  if (lane >= (R < 32 ? R : 32)) return;
  const int s = chunk_seg[c];
  const bool single = seg_chunk_off[s + 1] - seg_chunk_off[s] == 1;
#pragma unroll
  for (int i = 0; i < E; ++i) {
    if (single)
      out[static_cast<long long>(seg_row[s]) * R + r0 + 32 * i] = static_cast<O>(acc[i]);
    else
      part[c * R + r0 + 32 * i] = acc[i];
  }
}

// Level 2: segments with several chunks sum their chunk partials in order.
template <typename O, int R>
__global__ void __launch_bounds__(256) pull_seg_kernel(const double* __restrict__ part, long long n_mseg,
                                                       const int* __restrict__ mseg,
                                                       const int64_t* __restrict__ seg_chunk_off,
                                                       const int* __restrict__ seg_row, O* __restrict__ out) {
  constexpr int P = R >= 32 ? 1 : 32 / R;
  constexpr int E = R > 32 ? R / 32 : 1;
  const long long i = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (i >= n_mseg) return;
  const int lane = threadIdx.x & 31;
  const int r0 = R >= 32 ? lane : lane % R, k0 = R >= 32 ? 0 : lane / R;
  const int s = mseg[i];
  const long long b = seg_chunk_off[s], e = seg_chunk_off[s + 1];
  double acc[E];
#pragma unroll
  for (int q = 0; q < E; ++q) acc[q] = 0.0;
  for (long long k = b + k0; k < e; k += P)
#pragma unroll
    for (int q = 0; q < E; ++q) acc[q] += part[k * R + r0 + 32 * q];
#pragma unroll
  for (int q = 0; q < E; ++q)
    for (int o = 16; o >= R && o > 0; o >>= 1) acc[q] += __shfl_down_sync(0xffffffffu, acc[q], o);
  if (lane >= (R < 32 ? R : 32)) return;
#pragma unroll
  for (int q = 0; q < E; ++q) out[static_cast<long long>(seg_row[s]) * R + r0 + 32 * q] = static_cast<O>(acc[q]);
}

// Atomic scheme: the shared rows start from zero (the stage REDs into them).
template <typename O>
__global__ void zero_rows_kernel(const int* __restrict__ rows, long long n, int R, O* __restrict__ out) {
  const long long total = n * R;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total; i += stride) {
    const long long k = i / R;
    out[static_cast<long long>(rows[k]) * R + (i - k * R)] = O(0);
  }
}

// First and last output row of every slice (plan construction).  Delta
// streams (base != null): first = base[g], last = first + the slice's
// increments.
template <int W>
__global__ void pull_slice_rows_kernel(const uint64_t* __restrict__ keys, long long m, int tile, MsFields f, int mode,
                                       const int* __restrict__ base, int2* __restrict__ fl) {
  const int CH = tile >> 3;
  const long long ns = (m + CH - 1) / CH;
  const FSel fo = fsel_of(f, mode);
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long g = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; g < ns; g += stride) {
    const long long q0 = g * CH;
    const int len = static_cast<int>(min(static_cast<long long>(CH), m - q0));
    const long long sbase = (g >> 3) * tile + (g & 7);
    if (base) {
      unsigned r = static_cast<unsigned>(base[g]);
      const unsigned a = r;
      for (int j = 1; j < len; ++j) r += ms_field<W>(load_key<W>(keys, sbase + static_cast<long long>(j) * 8), fo);
      fl[g] = make_int2(static_cast<int>(a), static_cast<int>(r));
    } else {
      const unsigned a = ms_field<W>(load_key<W>(keys, sbase), fo);
      const unsigned z = ms_field<W>(load_key<W>(keys, sbase + static_cast<long long>(len - 1) * 8), fo);
      fl[g] = make_int2(static_cast<int>(a), static_cast<int>(z));
    }
  }
}

}  // namespace alto
