// alto_pull_impl.cuh — launch/dispatch of the K8/K9 pull engine (alto_pull.cuh),
// instantiated per key width in alto_pull_w1.cu / alto_pull_w2.cu.
#pragma once
#include <algorithm>

#include "alto_pull.cuh"

namespace alto {

// elements in flight per lane group: ~32 registers of gathered rows per lane
template <int N, int R, typename F>
constexpr int pull_u() {
  constexpr int ub = std::max(1, 32 / ((N - 1) * 4 * static_cast<int>(sizeof(F) / 4)));
  return std::min(R / 4, ub);
}

template <int W, typename V, typename F, typename O, int N, int R, bool AT, bool DELTA = false, int NV = N - 1>
int pull_launch(const alto_pull_args* a, const PullStage& S, cudaStream_t s) {
  using A = F;
  constexpr int U = pull_u<NV + 1, R, F>();
  auto kern = pull_stage_kernel<W, V, F, O, N, R, U, AT, DELTA, NV>;
  static int bps = 0;
  if (!bps) {
    int b = 1;
    ALTO_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, 256, 0));
    bps = std::max(b, 1);
  }
  if (AT && a->n_seg > 0) {
    zero_rows_kernel<O><<<grid_for(a->n_seg * R, 256), 256, 0, s>>>(a->seg_row, a->n_seg, R, static_cast<O*>(S.out));
    ALTO_LAUNCH_CHECK("alto_mttkrp_pull/zero_rows");
  }
  constexpr int GPW = 32 / (R / 4);
  const long long CH = S.tile / 8;
  const long long nslices = (S.m + CH - 1) / CH;
  const long long nwarps = (nslices + GPW - 1) / GPW;
  const long long grid = std::min<long long>((nwarps + 7) / 8, static_cast<long long>(kSMs) * bps);
  kern<<<static_cast<unsigned>(std::max<long long>(grid, 1)), 256, 0, s>>>(S);
  ALTO_LAUNCH_CHECK("alto_mttkrp_pull/stage");
  if (!AT && a->n_chunks > 0) {
    pull_chunk_kernel<A, O, R><<<static_cast<unsigned>((a->n_chunks + 7) / 8), 256, 0, s>>>(
        static_cast<const A*>(a->rec), a->n_chunks, a->chunk_off, a->chunk_seg, a->seg_chunk_off, a->seg_row,
        static_cast<O*>(S.out), a->part);
    ALTO_LAUNCH_CHECK("alto_mttkrp_pull/chunks");
    if (a->n_mseg > 0) {
      pull_seg_kernel<O, R><<<static_cast<unsigned>((a->n_mseg + 7) / 8), 256, 0, s>>>(
          a->part, a->n_mseg, a->mseg, a->seg_chunk_off, a->seg_row, static_cast<O*>(S.out));
      ALTO_LAUNCH_CHECK("alto_mttkrp_pull/segments");
    }
  }
  return ALTO_OK;
}

template <int W, typename V, typename F, typename O, bool AT, bool DELTA = false>
int pull_by_shape(const alto_pull_args* a, const PullStage& S, int order, cudaStream_t s) {
  const int R = a->rank;
  if (a->n_pairs > 0) {
    // paired input modes: float32 factors, rank 16, orders 4-5 (as the mode-stream kernel)
    if constexpr (sizeof(F) == 4 && sizeof(V) == 4) {
      if (R != 16) return ALTO_EUNSUPPORTED;
      if (order == 4 && a->n_pairs == 1) return pull_launch<W, V, F, O, 4, 16, AT, DELTA, 2>(a, S, s);
      if (order == 5 && a->n_pairs == 1) return pull_launch<W, V, F, O, 5, 16, AT, DELTA, 3>(a, S, s);
      if (order == 5 && a->n_pairs == 2) return pull_launch<W, V, F, O, 5, 16, AT, DELTA, 2>(a, S, s);
    }
    return ALTO_EUNSUPPORTED;
  }
#define ALTO_PULL_N(NN)                                                                  \
  if (order == NN) {                                                                     \
    if (R == 16) return pull_launch<W, V, F, O, NN, 16, AT, DELTA>(a, S, s);             \
    if (R == 32) return pull_launch<W, V, F, O, NN, 32, AT, DELTA>(a, S, s);             \
    if constexpr (sizeof(F) == 4 && sizeof(O) == 4 && !AT && !DELTA) {                   \
      if (R == 8) return pull_launch<W, V, F, O, NN, 8, AT>(a, S, s);                    \
      if (R == 64) return pull_launch<W, V, F, O, NN, 64, AT>(a, S, s);                  \
    }                                                                                    \
  }
  ALTO_PULL_N(3)
  ALTO_PULL_N(4)
  ALTO_PULL_N(5)
#undef ALTO_PULL_N
  return ALTO_EUNSUPPORTED;
}

template <int W, typename V, typename F, typename O>
int pull_by_atomic(const alto_pull_args* a, const PullStage& S, int order, cudaStream_t s) {
  return a->atomic ? pull_by_shape<W, V, F, O, true>(a, S, order, s) : pull_by_shape<W, V, F, O, false>(a, S, order, s);
}

// One-word delta streams (float32 values: the 128-bit-key configs).
inline int pull_run_delta(const alto_pull_args* a, const PullStage& S, int order, cudaStream_t s) {
  const int vd = a->value_dtype, fd = a->factor_dtype, od = a->out_dtype;
  if (vd != ALTO_F32) return ALTO_EUNSUPPORTED;
  if (fd == ALTO_F32 && od == ALTO_F32)
    return a->atomic ? pull_by_shape<1, float, float, float, true, true>(a, S, order, s)
                     : pull_by_shape<1, float, float, float, false, true>(a, S, order, s);
  if (fd == ALTO_F32 && od == ALTO_F64)
    return a->atomic ? pull_by_shape<1, float, float, double, true, true>(a, S, order, s)
                     : pull_by_shape<1, float, float, double, false, true>(a, S, order, s);
  if (fd == ALTO_F64 && od == ALTO_F64)
    return a->atomic ? pull_by_shape<1, float, double, double, true, true>(a, S, order, s)
                     : pull_by_shape<1, float, double, double, false, true>(a, S, order, s);
  return ALTO_EUNSUPPORTED;
}

template <int W>
int pull_run(const alto_pull_args* a, const PullStage& S, int order, cudaStream_t s) {
  const int vd = a->value_dtype, fd = a->factor_dtype, od = a->out_dtype;
  if (vd == ALTO_F32 && fd == ALTO_F32 && od == ALTO_F32) return pull_by_atomic<W, float, float, float>(a, S, order, s);
  if (vd == ALTO_F32 && fd == ALTO_F32 && od == ALTO_F64) return pull_by_atomic<W, float, float, double>(a, S, order, s);
  if (vd == ALTO_F64 && fd == ALTO_F64 && od == ALTO_F64) return pull_by_atomic<W, double, double, double>(a, S, order, s);
  if (vd == ALTO_F32 && fd == ALTO_F64 && od == ALTO_F64) return pull_by_atomic<W, float, double, double>(a, S, order, s);
  return ALTO_EUNSUPPORTED;
}

int pull_run_w1(const alto_pull_args* a, const PullStage& S, int order, cudaStream_t s);
int pull_run_w2(const alto_pull_args* a, const PullStage& S, int order, cudaStream_t s);
int pull_run_w1_delta(const alto_pull_args* a, const PullStage& S, int order, cudaStream_t s);

}  // namespace alto
